#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k host_t1 > gpurun_out/host_t1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/host_t1_tests.log
timeout 900 python bench.py > gpurun_out/bench_h1.log 2>&1
