#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -q -k "model_decode" > gpurun_out/model_tests.log 2>&1; echo "rc=$?" >> gpurun_out/model_tests.log
timeout 900 python bench.py > gpurun_out/bench_model.log 2>&1; echo "rc=$?" >> gpurun_out/bench_model.log
