#!/bin/bash
# Full GPU parity suite + smoke (round-end check), host-T1 tests first.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -k host_t1 > gpurun_out/host_t1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/host_t1_tests.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gpu_suite.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
