#!/bin/bash
# Full GPU suite, smoke, then the larger-config bench lines (14B configs[2]; 70B configs[4] one
# rank's share of the 8-way sequence split) -- outputs under gpurun_out/.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_suite.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_suite.log
tail -3 gpurun_out/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config 14b --steps 64 --warmup 8 --no-extras > gpurun_out/bench_14b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_14b.log
timeout 900 python bench.py --config 70b --positions 2048 --steps 32 --warmup 8 --no-extras > gpurun_out/bench_70b_share.log 2>&1; echo "rc=$?" >> gpurun_out/bench_70b_share.log
for f in gpurun_out/bench_14b.log gpurun_out/bench_70b_share.log; do echo $f; grep -o '"value": [0-9.]*' $f | head -1; grep -o '"frac": [0-9.]*' $f; tail -1 $f; done
