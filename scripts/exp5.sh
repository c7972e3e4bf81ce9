#!/bin/bash
set -x
T=${1:-c7}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/test_gpu_${T}.log 2>&1
timeout 300 python scripts/sweep_attn.py --splits 4,8 --variants 0,4 --steps 96 > gpurun_out/sweep_${T}.log 2>&1
timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace_${T}_s8.log 2>&1
timeout 300 python scripts/trace_attn.py --split 8 --variant 4 > gpurun_out/trace_${T}_s8v4.log 2>&1
