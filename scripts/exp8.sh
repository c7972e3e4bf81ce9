#!/bin/bash
set -x
T=${1:-c10}
KVT_TRACE_LOOP=1 python -c "from paper_2605_09490_b200 import build; build.build(force=True)" > gpurun_out/build_${T}_tl.log 2>&1
timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace_${T}_tl.log 2>&1
KVTIER_NOSCORE=1 timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace_${T}_tl_nosc.log 2>&1
python -c "from paper_2605_09490_b200 import build; build.build(force=True)" > gpurun_out/build_$T.log 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/test_gpu_${T}.log 2>&1
timeout 300 python scripts/sweep_attn.py --splits 8 --variants 0,4 --steps 96 > gpurun_out/sweep_${T}.log 2>&1
KVTIER_NOSCORE=1 timeout 300 python scripts/sweep_attn.py --splits 8 --variants 0 --steps 96 > gpurun_out/sweep_${T}_nosc.log 2>&1
