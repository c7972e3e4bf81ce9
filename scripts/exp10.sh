#!/bin/bash
set -x
T=${1:-c12}
python -c "from paper_2605_09490_b200 import build; build.build(force=True)" > gpurun_out/build_$T.log 2>&1
for pf in 1 0; do
  KVTIER_L2PF=$pf timeout 300 python scripts/sweep_attn.py --splits 4,8 --variants 0,4 --steps 96 > gpurun_out/sweep_${T}_pf$pf.log 2>&1
done
KVTIER_L2PF=1 KVTIER_PDL_PRE=1 timeout 300 python scripts/sweep_attn.py --splits 8 --variants 0,4 --steps 96 > gpurun_out/sweep_${T}_pf1_pre1.log 2>&1
KVTIER_L2PF=1 timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace_${T}_pf1.log 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/test_gpu_${T}.log 2>&1
