#!/bin/bash
set -x
T=${1:-c11}
python -c "from paper_2605_09490_b200 import build; build.build(force=True)" > gpurun_out/build_$T.log 2>&1
for pre in 0 1 2 3; do
  KVTIER_PDL_PRE=$pre timeout 300 python scripts/sweep_attn.py --splits 8 --variants 0 --steps 96 > gpurun_out/sweep_${T}_pre$pre.log 2>&1
done
KVTIER_NOPDL=1 timeout 300 python scripts/sweep_attn.py --splits 8 --variants 0 --steps 96 > gpurun_out/sweep_${T}_nopdl.log 2>&1
KVTIER_PDL_PRE=1 timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace_${T}_pre1.log 2>&1
