#!/bin/bash
set -x
T=${1:-c4}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$T.log 2>&1
KVTIER_CLUSTER=1 timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/test_gpu_${T}_cl1.log 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu -k "cluster" > gpurun_out/test_gpu_${T}_cl0.log 2>&1
for cl in 1 0; do
  KVTIER_CLUSTER=$cl timeout 300 python scripts/sweep_attn.py --splits 4,8 --variants 0,1,4 --steps 96 > gpurun_out/sweep_${T}_cl$cl.log 2>&1
  KVTIER_CLUSTER=$cl timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace_${T}_cl$cl.log 2>&1
done
