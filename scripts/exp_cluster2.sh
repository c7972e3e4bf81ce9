#!/bin/bash
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_c3.log 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/test_gpu_c3.log 2>&1
for cl in 0 1; do
  KVTIER_CLUSTER=$cl timeout 300 python scripts/sweep_attn.py --splits 2,4,8 --variants 0,1,4 --steps 96 > gpurun_out/sweep3_cl$cl.log 2>&1
  KVTIER_CLUSTER=$cl timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace3_cl$cl.log 2>&1
done
