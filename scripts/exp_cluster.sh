#!/bin/bash
# cluster-merge experiment: parity tests, sweep on/off, trace, ncu at the bench state
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_c.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "cluster" > gpurun_out/test_cluster.log 2>&1
for cl in 0 1; do
  KVTIER_CLUSTER=$cl timeout 300 python scripts/sweep_attn.py --splits 4,8 --variants 0,4 --steps 96 > gpurun_out/sweep_cl$cl.log 2>&1
  KVTIER_CLUSTER=$cl timeout 300 python scripts/trace_attn.py --split 8 > gpurun_out/trace_cl$cl.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 7140 -c 1 \
  -o gpurun_out/attn_full_t256 python scripts/prof_step.py --steps 257 > gpurun_out/attn_full_t256.log 2>&1
ls gpurun_out | tail -3
