#!/bin/bash
# One GPU call: build, full bench line, ncu launch list of a short bench, ncu --set full of the
# decode-attention kernel (traffic per launch).  Outputs under gpurun_out/.
set -x
TAG=${1:-r01}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 8 --warmup 3 --no-extras \
  > gpurun_out/ncu_bench_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 30 -c 1 \
  -o gpurun_out/attn_full_$TAG python scripts/prof_step.py > gpurun_out/attn_full_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_decode_merge -s 30 -c 1 \
  -o gpurun_out/merge_full_$TAG python scripts/prof_step.py > gpurun_out/merge_full_$TAG.log 2>&1
ls -la gpurun_out
