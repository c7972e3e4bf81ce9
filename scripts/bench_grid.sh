#!/bin/bash
# Round evidence: 7B beta x r grid, 14B line, and an ncu --set full capture of one
# steady-state decode_attention launch (step 66 of 7B beta50/r5) for roofline.traffic.
TAG=${1:-r01}
python -c "import __graft_entry__ as g; g.build()"
: > gpurun_out/grid_$TAG.jsonl
for hbm in 3000 5000 7000; do for ev in 300 500 1000; do
  timeout 300 python bench.py --no-extras --hbm $hbm --evict $ev --steps 128 --warmup 64 2>/dev/null >> gpurun_out/grid_$TAG.jsonl
done; done
timeout 600 python bench.py --no-extras --config 14b --hbm 5000 --evict 300 --steps 64 --warmup 64 2>/dev/null >> gpurun_out/grid_$TAG.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 1848 -c 1 \
  -o gpurun_out/attn_steady_$TAG python scripts/prof_step.py --steps 67 > gpurun_out/attn_steady_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_merge -s 1848 -c 1 \
  -o gpurun_out/merge_steady_$TAG python scripts/prof_step.py --steps 67 > gpurun_out/merge_steady_$TAG.log 2>&1
wc -l gpurun_out/grid_$TAG.jsonl
