#!/bin/bash
# Large-config sweep: 14B kernel variants x split, and the 32B config's per-GPU share under
# 2-way request sharding (B=16 of 32) on one B200.
python -c "import __graft_entry__ as g; g.build()" || exit 1
OUT=gpurun_out/large.jsonl; : > $OUT
for var in 0 1 2 3 5; do for sp in 0 1 2; do
  echo "var=$var split=$sp" >> $OUT
  timeout 240 python bench.py --no-extras --config 14b --hbm 5000 --evict 300 --variant $var --split $sp --steps 48 --warmup 16 2>&1 | tail -1 >> $OUT
done; done
echo "32b B=16" >> $OUT
timeout 600 python bench.py --no-extras --config 32b --batch 16 --steps 32 --warmup 8 2>&1 | tail -1 >> $OUT
echo "32b B=16 full" >> $OUT
timeout 900 python bench.py --config 32b --batch 16 --steps 32 --warmup 8 --cpu-seconds 5 2>&1 | tail -1 >> $OUT
