#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
KVTIER_ZRING=2 timeout 900 python -m pytest tests -m gpu -x -q -k "tiny_32 or multi_request or 7b_sampled or randomized_configs or redundancy" > gpurun_out/zring_tests.log 2>&1; echo "rc=$?" >> gpurun_out/zring_tests.log
OUT=gpurun_out/zring.jsonl; : > $OUT
for z in 2 4; do
  echo "32b B=16 zring=$z" >> $OUT
  KVTIER_ZRING=$z timeout 300 python bench.py --no-extras --config 32b --batch 16 --steps 32 --warmup 8 2>&1 | tail -1 >> $OUT
done
for z in 2 3 4; do
  echo "14b zring=$z" >> $OUT
  KVTIER_ZRING=$z timeout 300 python bench.py --no-extras --config 14b --evict 300 --steps 48 --warmup 16 2>&1 | tail -1 >> $OUT
done
for z in 2 4; do
  echo "7b zring=$z" >> $OUT
  KVTIER_ZRING=$z timeout 300 python bench.py --no-extras --steps 192 --warmup 64 2>&1 | tail -1 >> $OUT
done
