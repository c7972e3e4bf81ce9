#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "redundancy or randomized_configs" > gpurun_out/red_tests.log 2>&1; echo "rc=$?" >> gpurun_out/red_tests.log
OUT=gpurun_out/r32.jsonl; : > $OUT
for a in "--variant 3" "--variant 3 --split 1" "--variant 2 --split 2" "--scorer redundancy" "--scorer combined"; do
  cfg="--config 32b --batch 16"; case "$a" in *scorer*) cfg="";; esac
  echo "$cfg $a" >> $OUT
  timeout 300 python bench.py --no-extras $cfg $a --steps 32 --warmup 8 2>&1 | tail -1 >> $OUT
done
