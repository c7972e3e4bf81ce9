#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
OUT=gpurun_out/score_exp.txt; : > $OUT
timeout 300 python scripts/exp_noscore.py >> $OUT 2>&1
run() { timeout 300 python bench.py --no-extras --steps 192 --warmup 64 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.readlines()[-1]); print(round(j['value'],1))"; }
for g in 37 74 148 296; do echo "grid=$g $(KVTIER_SCORE_GRID=$g run)" >> $OUT; done
echo "lean $(KVTIER_SCORE_LEAN=1 run)" >> $OUT
echo "lean grid=296 $(KVTIER_SCORE_LEAN=1 KVTIER_SCORE_GRID=296 run)" >> $OUT
