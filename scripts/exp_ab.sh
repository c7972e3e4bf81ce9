#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
(cd scratch_ab/old && python -c "import __graft_entry__ as g; g.build()") || exit 1
OUT=$PWD/gpurun_out/ab.txt; : > $OUT
run() { (cd $1 && timeout 300 python bench.py --no-extras --steps 192 --warmup 64 2>/dev/null) | python -c "import json,sys; j=json.loads(sys.stdin.readlines()[-1]); print(round(j['value'],1))"; }
for i in 1 2 3; do
  for d in scratch_ab/old .; do echo "$d $(run $d)" >> $OUT; done
done
timeout 600 python -m pytest tests -m gpu -x -q -k "tiny_32 or multi_request or 7b_sampled or randomized_configs or host_t1 or redundancy" >> $OUT 2>&1
