#!/bin/bash
for d in A B; do (cd scratch_ab/$d && python -c "import __graft_entry__ as g; g.build()") || exit 1; done
OUT=$PWD/gpurun_out/ab_h1.txt; : > $OUT
for i in 1 2 3; do for d in A B; do echo "$d $(cd scratch_ab/$d && timeout 300 python scripts/exp_h1_only.py 2>&1 | tail -1)" >> $OUT; done; done
(cd scratch_ab/B && timeout 600 python -m pytest tests -m gpu -q -k host_t1 2>&1 | tail -1) >> $OUT
