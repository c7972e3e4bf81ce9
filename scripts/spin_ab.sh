#!/bin/bash
# Same-box A/B: the whole-step kernel's layer-chain waits spinning (product) vs suspended
# (KVT_SLEEP_CHAIN=1 -> -DKVT_SPIN_CHAIN=0), event-free 7B steps (scripts/split_sweep.py, auto shape), two rounds.
for round in 1 2; do
for mode in sleep spin; do
  if [ $mode = sleep ]; then KVT_SLEEP_CHAIN=1 python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$mode.log 2>&1;
  else python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$mode.log 2>&1; fi
  echo "$round $mode $(timeout 300 python scripts/split_sweep.py --splits 0 --steps 112 2>&1 | grep split=)"
done
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
