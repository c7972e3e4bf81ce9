#!/bin/bash
# Same-box A/B of the event's host offload: on the ctx's offload stream (product build) vs inside
# the migrate kernel (-DKVT_INLINE_OFFLOAD=1 build), 7B and 14B, two runs each, outputs under gpurun_out/.
for round in 1 2; do
for mode in stream inline; do
  if [ $mode = inline ]; then KVT_INLINE_OFFLOAD=1 python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1;
  else python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; fi
  for cfg in 7b 14b; do
    timeout 600 python bench.py --config $cfg --no-extras --steps 128 --warmup 8 > gpurun_out/ab_${mode}_${cfg}_$round.log 2>&1
    echo "$round $mode $cfg $(grep -o '"value": [0-9.]*' gpurun_out/ab_${mode}_${cfg}_$round.log | head -1) $(grep -o '"t_step_us": [0-9.]*' gpurun_out/ab_${mode}_${cfg}_$round.log) $(grep -o '"t_event_us": [0-9.]*' gpurun_out/ab_${mode}_${cfg}_$round.log)"
  done
done
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
