#!/bin/bash
# Round-2 evidence for the whole-step kernel: ncu launch list of a short bench, ncu --set full of
# one steady-state k_decode_step launch (cold and warm L2), outputs under gpurun_out/.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
  python bench.py --steps 8 --warmup 3 --no-extras > gpurun_out/launches_r02.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_decode_step -s 6 -c 1 \
  -o gpurun_out/step_full_r02 python scripts/prof_step.py --steps 9 > gpurun_out/step_full_r02.log 2>&1
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_decode_step -s 6 -c 1 \
  -o gpurun_out/step_full_warm_r02 python scripts/prof_step.py --steps 9 > gpurun_out/step_full_warm_r02.log 2>&1
ls -la gpurun_out/*r02*
