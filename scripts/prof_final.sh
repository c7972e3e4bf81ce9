#!/bin/bash
# Final round-1 evidence: ncu launch list of a short bench + ncu --set full of one steady-state
# decode / merge / score-flush launch (7B, step 66).
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 8 --warmup 3 --no-extras > gpurun_out/launches_final.log 2>&1
for k in k_decode_attn k_decode_merge k_score_flush; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1848 -c 1 \
    -o gpurun_out/${k}_final python scripts/prof_step.py --steps 67 > gpurun_out/${k}_final.log 2>&1
done
ls -la gpurun_out/*_final*
