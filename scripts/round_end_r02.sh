#!/bin/bash
# Round-2 final evidence: full GPU suite, smoke, default bench line, ncu launch list of a short
# bench and a warm full capture (with source) of one steady-state k_decode_step of the final build.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_suite.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_suite.log
tail -3 gpurun_out/gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "rc=$?" >> gpurun_out/bench_final.log
tail -c 300 gpurun_out/bench_final.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final_r02.csv \
  python bench.py --steps 8 --warmup 3 --no-extras > gpurun_out/launches_final_r02.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_decode_step -s 6 -c 1 \
  -o gpurun_out/step_full_final_r02 python scripts/prof_step.py --steps 9 > gpurun_out/step_full_final_r02.log 2>&1; echo "full rc=$?"
