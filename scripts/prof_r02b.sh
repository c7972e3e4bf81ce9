#!/bin/bash
# Round-2 (second pass): sequence-shard bench line on the library communicator, launch list of
# a short bench (event kernels included), and a warm full ncu capture (with source) of one
# steady-state k_decode_step.  Outputs under gpurun_out/.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python bench.py --shard sequence --steps 64 --warmup 8 > gpurun_out/bench_seq.log 2>&1; echo "rc=$?" >> gpurun_out/bench_seq.log
tail -c 1500 gpurun_out/bench_seq.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02b.csv \
  python bench.py --steps 8 --warmup 3 --no-extras > gpurun_out/launches_r02b.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --cache-control none --import-source on -k regex:k_decode_step -s 6 -c 1 \
  -o gpurun_out/step_full_warm_r02b python scripts/prof_step.py --steps 9 > gpurun_out/step_full_warm_r02b.log 2>&1; echo "full rc=$?"
ls -la gpurun_out/
