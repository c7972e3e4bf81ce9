#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "rc=$?" >> gpurun_out/bench_final.log
timeout 600 python bench.py --config 32b --batch 16 --steps 32 --warmup 8 --cpu-seconds 5 > gpurun_out/bench_32b.log 2>&1
timeout 600 python bench.py --config 14b --evict 300 --steps 48 --warmup 16 --cpu-seconds 5 > gpurun_out/bench_14b.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
