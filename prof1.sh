set -x
python bench.py --steps 4 --warmup 2 --no-extras > gpurun_out/bench_small.json 2> gpurun_out/bench_small.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_decode_attn -s 40 -c 2 -o gpurun_out/attn_full python bench.py --steps 3 --warmup 1 --no-extras > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
