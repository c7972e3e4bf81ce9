#!/bin/bash
# Launch list of the sequence-sharded step graph (N = 1, library NCCL communicator): per-kernel
# serialised times of one step, to split the step into decode / merge / all-gather / combine / score.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python bench.py --shard sequence --steps 64 --warmup 8 > gpurun_out/bench_seq2.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/bench_seq2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/seq_launches.csv python bench.py --shard sequence --steps 4 --warmup 3 \
  > gpurun_out/seq_ncu.log 2>&1; echo "ncu rc=$?"
