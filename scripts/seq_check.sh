#!/bin/bash
# Sequence-shard subset of the GPU suite + the sequence-sharded bench line (with the N = 1
# request-sharded comparison rates).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "sequence or lse or host_t1 or step_kernel or randomized" > gpurun_out/seqt.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/seqt.log
timeout 600 python bench.py --shard sequence --steps 64 --warmup 8 > gpurun_out/bench_seq3.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_seq3.log').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['request_sharded_n1'])"
