#!/bin/bash
# Code-path check of bench.py's multi-rank (request-sharded) mode on a ONE-GPU box: a copy of
# bench.py with every rank on cuda:0 and gloo for the host-side collectives (ranks never wait on
# each other's kernels in this mode).  Not a measurement: the numbers share one GPU.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
sed -e 's/    local = int(os.environ.get("LOCAL_RANK", "0"))/    local = 0/' \
    -e 's/dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))/dist.init_process_group("gloo")/' \
    bench.py > bench_n2_dryrun.py
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench_n2_dryrun.py --gpus 2 --steps 16 --warmup 4 > gpurun_out/n2_dryrun.log 2>&1; echo "rc=$?"
rm -f bench_n2_dryrun.py
tail -c 1200 gpurun_out/n2_dryrun.log
