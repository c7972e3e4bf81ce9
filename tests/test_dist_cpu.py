"""world_size-2 gloo tests of the request-sharding host logic (no GPU)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_09490_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        el = 1.5 + rank                       # per-rank elapsed seconds
        mx = D.max_over_ranks(el)
        steps = D.sum_over_ranks(192)
        D.barrier_sync()
        seed_off, reqs = D.shard_plan(world, rank, 8)
        q.put((rank, mx, steps, seed_off, reqs))
    finally:
        dist.destroy_process_group()


def test_request_sharding_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, mx0, st0, so0, rq0), (r1, mx1, st1, so1, rq1) = out
    assert mx0 == mx1 == 2.5                  # time = max over ranks
    assert st0 == st1 == 384                  # whole-job steps
    assert so0 != so1                         # independent request streams per rank
    assert set(rq0).isdisjoint(rq1) and sorted(rq0 + rq1) == list(range(16))


def test_shard_plan_rejects_bad_rank():
    with pytest.raises(ValueError):
        D.shard_plan(2, 2, 8)
    assert D.max_over_ranks(3.0) == 3.0      # no process group: identity
