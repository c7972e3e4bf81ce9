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


def _kvhead_worker(rank, world, port, q):
    import numpy as np
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, Hkv, N = 3, 4, 50
        h0, hl, q0, ql = D.kvhead_plan(world, rank, 16, Hkv)
        full = np.random.default_rng(7).random((B, Hkv, N), dtype=np.float32) * 100
        S_local = torch.from_numpy(full[:, h0:h0 + hl].copy())
        g = D.gather_scores(S_local)                       # [world][B][hl][N]
        q.put((rank, (h0, hl, q0, ql), g.numpy()))
    finally:
        dist.destroy_process_group()


def test_kvhead_gather_gloo_world2():
    """KV-head sharding host logic: the all-gather puts shards in global head order, and the
    ascending-head fp32 sum over the gathered parts is bitwise the unsharded S_i (AMB-14)."""
    import numpy as np
    from oracle import kvtier_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_kvhead_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=120) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, plan0, g0), (r1, plan1, g1) = out
    assert plan0 == (0, 2, 0, 8) and plan1 == (2, 2, 8, 8)
    assert np.array_equal(g0, g1)                          # every rank sees the same bytes
    full = np.random.default_rng(7).random((3, 4, 50), dtype=np.float32) * 100
    glob = np.concatenate(list(g0), axis=1)                # [B][H_kv][N] in global head order
    assert np.array_equal(glob, full)
    # the classify kernel's order: global head 0, 1, 2, 3 (ascending), fp32 adds
    s = glob[:, 0].copy()
    for h in range(1, 4):
        s = (s + glob[:, h]).astype(np.float32)
    for b in range(3):
        assert np.array_equal(s[b], O.total_score_fp32(full[b]))


def test_kvhead_plan_rejects_uneven():
    with pytest.raises(ValueError):
        D.kvhead_plan(3, 0, 16, 4)


# --------------------------------------------------------------------- sequence sharding
def _seq_worker(rank, world, port, q):
    """Each rank holds the keys/values of its own 64-position blocks; the all-gathered LSE
    combine must equal softmax attention over the whole sequence (float64 reference)."""
    import numpy as np
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(5)
        n, B, H, d = 300, 2, 3, 16
        qv = torch.randn(B, H, d, generator=g, dtype=torch.float64)
        K = torch.randn(B, n, d, generator=g, dtype=torch.float64)
        V = torch.randn(B, n, d, generator=g, dtype=torch.float64)
        z = torch.einsum("bhd,bnd->bhn", qv, K) / np.sqrt(d) * np.log2(np.e)      # log2 domain
        ref = torch.einsum("bhn,bnd->bhd", torch.softmax(z * np.log(2), dim=-1), V)
        own = torch.tensor(D.seq_owned_positions(n, world, rank))
        zl = z[:, :, own]
        m = zl.max(dim=-1).values
        p = torch.exp2(zl - m.unsqueeze(-1))
        l = p.sum(dim=-1)
        o_local = torch.einsum("bhn,bnd->bhd", p, V[:, own]) / l.unsqueeze(-1)
        o, lse = D.seq_combine(o_local, torch.stack([m, l], dim=-1), combine=_cpu_lse_combine)
        M_ref = z.max(dim=-1).values
        L_ref = torch.exp2(z - M_ref.unsqueeze(-1)).sum(dim=-1)
        q.put((rank, float((o.double() - ref).abs().max()), float((lse[..., 0].double() - M_ref).abs().max()),
               float(((lse[..., 1].double() - L_ref) / L_ref).abs().max()), own.tolist()[:3]))
    finally:
        dist.destroy_process_group()


def _cpu_lse_combine(o_parts, lse_parts):
    """Test-side twin of kv_tier_lse_combine for CPU tensors (the product has no CPU path):
    M = max_r m_r, w_r = 2^(m_r - M) l_r (0 for an empty shard), o = sum_r w_r o_r / sum_r w_r."""
    import torch
    m, l = lse_parts[..., 0], lse_parts[..., 1]
    M = m.max(dim=0).values
    w = torch.where(torch.isinf(m), torch.zeros_like(l), torch.exp2(m - M) * l)
    L = w.sum(dim=0)
    return (w.unsqueeze(-1) * o_parts).sum(dim=0) / L.unsqueeze(-1), torch.stack([M, L], dim=-1)


def test_product_lse_combine_has_no_cpu_path():
    import torch
    with pytest.raises(RuntimeError):
        D.lse_combine(torch.zeros(2, 1, 1, 4), torch.zeros(2, 1, 1, 2))


@pytest.mark.parametrize("world", [2, 3])
def test_sequence_sharding_lse_combine_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seq_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err_o, err_m, err_l, first in out:
        assert err_o < 1e-5 and err_m < 1e-6 and err_l < 1e-6, (rank, err_o, err_m, err_l)   # fp32 gather
        assert first == [64 * rank, 64 * rank + 1, 64 * rank + 2]


def test_sequence_ownership_formulas():
    # host twins of seq_owned_below / seq_pos_of (kv_internal.cuh) against brute force
    for world in (1, 2, 3, 8):
        for rank in range(world):
            owned = D.seq_owned_positions(1000, world, rank)
            for n in (0, 1, 63, 64, 65, 200, 999, 1000):
                assert sum(1 for p in owned if p < n) == _owned_below(world, rank, n)
            for j, p in enumerate(owned):
                assert _pos_of(world, rank, j) == p


def _owned_below(w, r, n):        # transcription of seq_owned_below
    if w <= 1:
        return n
    full, rem = n // 64, n % 64
    c = (full // w) * 64 + (64 if full % w > r else 0)
    return c + (rem if full % w == r else 0)


def _pos_of(w, r, j):             # transcription of seq_pos_of
    return j if w <= 1 else ((j // 64) * w + r) * 64 + j % 64
