"""Multi-GPU plumbing: one process per GPU, torch.distributed for the bytes.

* Request sharding (row 1): every rank owns its own batch of B requests (global request
  ids rank*B + b, seeds offset per rank); no collective inside the decode step.
* KV-head sharding (row 2): rank r owns kv heads [r*H_l, (r+1)*H_l) and their q heads;
  the step is local; at a manage event the ranks all-gather S_part (B*H_kv*N_max fp32 in
  total) and each classifies the identical gathered scores (kv_tier_classify_gathered),
  so tiers agree bit-for-bit across ranks and with the unsharded run.
* Sequence sharding (row 3): positions are owned block-cyclically (64-position blocks, block
  k on rank k % world).  Per layer every rank attends its own visible tokens
  (kv_tier_decode_attention_lse: o normalised by its partial sum + (m, l) per head), the
  ranks all-gather (o, m, l) and combine them in rank order (lse_combine: the LSE merge of
  Eq. 3 split by position), and each rank completes its fused score update with the global
  (M, L) (kv_tier_score_update_lse).  At an event the summed S_part (all-gather; each
  position has one owner, so the sum is exact) feeds kv_tier_classify_gathered on every rank.
Timing is the max over ranks."""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_plan(world, rank, B):
    """Weak scaling: every rank runs B requests; returns (seed_offset, global request ids)."""
    if not (0 <= rank < world) or B < 1:
        raise ValueError("bad shard")
    return 1000 * rank, list(range(rank * B, (rank + 1) * B))


def _dev():
    return torch.device("cuda") if dist.get_backend() == "nccl" else torch.device("cpu")


def max_over_ranks(x: float) -> float:
    """Max of a per-rank float across the process group (identity without one)."""
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier_sync():
    """synchronize + barrier + synchronize (bench timing contract)."""
    if torch.cuda.is_available():
        torch.cuda.synchronize()
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
    if torch.cuda.is_available():
        torch.cuda.synchronize()


def kvhead_plan(world, rank, Hq, Hkv):
    """KV-head sharding: (first kv head, kv heads, first q head, q heads) of `rank`."""
    if not (0 <= rank < world) or Hkv % world or Hq % Hkv:
        raise ValueError("H_kv must divide evenly over the ranks and H_q over H_kv")
    hl = Hkv // world
    G = Hq // Hkv
    return rank * hl, hl, rank * hl * G, hl * G


def gather_scores(S_local, group=None):
    """All-gather every rank's S_part [B][H_l][N] into [world][B][H_l][N] (rank order =
    global kv head order).  Works on CUDA (NCCL) and CPU (gloo) tensors."""
    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    x = S_local.contiguous()
    if world == 1:
        return x.unsqueeze(0)
    out = torch.empty((world,) + tuple(x.shape), dtype=x.dtype, device=x.device)
    if x.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, x, group=group)
    elif x.is_cuda:                         # gloo: stage through host memory
        hx = x.cpu()
        ho = torch.empty(out.shape, dtype=x.dtype)
        dist.all_gather(list(ho.unbind(0)), hx, group=group)
        out.copy_(ho)
    else:
        dist.all_gather(list(out.unbind(0)), x, group=group)
    return out


def kvhead_classify(kv, stream=None, group=None):
    """a5 under KV-head sharding: all-gather S_part, then classify the gathered scores."""
    with torch.cuda.stream(stream) if stream is not None else _null():
        S_all = gather_scores(kv.scores_tensor(), group)
        kv.classify_gathered(S_all, S_all.shape[0], stream=stream)
    return S_all


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ------------------------------------------------------------------ sequence sharding
SEQ_BLOCK = 64          # kv_internal.cuh


def seq_owner(pos, world):
    """Rank owning position `pos` (block-cyclic, SEQ_BLOCK positions per block)."""
    return (pos // SEQ_BLOCK) % world


def seq_owned_positions(n, world, rank):
    """Ascending positions below n owned by `rank` (host twin of seq_owned_below / seq_pos_of)."""
    return [p for p in range(n) if seq_owner(p, world) == rank]


def lse_combine(o_parts, lse_parts):
    """Combine per-rank partial attention results in rank order (deterministic) with the library
    kernel kv_tier_lse_combine.  o_parts [W][B][H][d] fp32 CUDA: each rank's o normalised by its
    own partial sum; lse_parts [W][B][H][2]: (m, l) per head, m in the log2 domain, l = sum
    2^(z - m) (a rank without visible tokens has m = -inf, l = 0, o = 0).  Returns (o [B][H][d],
    lse [B][H][2]) with M = max_r m_r, w_r = 2^(m_r - M) l_r, L = sum_r w_r, o = sum_r w_r o_r / L.
    No CPU path: host tensors raise."""
    if not o_parts.is_cuda:
        raise RuntimeError("lse_combine runs the CUDA kernel (kv_tier_lse_combine): CUDA tensors only")
    from . import kvtier as kt
    return kt.lse_combine(o_parts, lse_parts)


def seq_combine(o_local, lse_local, group=None, combine=None):
    """All-gather (o, lse) over the group (NCCL on CUDA tensors, gloo on CPU) and combine them
    (``combine`` defaults to the CUDA kernel; host-logic tests pass their own)."""
    og = gather_scores(o_local.float(), group)
    lg = gather_scores(lse_local, group)
    return (combine or lse_combine)(og, lg)


def seq_classify(kv, stream=None, group=None):
    """a5 under sequence sharding: sum of every rank's S_part (exact: one owner per position)
    via the all-gather, then the identical classify on every rank."""
    with torch.cuda.stream(stream) if stream is not None else _null():
        S_all = gather_scores(kv.scores_tensor(), group)
        kv.classify_gathered(S_all, S_all.shape[0], stream=stream)
    return S_all
