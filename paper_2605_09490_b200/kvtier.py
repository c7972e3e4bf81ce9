"""Thin ctypes binding of libkvtier.so (include/kv_tier.h) -- argument marshalling only.

Every step of the path runs in the library's CUDA kernels; PyTorch only provides
device memory (one arena tensor) and streams.  Functions keep the C names.
There is no fallback: if the library or a GPU is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "lib")

KV_TIER_OK = 0
STATUS = {0: "OK", -1: "E_INVAL", -2: "E_CUDA", -3: "E_NCCL", -4: "E_STATE", -5: "E_CAPACITY",
          -6: "E_OOM", -7: "E_NUMERIC"}
EVICT_TOTAL, EVICT_PER_EVENT = 0, 1
SHARD_REQUEST, SHARD_KVHEAD, SHARD_SEQUENCE = 0, 1, 2
POLICY_HIERARCHY, POLICY_STREAMING, POLICY_H2O, POLICY_RANDOM = 0, 1, 2, 3
SCORER_ATTENTION, SCORER_VATP, SCORER_REDUNDANCY, SCORER_COMBINED, SCORER_WINDOW, SCORER_RKV = 0, 1, 2, 3, 4, 5
STAGING_ALL = 0xFFFFFFFF
(X_SCORES, X_TIERS, X_IDX_T0, X_IDX_T1, X_IDX_T2, X_T0_ROWS, X_T1_ROWS, X_STAGING, X_T2_CODES, X_T2_SCALES,
 X_REDUNDANCY, X_SNAPSHOT) = range(12)


class KvTierError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "num_requests", "num_layers", "num_q_heads", "num_kv_heads", "head_dim", "max_tokens",
        "prompt_len", "sink_size", "window_size", "manage_interval")] + [
        ("hbm_ratio_bp", C.c_uint32), ("evict_ratio_bp", C.c_uint32), ("t2_fraction_bp", C.c_uint32),
        ("evict_mode", C.c_int32), ("staging_tokens", C.c_uint32),
        ("device", C.c_int32), ("rank", C.c_int32), ("world", C.c_int32), ("shard", C.c_int32),
        ("out_fp32", C.c_int32), ("split", C.c_int32), ("variant", C.c_int32),
        ("policy", C.c_int32), ("budget", C.c_int32), ("policy_seed", C.c_uint32), ("scorer", C.c_int32),
        ("step_kernel", C.c_int32)]


class Sizes(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in (
        "device_arena", "t0_store", "t1_staging", "t2_store", "scores", "meta", "host_t1", "host_t2")] + [
        ("cap_t0", C.c_int32), ("cap_t1", C.c_int32), ("cap_t2", C.c_int32)]


class Buffers(C.Structure):
    _fields_ = [("device_arena", C.c_void_p)]


_lib = None
_SIGS = {
    "kv_tier_query_sizes": [C.POINTER(Config), C.POINTER(Sizes)],
    "kv_tier_init": [C.POINTER(Config), C.POINTER(Buffers), C.c_void_p, C.POINTER(C.c_void_p)],
    "kv_tier_destroy": [C.c_void_p],
    "kv_tier_nccl_unique_id": [C.c_void_p, C.c_size_t],
    "kv_tier_load_prefix": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p],
    "kv_tier_begin_step": [C.c_void_p, C.c_void_p],
    "kv_tier_append": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p],
    "kv_tier_prefetch": [C.c_void_p, C.c_int32, C.c_void_p],
    "kv_tier_decode_attention": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_int32, C.c_void_p],
    "kv_tier_decode_attention_lse": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_int32, C.c_void_p],
    "kv_tier_score_update_lse": [C.c_void_p, C.c_void_p, C.c_void_p],
    "kv_tier_set_host_t1": [C.c_void_p, C.c_int32],
    "kv_tier_host_t1_attention": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p],
    "kv_tier_host_t1_score_update": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p],
    "kv_tier_host_t1_layer": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p],
    "kv_tier_lse_combine": [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                            C.c_void_p],
    "kv_tier_score_update": [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p],
    "kv_tier_visible_count": [C.c_void_p, C.POINTER(C.c_int32)],
    "kv_tier_layout": [C.c_void_p, C.c_void_p, C.c_void_p],
    "kv_tier_end_step": [C.c_void_p, C.c_void_p],
    "kv_tier_step": [C.c_void_p] + [C.c_void_p] * 4 + [C.c_int32, C.c_void_p, C.c_void_p],
    "kv_tier_step_graph_capture": [C.c_void_p] + [C.c_void_p] * 4 + [C.c_int32, C.c_void_p, C.c_void_p],
    "kv_tier_step_graph_launch": [C.c_void_p, C.c_void_p],
    "kv_tier_capture_begin": [C.c_void_p],
    "kv_tier_capture_end": [C.c_void_p],
    "kv_tier_graph_advance": [C.c_void_p],
    "kv_tier_classify": [C.c_void_p, C.c_void_p],
    "kv_tier_classify_gathered": [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p],
    "kv_tier_scores_device": [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)],
    "kv_tier_migrate": [C.c_void_p, C.c_void_p, C.c_void_p],
    "kv_tier_sync": [C.c_void_p],
    "kv_tier_census": [C.c_void_p, C.c_void_p, C.c_void_p],
    "kv_tier_position": [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
    "kv_tier_export_size": [C.c_void_p, C.c_int32, C.POINTER(C.c_size_t)],
    "kv_tier_export": [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t],
    "kv_tier_import_scores": [C.c_void_p, C.c_void_p, C.c_size_t],
    "kv_tier_debug_trace": [C.c_void_p, C.c_void_p, C.c_size_t],
    "kv_tier_debug_trace_len": [C.c_void_p, C.POINTER(C.c_size_t)],
    "kv_tier_last_error": [C.c_void_p],
    "kv_tier_version": [],
}
EXPORTED = sorted(_SIGS)


def lib_path(name="libkvtier.so"):
    return os.path.join(LIB_DIR, name)


def load():
    """dlopen libkvtier.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        p = lib_path()
        if not os.path.exists(p):
            raise FileNotFoundError(f"{p} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(p)
        for name, args in _SIGS.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = C.c_char_p if name in ("kv_tier_last_error", "kv_tier_version") else C.c_int
        _lib = lib
    return _lib


def _check(st, ctx=None):
    if st != KV_TIER_OK:
        msg = load().kv_tier_last_error(ctx)
        raise KvTierError(st, msg.decode() if msg else "")


def _stream_ptr(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


def make_config(B, L, Hq, Hkv, d, max_tokens, prompt_len, hbm_bp=5000, evict_bp=500, t2_bp=0,
                sink_size=4, window_size=128, manage_interval=64, evict_mode=EVICT_TOTAL,
                staging=STAGING_ALL, device=0, out_fp32=1, split=0, rank=0, world=1, variant=0,
                shard=0, policy=0, budget=0, policy_seed=0, scorer=0, step_kernel=0):
    return Config(num_requests=B, num_layers=L, num_q_heads=Hq, num_kv_heads=Hkv, head_dim=d,
                  max_tokens=max_tokens, prompt_len=prompt_len, sink_size=sink_size,
                  window_size=window_size, manage_interval=manage_interval, hbm_ratio_bp=hbm_bp,
                  evict_ratio_bp=evict_bp, t2_fraction_bp=t2_bp, evict_mode=evict_mode,
                  staging_tokens=staging, device=device, rank=rank, world=world, shard=shard,
                  out_fp32=out_fp32, split=split, variant=variant, policy=policy, budget=budget,
                  policy_seed=policy_seed, scorer=scorer, step_kernel=step_kernel)


NCCL_ID_BYTES = 128


def nccl_unique_id():
    """A fresh ncclUniqueId (bytes) for kv_tier_init: rank 0 draws it, every rank passes it."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    _check(load().kv_tier_nccl_unique_id(buf, NCCL_ID_BYTES))
    return buf.raw


def query_sizes(cfg):
    s = Sizes()
    _check(load().kv_tier_query_sizes(C.byref(cfg), C.byref(s)))
    return s


class KvTier:
    """One ctx.  The device arena is a torch uint8 tensor owned by this object."""

    def __init__(self, cfg: Config, nccl_id: bytes = None):
        """nccl_id: sequence sharding with the library's own communicator (kv_tier_nccl_unique_id
        bytes, identical on every rank); None: no collective inside the library."""
        import torch
        self.cfg = cfg
        self.sizes = query_sizes(cfg)
        self.arena = torch.empty(self.sizes.device_arena, dtype=torch.uint8, device=f"cuda:{cfg.device}")
        buf = Buffers(device_arena=C.c_void_p(self.arena.data_ptr()))
        h = C.c_void_p()
        idb = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), NCCL_ID_BYTES)
        _check(load().kv_tier_init(C.byref(cfg), C.byref(buf), idb, C.byref(h)))
        self.ctx = h

    def close(self):
        if self.ctx:
            load().kv_tier_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- the path (names as in kv_tier.h)
    def load_prefix(self, layer, k, v, n0, stream=None):
        _check(load().kv_tier_load_prefix(self.ctx, layer, C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                          n0, _stream_ptr(stream)), self.ctx)

    def begin_step(self, stream=None):
        _check(load().kv_tier_begin_step(self.ctx, _stream_ptr(stream)), self.ctx)

    def append(self, layer, k_new, v_new, stream=None):
        _check(load().kv_tier_append(self.ctx, layer, C.c_void_p(k_new.data_ptr()), C.c_void_p(v_new.data_ptr()),
                                     _stream_ptr(stream)), self.ctx)

    def prefetch(self, layer, side=None):
        _check(load().kv_tier_prefetch(self.ctx, layer, _stream_ptr(side)), self.ctx)

    def decode_attention(self, layer, q, o, fuse_score_update=1, stream=None, k_new=None, v_new=None):
        """k_new/v_new: fused append of the new token's row (None: kv_tier_append was called)."""
        kp = C.c_void_p(k_new.data_ptr()) if k_new is not None else None
        vp = C.c_void_p(v_new.data_ptr()) if v_new is not None else None
        _check(load().kv_tier_decode_attention(self.ctx, layer, C.c_void_p(q.data_ptr()), kp, vp,
                                               C.c_void_p(o.data_ptr()), fuse_score_update, _stream_ptr(stream)),
               self.ctx)

    def decode_attention_lse(self, layer, q, o, lse, fuse_score_update=1, stream=None, k_new=None, v_new=None):
        """As decode_attention, o normalised by this ctx's partial sum; lse [B][H_q][2] fp32 gets
        (max in the log2 domain, sum) per head (sequence sharding)."""
        kp = C.c_void_p(k_new.data_ptr()) if k_new is not None else None
        vp = C.c_void_p(v_new.data_ptr()) if v_new is not None else None
        _check(load().kv_tier_decode_attention_lse(self.ctx, layer, C.c_void_p(q.data_ptr()), kp, vp,
                                                   C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()),
                                                   fuse_score_update, _stream_ptr(stream)), self.ctx)

    def score_update_lse(self, lse_global, stream=None):
        _check(load().kv_tier_score_update_lse(self.ctx, C.c_void_p(lse_global.data_ptr()), _stream_ptr(stream)),
               self.ctx)

    # N1 host-T1 mode (kv_tier_set_host_t1): host tensors are CPU (ideally pinned) torch tensors
    def set_host_t1(self, on=True):
        _check(load().kv_tier_set_host_t1(self.ctx, 1 if on else 0), self.ctx)

    def host_t1_attention(self, layer, q_host, o_part, lse_part):
        """T1 partial of `layer` on the host cores: q_host bf16 [B][H_q][d] -> o_part fp32
        [B][H_q][d], lse_part fp32 [B][H_q][2] (CPU tensors)."""
        for x in (q_host, o_part, lse_part):
            if x.is_cuda or not x.is_contiguous():
                raise ValueError("host_t1_attention takes contiguous CPU tensors")
        _check(load().kv_tier_host_t1_attention(self.ctx, layer, C.c_void_p(q_host.data_ptr()),
                                                C.c_void_p(o_part.data_ptr()), C.c_void_p(lse_part.data_ptr())),
               self.ctx)

    def host_t1_score_update(self, layer, lse_global_host, stream=None):
        if lse_global_host.is_cuda or not lse_global_host.is_contiguous():
            raise ValueError("host_t1_score_update takes a contiguous CPU lse tensor")
        _check(load().kv_tier_host_t1_score_update(self.ctx, layer, C.c_void_p(lse_global_host.data_ptr()),
                                                   _stream_ptr(stream)), self.ctx)

    def host_t1_layer(self, layer, q, o, stream=None, k_new=None, v_new=None):
        """One whole host-T1 layer (kv_tier_host_t1_layer): o fp32 [B][H_q][d] on the device."""
        kp = C.c_void_p(k_new.data_ptr()) if k_new is not None else None
        vp = C.c_void_p(v_new.data_ptr()) if v_new is not None else None
        _check(load().kv_tier_host_t1_layer(self.ctx, layer, C.c_void_p(q.data_ptr()), kp, vp,
                                            C.c_void_p(o.data_ptr()), _stream_ptr(stream)), self.ctx)

    def score_update(self, layer, probs, stream=None):
        _check(load().kv_tier_score_update(self.ctx, layer, C.c_void_p(probs.data_ptr()), _stream_ptr(stream)),
               self.ctx)

    def visible_count(self):
        n = C.c_int32()
        _check(load().kv_tier_visible_count(self.ctx, C.byref(n)), self.ctx)
        return n.value

    def layout(self):
        """(tier counts [T0, T1, T2, T3] of the current layout, step-kernel shape [CTAs, CTAs per
        kv head, kv heads per CTA, consumer warps]) from the host mirror (no device sync)."""
        c = np.zeros(4, dtype=np.int32)
        sh = np.zeros(4, dtype=np.int32)
        _check(load().kv_tier_layout(self.ctx, c.ctypes.data_as(C.c_void_p), sh.ctypes.data_as(C.c_void_p)), self.ctx)
        return c.tolist(), sh.tolist()

    def end_step(self, stream=None):
        _check(load().kv_tier_end_step(self.ctx, _stream_ptr(stream)), self.ctx)

    def step(self, q, k_new, v_new, o, fuse_score_update=1, stream=None, side=None):
        _check(load().kv_tier_step(self.ctx, *(C.c_void_p(x.data_ptr()) for x in (q, k_new, v_new, o)),
                                   fuse_score_update, _stream_ptr(stream), _stream_ptr(side)), self.ctx)

    def step_graph_capture(self, q, k_new, v_new, o, fuse_score_update=1, stream=None, side=None):
        _check(load().kv_tier_step_graph_capture(self.ctx, *(C.c_void_p(x.data_ptr()) for x in (q, k_new, v_new, o)),
                                                 fuse_score_update, _stream_ptr(stream), _stream_ptr(side)), self.ctx)

    def step_graph_launch(self, stream=None):
        _check(load().kv_tier_step_graph_launch(self.ctx, _stream_ptr(stream)), self.ctx)

    def capture_begin(self):
        """Open an external capture (the caller's CUDA graph records this ctx's step calls)."""
        _check(load().kv_tier_capture_begin(self.ctx), self.ctx)

    def capture_end(self):
        _check(load().kv_tier_capture_end(self.ctx), self.ctx)

    def graph_advance(self):
        """Advance the host state machine by the one step a replay of the caller's graph ran."""
        _check(load().kv_tier_graph_advance(self.ctx), self.ctx)

    def classify(self, stream=None):
        _check(load().kv_tier_classify(self.ctx, _stream_ptr(stream)), self.ctx)

    def classify_gathered(self, S_all, parts, stream=None):
        """a5 from all-gathered scores: S_all is a contiguous fp32 CUDA tensor
        [parts][B][H_kv][N_max] (KV-head sharding, rank order = global head order)."""
        assert S_all.is_cuda and S_all.dtype.itemsize == 4 and S_all.is_contiguous()
        _check(load().kv_tier_classify_gathered(self.ctx, C.c_void_p(S_all.data_ptr()), parts, _stream_ptr(stream)),
               self.ctx)

    def scores_tensor(self):
        """Zero-copy torch view [B][H_kv][N_max] fp32 of this ctx's S_part (inside the arena)."""
        ptr, nbytes = C.c_void_p(), C.c_size_t()
        _check(load().kv_tier_scores_device(self.ctx, C.byref(ptr), C.byref(nbytes)), self.ctx)
        off = ptr.value - self.arena.data_ptr()
        assert 0 <= off and off + nbytes.value <= self.arena.numel()
        B, H = self.cfg.num_requests, self.cfg.num_kv_heads
        return self.arena[off:off + nbytes.value].view(dtype=__import__("torch").float32).view(B, H, -1)

    def migrate(self, stream=None, side=None):
        _check(load().kv_tier_migrate(self.ctx, _stream_ptr(stream), _stream_ptr(side)), self.ctx)

    def sync(self):
        _check(load().kv_tier_sync(self.ctx), self.ctx)

    def census(self):
        counts = np.zeros((self.cfg.num_requests, 4), dtype=np.int32)
        rows = C.c_int64()
        _check(load().kv_tier_census(self.ctx, counts.ctypes.data_as(C.c_void_p), C.byref(rows)), self.ctx)
        return counts, rows.value

    def position(self):
        n, t = C.c_int32(), C.c_int32()
        _check(load().kv_tier_position(self.ctx, C.byref(n), C.byref(t)), self.ctx)
        return n.value, t.value

    def export(self, what, layer=0):
        """Canonical (ascending-position) export.  Per-request results are stacked into one
        array when every request has the same counts (always, except under sequence sharding,
        where a list of per-request arrays is returned)."""
        nbytes = C.c_size_t()
        _check(load().kv_tier_export_size(self.ctx, what, C.byref(nbytes)), self.ctx)
        buf = np.zeros(nbytes.value, dtype=np.uint8)
        _check(load().kv_tier_export(self.ctx, what, layer, buf.ctypes.data_as(C.c_void_p), nbytes.value), self.ctx)
        B, H, D = self.cfg.num_requests, self.cfg.num_kv_heads, self.cfg.head_dim
        if what in (X_SCORES, X_REDUNDANCY, X_SNAPSHOT):
            return buf.view(np.float32).reshape(B, H, -1)
        if what == X_TIERS:
            return buf.reshape(B, -1)
        counts, _ = self.census()
        T = {X_IDX_T0: 0, X_IDX_T1: 1, X_IDX_T2: 2, X_T0_ROWS: 0, X_T1_ROWS: 1, X_STAGING: 1,
             X_T2_CODES: 2, X_T2_SCALES: 2}[what]
        if what in (X_IDX_T0, X_IDX_T1, X_IDX_T2):
            per, dt, shape = 4, np.int32, lambda c: (c,)
        elif what in (X_T0_ROWS, X_T1_ROWS, X_STAGING):
            per, dt, shape = H * 2 * D * 2, np.uint16, lambda c: (H, c, 2, D)
        elif what == X_T2_CODES:
            per, dt, shape = H * 2 * D, np.int8, lambda c: (H, c, 2, D)
        else:
            per, dt, shape = H * 2 * 4, np.float32, lambda c: (H, c, 2)
        out, off = [], 0
        for b in range(B):
            c = int(counts[b][T])
            out.append(buf[off:off + c * per].view(dt).reshape(shape(c)))
            off += c * per
        assert off == buf.size
        return np.stack(out) if len({x.shape for x in out}) == 1 else out

    def debug_trace(self):
        """[L][CTAs][NTRACE] %globaltimer ns checkpoints of the last step (KVTIER_TRACE=1)."""
        ln = C.c_size_t(0)
        _check(load().kv_tier_debug_trace_len(self.ctx, C.byref(ln)), self.ctx)
        n = ln.value
        buf = np.zeros(n, dtype=np.uint64)
        _check(load().kv_tier_debug_trace(self.ctx, buf.ctypes.data_as(C.c_void_p), n), self.ctx)
        return buf.reshape(self.cfg.num_layers, -1, NTRACE)

    def _split(self):
        if self.cfg.split:
            return self.cfg.split
        units = self.cfg.num_requests * self.cfg.num_kv_heads
        return max(1, min(8, (2 * 148) // units))

    def import_scores(self, S):
        S = np.ascontiguousarray(S, dtype=np.float32)
        _check(load().kv_tier_import_scores(self.ctx, S.ctypes.data_as(C.c_void_p), S.nbytes), self.ctx)


NTRACE = 24            # trace slots per CTA (kv_internal.cuh)


def lse_combine(o_parts, lse_parts, stream=None):
    """Rank combine of sequence-shard partials on the GPU (kv_tier_lse_combine): o_parts
    [W][..., d] fp32, lse_parts [W][..., 2] fp32 (contiguous CUDA tensors) -> (o, lse)."""
    import torch
    assert o_parts.is_cuda and o_parts.dtype == torch.float32 and lse_parts.dtype == torch.float32
    o_parts, lse_parts = o_parts.contiguous(), lse_parts.contiguous()
    W, d = o_parts.shape[0], o_parts.shape[-1]
    rows = o_parts[0].numel() // d
    o = torch.empty(o_parts.shape[1:], dtype=torch.float32, device=o_parts.device)
    lse = torch.empty(lse_parts.shape[1:], dtype=torch.float32, device=o_parts.device)
    s = stream if stream is not None else torch.cuda.current_stream(o_parts.device)
    _check(load().kv_tier_lse_combine(C.c_void_p(o_parts.data_ptr()), C.c_void_p(lse_parts.data_ptr()), W, rows, d,
                                      C.c_void_p(o.data_ptr()), C.c_void_p(lse.data_ptr()), _stream_ptr(s)))
    return o, lse


def version():
    return load().kv_tier_version().decode()
