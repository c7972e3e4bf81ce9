"""Seeded synthetic inputs for the tiered-decode hot path (CPU twin).

This module is the ONE piece of code shared by the oracle and the CUDA path
(test plumbing only): it turns (seed, tensor id, indices) into bf16 K/V/q rows
and fp32 score fixtures.  It holds none of the method's arithmetic (no
softmax, no scoring, no classification, no quantisation).

The GPU twin is ``synth.cu`` (``libkvsynth.so``); both implement the same
integer-only counter hash, so the bf16 bit patterns are byte-identical
(checked by ``tests/test_gpu_parity.py::test_synth_gpu_matches_cpu``).

Recipe:
  * hash      splitmix64 chain over (seed, tensor id, i0, i1, i2, i3) -> row key;
              element u = splitmix64(row_key + dim)                 (wrapping u64)
  * normal    x = (sum of the four 16-bit fields of u - 131070) * 2^-15
              (integer-exact in fp32; mean 0, std 1.1547)
  * salience  a[b,pos] = x * SIG_A, sinks (positions P..P+k_s-1) get + 4*SIG_A
              (persistent per-token importance shared by all layers/heads, so the
              cumulative score has the long tail of PAPER.md §2.1)
  * direction w[l,g,dim] = +-W_MAG (sign = top hash bit)
  * K = bf16(x*SIG_K + a*w), V = bf16(x*SIG_V), q = bf16(x*SIG_Q + C_Q*w[l, h//G])
All fp32 products/sums are single IEEE round-to-nearest operations (no FMA), and
fp32 -> bf16 is round-to-nearest-even on the bit pattern.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# tensor ids
TID_K, TID_V, TID_Q, TID_SAL, TID_DIR, TID_SCORE = 0, 1, 2, 3, 4, 5

# fp32 constants of the recipe (identical literals in synth.cu)
SIG_K = np.float32(0.8660254)
SIG_V = np.float32(0.8660254)
SIG_Q = np.float32(0.8660254)
C_Q = np.float32(1.0)
W_MAG = np.float32(0.25)
SIG_A_DEFAULT = np.float32(1.125)   # calibrated: cumulative top-20% share 0.566 at t=64 (P:76 says 0.565)
TWO_M15 = np.float32(2.0 ** -15)


def splitmix64(x):
    """splitmix64 finaliser on uint64 numpy arrays/scalars (wrapping)."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def row_key(seed, tid, i0, i1, i2, i3):
    """Chain-hash the row coordinates; every argument may be a broadcastable array."""
    h = splitmix64(np.uint64(seed))
    for f in (tid, i0, i1, i2, i3):
        h = splitmix64(h ^ np.asarray(f, dtype=np.int64).astype(np.uint64))
    return h


def gauss_from_u64(u):
    """Integer-only approx N(0, 1.1547^2) -> float32 (exact)."""
    u = np.asarray(u, dtype=np.uint64)
    m = np.uint64(0xFFFF)
    s = (u & m).astype(np.int64) + ((u >> np.uint64(16)) & m).astype(np.int64) \
        + ((u >> np.uint64(32)) & m).astype(np.int64) + (u >> np.uint64(48)).astype(np.int64)
    return (s - 131070).astype(np.float32) * TWO_M15


def elem_u64(key, d):
    """u64 per element: splitmix64(key + dim) for dim in [0, d) (appended axis)."""
    with np.errstate(over="ignore"):
        return splitmix64(np.asarray(key, dtype=np.uint64)[..., None] + np.arange(d, dtype=np.uint64))


def f32_to_bf16_bits(x):
    """fp32 -> bf16 round-to-nearest-even, returned as uint16 bit patterns (no NaNs here)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    return ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32(b):
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def salience(seed, b_idx, pos, prompt_len, sink_size, sig_a=SIG_A_DEFAULT):
    """a[b,pos] (float32), shapes broadcast."""
    b_idx = np.asarray(b_idx, dtype=np.int64)
    pos = np.asarray(pos, dtype=np.int64)
    key = row_key(seed, TID_SAL, b_idx, pos, 0, 0)
    a = gauss_from_u64(splitmix64(key)) * np.float32(sig_a)
    sink = (pos >= prompt_len) & (pos < prompt_len + sink_size)
    return np.where(sink, a + np.float32(4.0) * np.float32(sig_a), a).astype(np.float32)


def direction(seed, layer, g, d):
    """w[layer, g, :] = +-W_MAG, float32 [..., d]."""
    key = row_key(seed, TID_DIR, layer, g, 0, 0)
    u = elem_u64(key, d)
    return np.where((u >> np.uint64(63)) == np.uint64(1), -W_MAG, W_MAG).astype(np.float32)


def gen_kv(seed, which, L, B, Hkv, d, pos0, npos, prompt_len, sink_size,
           sig_a=SIG_A_DEFAULT, layers=None, reqs=None, heads=None):
    """bf16 bits [L'][B'][H'][npos][d] of K (which='k') or V (which='v') for positions
    pos0..pos0+npos-1.  ``layers/reqs/heads`` select subsets (default: all)."""
    layers = np.arange(L) if layers is None else np.asarray(layers)
    reqs = np.arange(B) if reqs is None else np.asarray(reqs)
    heads = np.arange(Hkv) if heads is None else np.asarray(heads)
    pos = np.arange(pos0, pos0 + npos, dtype=np.int64)
    lg, bg, hg, pg = np.meshgrid(layers, reqs, heads, pos, indexing="ij")
    tid = TID_K if which == "k" else TID_V
    x = gauss_from_u64(elem_u64(row_key(seed, tid, lg, bg, hg, pg), d))
    if which == "v":
        return f32_to_bf16_bits(x * SIG_V)
    a = salience(seed, bg, pg, prompt_len, sink_size, sig_a)          # [..]
    w = np.stack([np.stack([direction(seed, l, g, d) for g in heads]) for l in layers])  # [L'][H'][d]
    w = w[:, None, :, None, :]                                          # [L'][1][H'][1][d]
    return f32_to_bf16_bits(x * SIG_K + a[..., None] * w)


def gen_q(seed, t0, T, L, B, Hq, Hkv, d, layers=None, reqs=None):
    """bf16 bits [T][L'][B'][Hq][d] of the decode queries for steps t0..t0+T-1."""
    G = Hq // Hkv
    layers = np.arange(L) if layers is None else np.asarray(layers)
    reqs = np.arange(B) if reqs is None else np.asarray(reqs)
    ts = np.arange(t0, t0 + T, dtype=np.int64)
    tg, lg, bg, hg = np.meshgrid(ts, layers, reqs, np.arange(Hq), indexing="ij")
    x = gauss_from_u64(elem_u64(row_key(seed, TID_Q, tg, lg, bg, hg), d))
    w = np.stack([np.stack([direction(seed, l, h // G, d) for h in range(Hq)]) for l in layers])  # [L'][Hq][d]
    w = w[None, :, None, :, :]
    return f32_to_bf16_bits(x * SIG_Q + C_Q * w)


def gen_scores(seed, B, Hkv, N, kind="ties"):
    """Synthetic per-kv-head partial scores S_part [B][Hkv][N] float32 (classify fixtures).

    kind='ties': multiples of 1/16 in [0, 6) -> many exact ties across positions
    kind='cont': continuous-looking positive values (all bits used)."""
    bg, hg, pg = np.meshgrid(np.arange(B), np.arange(Hkv), np.arange(N), indexing="ij")
    u = splitmix64(row_key(seed, TID_SCORE, bg, hg, pg, 0))
    if kind == "ties":
        return ((u % np.uint64(96)).astype(np.float32) * np.float32(0.0625)).astype(np.float32)
    # uniform in (0, 8): 24-bit mantissa fraction
    return (((u >> np.uint64(40)).astype(np.float32) + np.float32(1.0)) * np.float32(2.0 ** -21)).astype(np.float32)


# ---------------------------------------------------------------- workloads
# BASELINE.json configs (shapes), SURVEY §8(d) (P, beta, r, seeds; AMB-22/23).
WORKLOADS = {
    "tiny": dict(B=1, L=1, Hq=4, Hkv=2, d=64, N=256, P=16, hbm_bp=5000, evict_bp=500,
                 steps=32, seed=1),
    "7b": dict(B=8, L=28, Hq=28, Hkv=4, d=128, N=2000, P=64, hbm_bp=5000, evict_bp=500,
               steps=256, seed=2),
    "14b": dict(B=16, L=48, Hq=40, Hkv=8, d=128, N=4096, P=64, hbm_bp=5000, evict_bp=300,
                steps=256, seed=3),
    "32b": dict(B=32, L=64, Hq=40, Hkv=8, d=128, N=8192, P=64, hbm_bp=5000, evict_bp=500,
                steps=256, seed=4),
    "70b": dict(B=64, L=80, Hq=64, Hkv=8, d=128, N=16384, P=64, hbm_bp=5000, evict_bp=500,
                steps=256, seed=5),
}
SINK_SIZE, WINDOW_SIZE, MANAGE_INTERVAL = 4, 128, 64
