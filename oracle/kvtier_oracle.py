"""CPU oracle of the tiered-decode hot path (arXiv 2605.09490) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path (the CUDA
library behind ``include/kv_tier.h``) never calls it and shares no code with it;
the only common code is the seeded input generator
``paper_2605_09490_b200/synth/synth.py`` (no method arithmetic).

Plain, slow, obviously-correct definitions, fp64 except where the paper's
reading fixes fp32 (scores, AMB-14; T2 codec, AMB-12).  Citations: P:n =
PAPER.md line n, S:n = SPEC.md line n, AMB-k = ambiguity reading k.

Pinned by tests/test_oracle_pins.py (-m "not gpu"); every function below has a
pin there.  tests/test_oracle_mutants.py checks that those pins fail on plausible
mistakes (T3 attended, T2 at full precision, one head per group in the external
update, lossless T2 exit, window/floor/scale/T2-order errors).  No function is
"parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

T0, T1, T2, T3 = 0, 1, 2, 3
EVICT_TOTAL, EVICT_PER_EVENT = 0, 1
# tier policies: the paper's hierarchy and its pure-eviction baselines (§4.1 P:276-280;
# SPEC §baselines)
POLICY_HIERARCHY, POLICY_STREAMING, POLICY_H2O, POLICY_RANDOM = 0, 1, 2, 3
# token scorers (§4 ablation P:707-714): Eq. 1 attention; VATP, attention x ||v||
# (P:712); redundancy, attention - neighbour cosine; combined, attention x ||v|| -
# redundancy.  Readings AMB-30/31 in DESIGN.md.  Windowed attention ("the last
# alpha = 8 observation tokens", max-pooled with kernel 7, App. E) and R-KV's
# Z = lambda I - (1 - lambda) R (App. E).  Readings AMB-32/33 in DESIGN.md.
SCORER_ATTENTION, SCORER_VATP, SCORER_REDUNDANCY, SCORER_COMBINED = 0, 1, 2, 3
SCORER_WINDOW, SCORER_RKV = 4, 5
RKV_ALPHA = 8                      # observation tokens
RKV_POOL = 7                       # max-pool kernel size
RKV_LAMBDA = np.float32(0.07)      # lambda
RKV_ONE_MINUS_LAMBDA = np.float32(0.93)


# ----------------------------------------------------------------- attention
def attention_weights(q, K):
    """alpha_i = softmax_i(q.k_i / sqrt(d)) in fp64 (Eq. 2 context).

    q: [d], K: [n][d] (any real dtype).  n >= 1 else ValueError."""
    q = np.asarray(q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    if K.ndim != 2 or K.shape[0] == 0:
        raise ValueError("empty key set")
    if K.shape[1] != q.shape[0]:
        raise ValueError("dimension mismatch")
    z = (K @ q) / math.sqrt(q.shape[0])
    m = np.max(z)
    e = np.exp(z - m)
    return e / np.sum(e)


def attention_output(q, K, V):
    """Exact attention o = sum_i alpha_i v_i (Eq. 2)."""
    a = attention_weights(q, K)
    return a @ np.asarray(V, dtype=np.float64)


def evicted_attention_output(q, K, V, evicted):
    """o_hat = (1/Z') sum_{i not in E} exp(q.k_i/sqrt d) v_i (Eq. 3).

    The softmax is restricted to the survivors (ascending position order)."""
    n = np.asarray(K).shape[0]
    keep = np.ones(n, dtype=bool)
    keep[list(evicted)] = False
    if not keep.any():
        raise ValueError("empty survivor set")
    return attention_output(q, np.asarray(K)[keep], np.asarray(V)[keep])


def eviction_error_bound(alpha, V, evicted):
    """2 * sum_{i in E} alpha_i ||v_i|| with full-cache alpha (Eq. 4)."""
    V = np.asarray(V, dtype=np.float64)
    return 2.0 * float(sum(alpha[i] * np.linalg.norm(V[i]) for i in evicted))


def eviction_error_bound_triangle(alpha, V, evicted):
    """A bound that always holds (reading R-EQ4): with eps = sum_{i in E} alpha_i,
    o_hat - o = eps * o_hat - sum_{i in E} alpha_i v_i (from Eq. 2/3), so by the triangle
    inequality ||o_hat - o|| <= eps ||o_hat|| + sum_E alpha_i ||v_i|| <= 2 eps max_i ||v_i||.
    Eq. 4 as printed drops the eps ||o_hat|| term's dependence on the surviving values and
    fails when survivors have larger norms than the evicted rows (tests pin a counterexample)."""
    V = np.asarray(V, dtype=np.float64)
    ev = list(evicted)
    eps = float(sum(alpha[i] for i in ev))
    keep = np.ones(len(V), dtype=bool)
    keep[ev] = False
    o_hat = (alpha[keep] @ V[keep]) / (1.0 - eps)
    return eps * float(np.linalg.norm(o_hat)) + float(sum(alpha[i] * np.linalg.norm(V[i]) for i in ev))


def lse_merge(parts):
    """Merge split-K partials [(m_k, l_k, o_k)] of one softmax, where
    m_k = max logit, l_k = sum exp(z - m_k), o_k = sum exp(z - m_k) v (unnormalised).
    Returns the normalised output sum_k exp(m_k - M) o_k / sum_k exp(m_k - M) l_k.
    (Associativity of the softmax sum, used by the sequence split.)"""
    M = max(p[0] for p in parts)
    L = sum(math.exp(p[0] - M) * p[1] for p in parts)
    O = sum(math.exp(p[0] - M) * np.asarray(p[2], dtype=np.float64) for p in parts)
    return O / L


def partial_softmax(q, K, V):
    """(m, l, o_unnormalised) over a key subset, for lse_merge."""
    q = np.asarray(q, dtype=np.float64)
    z = (np.asarray(K, dtype=np.float64) @ q) / math.sqrt(q.shape[0])
    m = float(np.max(z))
    e = np.exp(z - m)
    return m, float(np.sum(e)), e @ np.asarray(V, dtype=np.float64)


# ----------------------------------------------------------------- T2 codec
def quantize_int8(x):
    """Per-row symmetric int8 (AMB-12; "e.g., 8-bit quantization").

    x: fp32 row (the bf16 value).  scale = fp32(absmax / 127) (IEEE RN division);
    code = clamp(rint_half_even(fp32(x / scale)), -127, 127); all-zero row ->
    scale 1, codes 0."""
    x = np.asarray(x, dtype=np.float32)
    amax = np.float32(np.max(np.abs(x))) if x.size else np.float32(0)
    if amax == 0:
        return np.zeros(x.shape, dtype=np.int8), np.float32(1.0)
    scale = np.float32(amax / np.float32(127.0))
    qv = (x / scale).astype(np.float32)
    codes = np.clip(np.rint(qv), -127, 127).astype(np.int8)
    return codes, scale


def dequantize_int8(codes, scale):
    """fp32(code * scale) (AMB-12)."""
    return (np.asarray(codes, dtype=np.float32) * np.float32(scale)).astype(np.float32)


def f32_to_bf16_value(x):
    """fp32 -> nearest-even bf16, returned as fp32 values (lossy store of a T2 row
    that leaves T2, AMB-12)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint32) << np.uint32(16)
    return r.view(np.float32)


# ----------------------------------------------------------------- tier logic
def protected_mask(n, prompt_len, sink_size, window_size):
    """Protected set P = [0,P) u [P, min(P+k_s, n)) u [max(0, n-k_w), n)  (0-based;
    §3.2, Alg. 1 line P:190, AMB-6).  Boolean mask of length n."""
    m = np.zeros(n, dtype=bool)
    m[:min(prompt_len, n)] = True
    m[prompt_len:min(prompt_len + sink_size, n)] = True
    m[max(0, n - window_size):n] = True
    return m


def total_score_fp32(S_part_b):
    """S_i = fp32 sum over kv heads g = 0..H_kv-1 in ascending order (AMB-1, AMB-14)."""
    S = np.array(S_part_b[0], dtype=np.float32, copy=True)
    for g in range(1, S_part_b.shape[0]):
        S = (S + S_part_b[g]).astype(np.float32)
    return S


def tier_counts(n_protected, n_live, n_t3, hbm_bp, evict_bp, t2_bp, mode=EVICT_TOTAL):
    """Floor arithmetic of Alg. 1 in integer basis points (AMB-8/9/11).

    Returns (n_new_evict, n_hbm, n_t2, n_t1)."""
    if mode == EVICT_TOTAL:
        n_tot = (evict_bp * (n_live + n_t3)) // 10000
        n_new = max(0, n_tot - n_t3)
    else:
        n_new = (evict_bp * n_live) // 10000
    surv = n_live - n_new
    n_hbm = (hbm_bp * surv) // 10000
    n_t2 = (t2_bp * (surv - n_hbm)) // 10000
    return n_new, n_hbm, n_t2, surv - n_hbm - n_t2


_M64 = (1 << 64) - 1


def splitmix64(x):
    """SplitMix64 finaliser on a Python int (mod 2^64): the counter-based generator the
    RANDOM policy draws its keys from (each side of the parity test implements it)."""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def random_key32(seed, req, pos):
    """RANDOM policy rank key of (request, position): high 32 bits of
    splitmix64(splitmix64(seed << 32 | req) ^ pos)."""
    return splitmix64(splitmix64(((seed & 0xFFFFFFFF) << 32) | (req & 0xFFFFFFFF)) ^ pos) >> 32


def policy_counts(policy, budget, n_protected, n_live, n_t3, cfg):
    """(n_new_evict, n_hbm, n_t2, n_t1) of a manage event under a tier policy.

    HIERARCHY: Alg. 1 (tier_counts).  STREAMING (StreamingLLM): keep only the
    protected sinks + window, every live non-protected token is evicted.  H2O / RANDOM
    (P:279-280): keep the protected set plus max(0, budget - |P|) live tokens,
    all in HBM (pure eviction: no T1/T2)."""
    if policy == POLICY_HIERARCHY:
        return tier_counts(n_protected, n_live, n_t3, cfg.hbm_bp, cfg.evict_bp, cfg.t2_bp, cfg.evict_mode)
    if policy == POLICY_STREAMING:
        return n_live, 0, 0, 0
    keep = min(n_live, max(0, budget - n_protected))
    return n_live - keep, keep, 0, 0


def ordered_bits(f):
    """Order-preserving map fp32 -> uint32 (sign-magnitude to unsigned): for non-negative
    values it orders exactly like the raw bits (AMB-7); negatives sort below every positive."""
    u = np.asarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return np.where(u & 0x80000000, 0xFFFFFFFF - u, u | 0x80000000).astype(np.uint64)


def key_redundancy(K):
    """Neighbour-cosine redundancy (reading AMB-30): per layer l and kv head g,
    c_i = cos(k_i, k_{i-1}) of the ORIGINAL key rows (fp64, rounded to fp32), c_0 = 0, 0 when
    either row is zero; R_part[b][g][i] = fp32 sum over layers in ascending l.
    K: fp32 [L][B][H_kv][N][d].  Returns R_part fp32 [B][H_kv][N]."""
    K = np.asarray(K, dtype=np.float64)
    L, B, Hkv, N, d = K.shape
    c = np.zeros((L, B, Hkv, N), dtype=np.float32)
    if N > 1:
        a, p = K[..., 1:, :], K[..., :-1, :]
        dot = np.sum(a * p, axis=-1)
        na, nb = np.sum(a * a, axis=-1), np.sum(p * p, axis=-1)
        ok = (na > 0) & (nb > 0)
        c[..., 1:] = np.where(ok, dot / np.sqrt(np.where(ok, na * nb, 1.0)), 0.0).astype(np.float32)
    R = np.zeros((B, Hkv, N), dtype=np.float32)
    for l in range(L):
        R = (R + c[l]).astype(np.float32)
    return R


def classify_scores(S, R_part_b, live, cfg):
    """The fp32 value ranked by classify (AMB-31).  Attention / VATP: S itself.  Redundancy /
    combined ("attn - redundancy"): I_i - rho_i with I_i = fp32(S_i / S_max)
    (S_max = max of S over the live set, I = 0 if S_max = 0) and rho_i = fp32(fp32(sum_g
    R_part[g][i]) / (L * H_kv)), the mean neighbour cosine over layers and kv heads."""
    scorer = getattr(cfg, "scorer", SCORER_ATTENTION)
    if scorer < SCORER_REDUNDANCY or scorer == SCORER_WINDOW:
        return S
    n = S.shape[0]
    smax = np.float32(S[live].max()) if live.any() else np.float32(0)
    I = (S / smax).astype(np.float32) if smax > 0 else np.zeros(n, dtype=np.float32)
    rsum = np.zeros(n, dtype=np.float32)
    for g in range(R_part_b.shape[0]):
        rsum = (rsum + R_part_b[g, :n]).astype(np.float32)
    rho = (rsum / np.float32(cfg.L * cfg.Hkv)).astype(np.float32)
    if scorer == SCORER_RKV:   # Z = lambda I - (1 - lambda) R, each product rounded to fp32 (AMB-33)
        return ((RKV_LAMBDA * I).astype(np.float32) - (RKV_ONE_MINUS_LAMBDA * rho).astype(np.float32)).astype(np.float32)
    return (I - rho).astype(np.float32)


def observation_window(cfg):
    """Steps in the windowed scorers' observation window: alpha = 8, at most the
    manage interval (AMB-32: a window never reaches back past the previous event)."""
    return min(RKV_ALPHA, cfg.manage_interval)


def snapshot_due(cfg, t):
    """AMB-32: the windowed scorers snapshot S_part at the START of step t when t + w - 1 is a
    multiple of Delta (w = observation_window), so that at the event of step t_e = t + w - 1 the
    windowed score S(after t_e) - S(snapshot) sums the probabilities of steps t_e-w+1 .. t_e."""
    w = observation_window(cfg)
    return (t + w - 1) % cfg.manage_interval == 0


def max_pool_visible(W, vis, k=RKV_POOL):
    """R-KV's max-pool (kernel k, stride 1, (k-1)/2 padding that never wins) over the cache in
    its stored order: the non-T3 positions ``vis`` ascending (AMB-32).  Returns an array like W
    whose entries at ``vis`` are the pooled values (other entries 0)."""
    out = np.zeros_like(W)
    h = k // 2
    m = len(vis)
    for j in range(m):
        out[vis[j]] = max(W[vis[x]] for x in range(max(0, j - h), min(m, j + h + 1)))
    return out


def windowed_scores(S_part_b, S_snap_b, tier_b, n):
    """Windowed attention importance of the windowed / R-KV scorers (AMB-32):
    W_i = fp32(S_i(now)) - fp32(S_i(snapshot)), each S the fp32 sum over kv heads in ascending
    order, then max-pooled over the non-T3 positions in position order."""
    W = (total_score_fp32(np.asarray(S_part_b)[:, :n]) - total_score_fp32(np.asarray(S_snap_b)[:, :n])).astype(np.float32)
    vis = np.nonzero(np.asarray(tier_b[:n]) != T3)[0]
    return max_pool_visible(W, vis)


def classify_request(S_part_b, tier_b, n, cfg, req=0, R_part_b=None, S_snap_b=None):
    """One manage event for one request (Alg. 1 lines P:189-197; §3.3).

    S_part_b: [H_kv][>=n] fp32, tier_b: [>=n] u8 current tiers (T3 sticky, AMB-16/24),
    R_part_b: [H_kv][>=n] fp32 redundancy partials (redundancy / combined / R-KV scorers only).
    S_snap_b: [H_kv][>=n] fp32 snapshot of S_part (windowed / R-KV scorers only, AMB-32).
    Returns the new tier array [n] (uint8)."""
    if getattr(cfg, "scorer", SCORER_ATTENTION) in (SCORER_WINDOW, SCORER_RKV):
        S = windowed_scores(S_part_b, S_snap_b, tier_b, n)
    else:
        S = total_score_fp32(np.asarray(S_part_b)[:, :n])
    prot = protected_mask(n, cfg.prompt_len, cfg.sink_size, cfg.window_size)
    old = np.asarray(tier_b[:n])
    t3 = old == T3
    live = ~prot & ~t3
    pos_live = np.nonzero(live)[0]
    # order U_live by the unique key (bits(score_i), i) ascending (AMB-7); RANDOM: (hash, i)
    if cfg.policy == POLICY_RANDOM:
        primary = np.array([random_key32(cfg.policy_seed, req, int(p)) for p in pos_live], dtype=np.uint64)
    else:
        primary = ordered_bits(classify_scores(S, R_part_b, live, cfg)[pos_live])
    order = np.lexsort((pos_live, primary))
    sorted_pos = pos_live[order]
    n_new, n_hbm, n_t2, n_t1 = policy_counts(cfg.policy, cfg.budget, int(prot.sum()), len(pos_live),
                                             int(t3.sum()), cfg)
    new = np.full(n, T0, dtype=np.uint8)          # protected -> T0
    new[t3] = T3
    new[sorted_pos[:n_new]] = T3
    surv = sorted_pos[n_new:]
    new[surv[:n_t2]] = T2
    new[surv[n_t2:len(surv) - n_hbm]] = T1
    new[surv[len(surv) - n_hbm:]] = T0
    return new


# ----------------------------------------------------------------- simulation
@dataclass
class OracleConfig:
    B: int
    L: int
    Hq: int
    Hkv: int
    d: int
    prompt_len: int
    sink_size: int = 4
    window_size: int = 128
    manage_interval: int = 64
    hbm_bp: int = 5000
    evict_bp: int = 500
    t2_bp: int = 0
    evict_mode: int = EVICT_TOTAL
    policy: int = POLICY_HIERARCHY
    budget: int = 0
    policy_seed: int = 0
    req_ids: list = None       # the library's request index of each oracle request (RANDOM keys)
    scorer: int = SCORER_ATTENTION

    @property
    def G(self):
        return self.Hq // self.Hkv


@dataclass
class OracleState:
    """Per-request tier state keyed by position (SURVEY §8c "Stores")."""
    cfg: OracleConfig
    n: int
    tier: np.ndarray           # [B][Nmax] u8
    S_part: np.ndarray         # [B][Hkv][Nmax] fp32
    rowK: np.ndarray           # [L][B][Hkv][Nmax][d] fp32 (bf16-valued) for T0/T1
    rowV: np.ndarray
    codeK: np.ndarray          # [L][B][Hkv][Nmax][d] int8 for T2
    codeV: np.ndarray
    scaleK: np.ndarray         # [L][B][Hkv][Nmax] fp32
    scaleV: np.ndarray
    t: int = 0
    events: list = field(default_factory=list)
    vnorm: np.ndarray = None   # VATP / combined: [L][B][Hkv][Nmax] fp32 ||v|| of every original V row
    R_part: np.ndarray = None  # redundancy / combined / R-KV: [B][Hkv][Nmax] fp32 (key_redundancy)
    S_snap: np.ndarray = None  # windowed / R-KV: [B][Hkv][Nmax] fp32 S_part at the window start (AMB-32)


def init_state(cfg, Kbits, Vbits, n0):
    """Alg. 1 lines P:173-174: prefix of n0 tokens, all T0, scores 0.

    Kbits/Vbits: bf16 bit patterns [L][B][Hkv][Nmax][d] for every position the run
    will ever generate (the never-migrated originals)."""
    from paper_2605_09490_b200.synth.synth import bf16_bits_to_f32   # input decoding only
    L, B, Hkv, Nmax, d = Kbits.shape
    vnorm = R_part = S_snap = None
    scorer = getattr(cfg, "scorer", SCORER_ATTENTION)
    if scorer in (SCORER_VATP, SCORER_COMBINED):
        vnorm = value_norms(bf16_bits_to_f32(Vbits))
    if scorer in (SCORER_REDUNDANCY, SCORER_COMBINED, SCORER_RKV):
        R_part = key_redundancy(bf16_bits_to_f32(Kbits))
    if scorer in (SCORER_WINDOW, SCORER_RKV):
        S_snap = np.zeros((B, Hkv, Nmax), dtype=np.float32)
    return OracleState(
        cfg=cfg, n=n0, vnorm=vnorm, R_part=R_part, S_snap=S_snap,
        tier=np.full((B, Nmax), T0, dtype=np.uint8),
        S_part=np.zeros((B, Hkv, Nmax), dtype=np.float32),
        rowK=bf16_bits_to_f32(Kbits).copy(), rowV=bf16_bits_to_f32(Vbits).copy(),
        codeK=np.zeros((L, B, Hkv, Nmax, d), dtype=np.int8),
        codeV=np.zeros((L, B, Hkv, Nmax, d), dtype=np.int8),
        scaleK=np.ones((L, B, Hkv, Nmax), dtype=np.float32),
        scaleV=np.ones((L, B, Hkv, Nmax), dtype=np.float32),
    )


def value_norms(V):
    """VATP weights: fp32 L2 norm of each V row (last axis), summed in float64."""
    return np.sqrt(np.sum(np.asarray(V, dtype=np.float64) ** 2, axis=-1)).astype(np.float32)


def score_increment(psum, st, l, b, g, vis):
    """fp32 increment of S_part for positions vis: fp32(sum_h p) (Eq. 1, AMB-14), times the
    token's V-row norm under VATP: fp32(fp32(sum_h p) * ||v||)."""
    inc = psum.astype(np.float32)
    if st.vnorm is not None:
        inc = (inc * st.vnorm[l, b, g, vis]).astype(np.float32)
    return inc


def effective_rows(st, l, b, g, vis):
    """K/V values attention uses for positions ``vis``:
    T0/T1 -> stored bf16 row; T2 -> fp32 dequant (AMB-12)."""
    K = st.rowK[l, b, g, vis].astype(np.float64)
    V = st.rowV[l, b, g, vis].astype(np.float64)
    t2 = st.tier[b, vis] == T2
    if t2.any():
        p2 = vis[t2]
        K[t2] = (st.codeK[l, b, g, p2].astype(np.float32) * st.scaleK[l, b, g, p2][:, None]).astype(np.float32)
        V[t2] = (st.codeV[l, b, g, p2].astype(np.float32) * st.scaleV[l, b, g, p2][:, None]).astype(np.float32)
    return K, V


def decode_layer(st, l, qbits_l):
    """Attention + score update of one layer at the current step.

    For every (b, h), g = h // G (AMB-4): masked softmax over the visible set
    V = {i < n : tier != T3} in ascending position order (Eq. 3, Prop. 1
    P:416-427), then S_part[b][g][i] = fp32(S_part + fp32(sum_{h in g} p_h,i))
    (Eq. 1, Alg. 1; AMB-1, AMB-14, AMB-15).
    qbits_l: bf16 bits [B][Hq][d].  Returns o [B][Hq][d] fp64."""
    from paper_2605_09490_b200.synth.synth import bf16_bits_to_f32
    cfg = st.cfg
    B = qbits_l.shape[0]
    q = bf16_bits_to_f32(qbits_l).astype(np.float64)
    o = np.zeros((B, cfg.Hq, cfg.d), dtype=np.float64)
    inv_sqrt_d = 1.0 / math.sqrt(cfg.d)
    for b in range(B):
        vis = np.nonzero(st.tier[b, :st.n] != T3)[0]
        if vis.size == 0:
            raise ValueError("empty visible set")
        for g in range(cfg.Hkv):
            K, V = effective_rows(st, l, b, g, vis)
            psum = np.zeros(vis.size, dtype=np.float64)
            for h in range(g * cfg.G, (g + 1) * cfg.G):
                z = (K @ q[b, h]) * inv_sqrt_d
                e = np.exp(z - np.max(z))
                p = e / np.sum(e)
                o[b, h] = p @ V
                psum += p
            if not np.all(np.isfinite(psum)):
                raise FloatingPointError("non-finite probability (E_NUMERIC)")
            st.S_part[b, g, vis] = (st.S_part[b, g, vis] + score_increment(psum, st, l, b, g, vis)).astype(np.float32)
    return o


def visible_positions(st, b):
    """Ascending positions of request b that attention sees: tier != T3 (Eq. 3)."""
    return np.nonzero(st.tier[b, :st.n] != T3)[0]


def score_update_external(S_part_b, vis, probs_b, G):
    """Eq. 1 with externally supplied probabilities (Alg. 1, AMB-14):
    S_part[g][vis[j]] = fp32(S_part[g][vis[j]] + fp32(sum_{h in g} probs[h][j])).
    S_part_b: [H_kv][N] fp32 (updated in place); probs_b: [H_q][len(vis)]."""
    Hkv = S_part_b.shape[0]
    for g in range(Hkv):
        inc = np.zeros(len(vis), dtype=np.float64)
        for h in range(g * G, (g + 1) * G):
            inc += np.asarray(probs_b[h], dtype=np.float64)
        S_part_b[g, vis] = (S_part_b[g, vis] + inc.astype(np.float32)).astype(np.float32)
    return S_part_b


def manage_event(st):
    """Classify every request then migrate its rows (Alg. 1, AMB-11/12).

    Transitions: ->T3 drop; T0/T1->T2 quantise the stored bf16 row; T2->T0/T1
    keep bf16(dequant) (lossy); T0<->T1 unchanged bytes."""
    cfg = st.cfg
    B = st.tier.shape[0]
    for b in range(B):
        old = st.tier[b, :st.n].copy()
        new = classify_request(st.S_part[b], old, st.n, cfg, req=cfg.req_ids[b] if cfg.req_ids else b,
                               R_part_b=None if st.R_part is None else st.R_part[b],
                               S_snap_b=None if st.S_snap is None else st.S_snap[b])
        to_t2 = (new == T2) & (old != T2)
        from_t2 = (old == T2) & ((new == T0) | (new == T1))
        for p in np.nonzero(to_t2)[0]:
            for l in range(cfg.L):
                for g in range(cfg.Hkv):
                    st.codeK[l, b, g, p], st.scaleK[l, b, g, p] = quantize_int8(st.rowK[l, b, g, p])
                    st.codeV[l, b, g, p], st.scaleV[l, b, g, p] = quantize_int8(st.rowV[l, b, g, p])
        for p in np.nonzero(from_t2)[0]:
            st.rowK[:, b, :, p] = f32_to_bf16_value(dequantize_int8(st.codeK[:, b, :, p], st.scaleK[:, b, :, p][..., None]))
            st.rowV[:, b, :, p] = f32_to_bf16_value(dequantize_int8(st.codeV[:, b, :, p], st.scaleV[:, b, :, p][..., None]))
        st.tier[b, :st.n] = new
    st.events.append(st.t)


def decode_step(st, qbits_t, manage=True):
    """One decode step t of Alg. 1: the new token (position n, already
    present in rowK/rowV from the generator) joins T0, attention + scores over all
    layers, then a manage event if t mod Delta == 0 (t = 0 included, AMB-10).

    Windowed / R-KV scorers: S_part is snapshot first when the observation window of the next
    event starts at this step (snapshot_due, AMB-32).

    qbits_t: [L][B][Hq][d] bf16 bits.  Returns o [L][B][Hq][d] fp64."""
    if st.S_snap is not None and snapshot_due(st.cfg, st.t):
        st.S_snap = st.S_part.copy()
    st.tier[:, st.n] = T0
    st.n += 1
    o = np.stack([decode_layer(st, l, qbits_t[l]) for l in range(st.cfg.L)])
    if manage and st.t % st.cfg.manage_interval == 0:
        manage_event(st)
    st.t += 1
    return o


def census(st, b):
    """Tier counts [T0, T1, T2, T3] of request b over positions [0, n)."""
    return np.bincount(st.tier[b, :st.n], minlength=4)[:4]


def export_index(st, b, tier):
    """Ascending positions of request b in ``tier`` (canonical index list)."""
    return np.nonzero(st.tier[b, :st.n] == tier)[0].astype(np.int32)
