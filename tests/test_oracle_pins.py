"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Every oracle function is pinned by at least one of: a value the paper/spec prints
(tests/golden/*), a closed form, an invariant, a special case that reduces to a
library routine (torch SDPA in float64), or brute force on tiny inputs written
as plain Python loops (an independent implementation, not a re-call).
"""
import json
import math
import os
import random

import numpy as np
import pytest
import torch

from oracle import kvtier_oracle as O
from paper_2605_09490_b200.synth import synth as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# ------------------------------------------------------------ Eq. 2 / Eq. 3
def test_single_key_weight_is_one():
    assert O.attention_weights([0.3, -1.0], [[5.0, 2.0]]).tolist() == [1.0]


def test_identical_keys_uniform():
    w = O.attention_weights([1.0, 2.0, 3.0], [[0.5, 0.1, 0.2]] * 4)
    assert np.allclose(w, 0.25, rtol=0, atol=1e-15)


def test_d2_hand_softmax():
    # q=(1,0), keys (1,0),(0,1): logits 1/sqrt2 and 0; weight_0 = logistic(1/sqrt2)
    w = O.attention_weights([1.0, 0.0], [[1.0, 0.0], [0.0, 1.0]])
    x = 1.0 / math.sqrt(2.0)
    w0 = 0.5 * (1.0 + math.tanh(x / 2.0))                  # logistic via tanh (independent form)
    assert abs(w[0] - w0) < 1e-15 and abs(w[1] - (1.0 - w0)) < 1e-15
    assert abs(w0 - 0.6697615493266569) < 1e-12             # hand-evaluated value


def test_one_pair_and_identical_values():
    v = [0.25, -1.5, 3.0]
    assert O.attention_output([1.0, 1.0, 1.0], [[0.1, 0.2, 0.3]], [v]).tolist() == v
    rng = np.random.default_rng(0)
    out = O.attention_output(rng.normal(size=3), rng.normal(size=(7, 3)), [v] * 7)
    assert np.allclose(out, v, rtol=0, atol=1e-14)


def _brute_attention(q, K, V, skip=()):
    """Plain double loop (independent implementation)."""
    d = len(q)
    idx = [i for i in range(len(K)) if i not in skip]
    logits = {}
    for i in idx:
        s = 0.0
        for k in range(d):
            s += q[k] * K[i][k]
        logits[i] = s / math.sqrt(d)
    m = max(logits.values())
    Z = sum(math.exp(logits[i] - m) for i in idx)
    out = [0.0] * len(V[0])
    for i in idx:
        a = math.exp(logits[i] - m) / Z
        for k in range(len(out)):
            out[k] += a * V[i][k]
    return out


def test_attention_bruteforce_5_tokens():
    rng = random.Random(5)
    q = [rng.uniform(-2, 2) for _ in range(4)]
    K = [[rng.uniform(-2, 2) for _ in range(4)] for _ in range(5)]
    V = [[rng.uniform(-2, 2) for _ in range(3)] for _ in range(5)]
    assert np.allclose(O.attention_output(q, K, V), _brute_attention(q, K, V), rtol=0, atol=1e-13)


def test_eq3_empty_eviction_is_bitwise_eq2():
    rng = np.random.default_rng(1)
    q, K, V = rng.normal(size=8), rng.normal(size=(9, 8)), rng.normal(size=(9, 8))
    assert np.array_equal(O.evicted_attention_output(q, K, V, []), O.attention_output(q, K, V))


def test_eq3_single_survivor_and_bruteforce():
    rng = np.random.default_rng(2)
    q, K, V = rng.normal(size=4), rng.normal(size=(6, 4)), rng.normal(size=(6, 3))
    out = O.evicted_attention_output(q, K, V, [0, 1, 2, 4, 5])
    assert np.allclose(out, V[3], rtol=0, atol=1e-15)
    out = O.evicted_attention_output(q, K, V, [1, 4])   # "evict {2,5}" 1-based
    ref = _brute_attention(q.tolist(), K.tolist(), V.tolist(), skip=(1, 4))
    assert np.allclose(out, ref, rtol=0, atol=1e-13)
    with pytest.raises(ValueError):
        O.evicted_attention_output(q, K, V, range(6))


def test_eq4_bound_sound_equal_norms_1000_instances():
    """Eq. 4 as printed holds when every value row has the same norm (then
    ||o_hat|| <= ||v||), and the always-valid triangle bound holds everywhere."""
    rng = np.random.default_rng(3)
    worst = 0.0
    for _ in range(1000):
        n, d = rng.integers(2, 64), rng.integers(1, 16)
        q, K = rng.normal(size=d) * 2, rng.normal(size=(n, d))
        V = rng.normal(size=(n, d))
        V /= np.linalg.norm(V, axis=1, keepdims=True)
        ev = [i for i in range(n) if rng.random() < 0.3][: n - 1]
        a = O.attention_weights(q, K)
        err = np.linalg.norm(O.evicted_attention_output(q, K, V, ev) - a @ V)
        bound = O.eviction_error_bound(a, V, ev)
        assert err <= bound + 1e-12
        assert err <= O.eviction_error_bound_triangle(a, V, ev) + 1e-12
        worst = max(worst, err / bound if bound > 0 else 0)
    assert worst > 0.05          # the bound is exercised, not vacuous


def test_eq4_counterexample_and_triangle_bound():               # reading R-EQ4
    """Eq. 4 is not a bound for arbitrary values: golden counterexample (3 tokens)."""
    g = _golden("eq4_counterexample.json")
    q, K, V, ev = (np.array(g[k], dtype=np.float64) for k in ("q", "K", "V", "evicted"))
    ev = ev.astype(int).tolist()
    a = O.attention_weights(q, K)
    err = np.linalg.norm(O.evicted_attention_output(q, K, V, ev) - a @ V)
    assert err > O.eviction_error_bound(a, V, ev) * 1.5          # Eq. 4 violated
    assert err <= O.eviction_error_bound_triangle(a, V, ev) + 1e-12
    rng = np.random.default_rng(33)
    for _ in range(1000):                                        # triangle bound: always
        n, d = rng.integers(2, 64), rng.integers(1, 16)
        q, K, V = rng.normal(size=d) * 2, rng.normal(size=(n, d)), rng.normal(size=(n, d)) * rng.uniform(0.1, 3, size=(n, 1))
        ev = [i for i in range(n) if rng.random() < 0.3][: n - 1]
        a = O.attention_weights(q, K)
        err = np.linalg.norm(O.evicted_attention_output(q, K, V, ev) - a @ V)
        assert err <= O.eviction_error_bound_triangle(a, V, ev) + 1e-12


def test_eq4_single_eviction_instantiation():
    rng = np.random.default_rng(4)
    q, K, V = rng.normal(size=5), rng.normal(size=(7, 5)), rng.normal(size=(7, 5))
    a = O.attention_weights(q, K)
    assert O.eviction_error_bound(a, V, [3]) == pytest.approx(2 * a[3] * np.linalg.norm(V[3]), rel=1e-15)
    assert O.eviction_error_bound(a, V, []) == 0.0


def test_masked_attention_matches_torch_sdpa_float64():       # library routine (SDPA)
    rng = np.random.default_rng(5)
    q, K, V = rng.normal(size=(1, 64)), rng.normal(size=(40, 64)), rng.normal(size=(40, 64))
    ev = [2, 7, 8, 30]
    mask = torch.ones(1, 40, dtype=torch.bool)
    mask[0, ev] = False
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(q)[None], torch.from_numpy(K)[None], torch.from_numpy(V)[None],
        attn_mask=mask[None])[0, 0].numpy()
    assert np.allclose(O.evicted_attention_output(q[0], K, V, ev), ref, rtol=0, atol=1e-13)


# ------------------------------------------------------------ LSE merge
@pytest.mark.parametrize("k", [1, 2, 3, 5, 8])
def test_lse_merge_equals_unsplit(k):
    rng = np.random.default_rng(10 + k)
    q, K, V = rng.normal(size=16) * 3, rng.normal(size=(97, 16)), rng.normal(size=(97, 16))
    cuts = np.linspace(0, 97, k + 1).astype(int)
    parts = [O.partial_softmax(q, K[a:b], V[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    assert np.allclose(O.lse_merge(parts), O.attention_output(q, K, V), rtol=0, atol=1e-13)


# ------------------------------------------------------------ T2 codec (AMB-12)
def test_int8_zero_row_exact():
    c, s = O.quantize_int8(np.zeros(16, np.float32))
    assert s == np.float32(1.0) and not c.any()
    assert not O.dequantize_int8(c, s).any()


def test_int8_absmax_maps_to_127_and_exact_grid():
    x = np.array([127.0, -3.0, 64.0, -127.0, 0.0], np.float32)
    c, s = O.quantize_int8(x)
    assert s == np.float32(1.0)
    assert c.tolist() == [127, -3, 64, -127, 0]
    assert np.array_equal(O.dequantize_int8(c, s), x)


def test_int8_round_trip_bound_half_scale():                 # S:94 (tighter: scale/2)
    rng = np.random.default_rng(6)
    for _ in range(200):
        x = S.bf16_bits_to_f32(S.f32_to_bf16_bits(rng.normal(size=128).astype(np.float32) * rng.uniform(0.01, 10)))
        c, s = O.quantize_int8(x)
        assert np.max(np.abs(c.astype(int))) == 127
        err = np.abs(O.dequantize_int8(c, s).astype(np.float64) - x.astype(np.float64))
        assert np.all(err <= float(s) * (0.5 + 2e-5))        # + fp32 rounding of x/scale and code*scale


def test_bf16_rounding_matches_torch():                      # library routine
    rng = np.random.default_rng(7)
    x = (rng.normal(size=100000) * np.exp(rng.normal(size=100000) * 3)).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(O.f32_to_bf16_value(x), ref)
    assert np.array_equal(S.bf16_bits_to_f32(S.f32_to_bf16_bits(x)), ref)


# ------------------------------------------------------------ protected set / counts
def test_protected_set_spec_example():                       # S:261 (AMB-6)
    g = _golden("protected_set.json")
    for case in g["cases"]:
        m = O.protected_mask(case["n"], case["P"], case["k_s"], case["k_w"])
        assert int(m.sum()) == case["size"], case
        if "ranges" in case:
            want = np.zeros(case["n"], bool)
            for a, b in case["ranges"]:
                want[a:b] = True
            assert np.array_equal(m, want)


def test_tier_counts_golden():                                # S:270, SURVEY §8d table, AMB-8
    g = _golden("tier_counts.json")
    for c in g["cases"]:
        got = O.tier_counts(c["n_protected"], c["n_live"], c["n_t3"], c["hbm_bp"],
                            c["evict_bp"], c.get("t2_bp", 0), c.get("mode", 0))
        assert list(got) == c["expect"], c


def test_floor_is_exact_integer_not_float():                  # AMB-8: 0.7*90 = 62.999.. in double
    assert math.floor(0.7 * 90) == 62
    assert O.tier_counts(0, 90, 0, 7000, 0, 0)[1] == 63


def _brute_classify(S_list, tier_old, n, P, ks, kw, hbm_bp, evict_bp, t2_bp, mode):
    """Independent loop implementation of Alg. 1 lines P:189-197 + AMB rules."""
    prot = set(range(min(P, n))) | set(range(P, min(P + ks, n))) | set(range(max(0, n - kw), n))
    t3_old = [i for i in range(n) if tier_old[i] == 3]
    live = [i for i in range(n) if i not in prot and tier_old[i] != 3]
    live.sort(key=lambda i: (S_list[i], i))     # float order == bit order for S >= 0
    if mode == 0:
        n_new = max(0, (evict_bp * (len(live) + len(t3_old))) // 10000 - len(t3_old))
    else:
        n_new = (evict_bp * len(live)) // 10000
    surv = live[n_new:]
    n_hbm = (hbm_bp * len(surv)) // 10000
    n_t2 = (t2_bp * (len(surv) - n_hbm)) // 10000
    out = [0] * n
    for i in t3_old + live[:n_new]:
        out[i] = 3
    for j, i in enumerate(surv):
        if j < n_t2:
            out[i] = 2
        elif j < len(surv) - n_hbm:
            out[i] = 1
        else:
            out[i] = 0
    return out


@pytest.mark.parametrize("kind", ["ties", "cont"])
@pytest.mark.parametrize("mode", [0, 1])
def test_classify_matches_bruteforce(kind, mode):
    cfg = O.OracleConfig(B=3, L=1, Hq=4, Hkv=2, d=8, prompt_len=16, hbm_bp=5000,
                         evict_bp=1000, t2_bp=5000, evict_mode=mode)
    Sp = S.gen_scores(11, 3, 2, 600, kind)
    for b in range(3):
        tier = np.zeros(600, np.uint8)
        for n in (150, 420, 600):                       # three successive events
            new = O.classify_request(Sp[b], tier, n, cfg)
            S_tot = [float(np.float32(Sp[b, 0, i]) + np.float32(Sp[b, 1, i])) for i in range(n)]
            ref = _brute_classify(S_tot, tier[:n].tolist(), n, 16, 4, 128, 5000, 1000, 5000, mode)
            assert new.tolist() == ref
            # permanence: old T3 stays T3
            assert np.all(new[tier[:n] == 3] == 3)
            tier[:n] = new
            Sp[b] += np.float32(0.5)     # scores evolve between events


def test_classify_invariants_and_budget():
    cfg = O.OracleConfig(B=1, L=1, Hq=2, Hkv=1, d=8, prompt_len=64, hbm_bp=3000, evict_bp=300)
    Sp = S.gen_scores(12, 1, 1, 2000, "cont")
    new = O.classify_request(Sp[0], np.zeros(2000, np.uint8), 2000, cfg)
    prot = O.protected_mask(2000, 64, 4, 128)
    assert np.all(new[prot] == 0)
    cnt = np.bincount(new, minlength=4)
    # SURVEY §8d 7B r=3% beta=30%: |P|=196 |U|=1804 n_evict=54 n_hbm=525 T1=1225
    assert cnt.tolist() == [196 + 525, 1225, 0, 54]
    # evicted are the lowest-scored non-protected tokens
    S_tot = Sp[0, 0]
    assert S_tot[new == 3].max() <= S_tot[(new != 3) & ~prot].min()
    assert S_tot[(new == 0) & ~prot].min() >= S_tot[new == 1].max()


def test_r0_beta100_all_t0():
    cfg = O.OracleConfig(B=1, L=1, Hq=2, Hkv=1, d=8, prompt_len=8, hbm_bp=10000, evict_bp=0)
    new = O.classify_request(S.gen_scores(3, 1, 1, 500)[0], np.zeros(500, np.uint8), 500, cfg)
    assert np.all(new == 0)


# ------------------------------------------------------------ full decode loop
def _tiny_run(hbm_bp=5000, evict_bp=500, t2_bp=0, interval=64, steps=32, mode=0, L=1):
    w = S.WORKLOADS["tiny"]
    n0 = w["N"] - 1
    K = S.gen_kv(w["seed"], "k", L, w["B"], w["Hkv"], w["d"], 0, n0 + steps, w["P"], 4)
    V = S.gen_kv(w["seed"], "v", L, w["B"], w["Hkv"], w["d"], 0, n0 + steps, w["P"], 4)
    Q = S.gen_q(w["seed"], 0, steps, L, w["B"], w["Hq"], w["Hkv"], w["d"])
    cfg = O.OracleConfig(B=w["B"], L=L, Hq=w["Hq"], Hkv=w["Hkv"], d=w["d"], prompt_len=w["P"],
                         manage_interval=interval, hbm_bp=hbm_bp, evict_bp=evict_bp,
                         t2_bp=t2_bp, evict_mode=mode)
    st = O.init_state(cfg, K, V, n0)
    outs, t3s = [], []
    for t in range(steps):
        outs.append(O.decode_step(st, Q[t]))
        t3s.append(O.export_index(st, 0, 3))
    return st, outs, t3s, (K, V, Q)


def test_tiny_first_event_counts():                           # SURVEY §8d tiny row
    st, _, _, _ = _tiny_run(steps=1)
    assert O.census(st, 0).tolist() == [148 + 51, 52, 0, 5]


def test_prop1_bitwise_over_beta():                           # Prop. 1
    runs = [_tiny_run(hbm_bp=b, interval=8, steps=32) for b in (3000, 5000, 7000)]
    for st, outs, t3s, _ in runs[1:]:
        for a, b in zip(outs, runs[0][1]):
            assert np.array_equal(a, b)
        for a, b in zip(t3s, runs[0][2]):
            assert np.array_equal(a, b)
    # the T0/T1 split really differs between the runs
    assert O.census(runs[0][0], 0)[1] != O.census(runs[2][0], 0)[1]


def test_r0_equals_full_attention_sdpa():                     # Prop. 1 + north star pin
    st, outs, _, (K, V, Q) = _tiny_run(hbm_bp=3000, evict_bp=0, interval=8, steps=20)
    n0 = 255
    for t in (0, 9, 19):
        n = n0 + t + 1
        k = torch.from_numpy(S.bf16_bits_to_f32(K[0, 0, :, :n]).astype(np.float64))   # [Hkv][n][d]
        v = torch.from_numpy(S.bf16_bits_to_f32(V[0, 0, :, :n]).astype(np.float64))
        q = torch.from_numpy(S.bf16_bits_to_f32(Q[t, 0, 0]).astype(np.float64))       # [Hq][d]
        G = 2
        ref = torch.nn.functional.scaled_dot_product_attention(
            q[:, None, :], k.repeat_interleave(G, 0), v.repeat_interleave(G, 0))[:, 0].numpy()
        assert np.allclose(outs[t][0, 0], ref, rtol=0, atol=1e-12)


def test_score_mass_and_monotone():                            # north star "sum = steps x heads"
    st, _, _, _ = _tiny_run(interval=8, steps=32)
    total = float(np.sum(st.S_part[0].astype(np.float64)))
    assert abs(total - 32 * 4 * 1) <= 1e-5 * 32 * 4            # t * H_q * L
    st2, _, _, _ = _tiny_run(interval=8, steps=31)
    assert np.all(st.S_part[0][:, :st2.n] >= st2.S_part[0][:, :st2.n])


def test_score_update_bruteforce_tiny():                        # S:151 brute force
    """Nested-loop Eq. 1 (S = sum over layers, heads of alpha) on a 2-layer run with
    no eviction; compares the fp32 scores within 1e-6 rel."""
    w = S.WORKLOADS["tiny"]
    L, steps, n0 = 2, 3, 40
    K = S.gen_kv(7, "k", L, 1, 2, 64, 0, n0 + steps, 16, 4)
    V = S.gen_kv(7, "v", L, 1, 2, 64, 0, n0 + steps, 16, 4)
    Q = S.gen_q(7, 0, steps, L, 1, 4, 2, 64)
    cfg = O.OracleConfig(B=1, L=L, Hq=4, Hkv=2, d=64, prompt_len=16, hbm_bp=5000, evict_bp=0)
    st = O.init_state(cfg, K, V, n0)
    for t in range(steps):
        O.decode_step(st, Q[t], manage=False)
    Kf, Qf = S.bf16_bits_to_f32(K), S.bf16_bits_to_f32(Q)
    ref = [0.0] * (n0 + steps)
    for t in range(steps):
        n = n0 + t + 1
        for l in range(L):
            for h in range(4):
                g = h // 2
                z = [sum(float(Qf[t, l, 0, h, k]) * float(Kf[l, 0, g, i, k]) for k in range(64)) / 8.0
                     for i in range(n)]
                m = max(z)
                Z = sum(math.exp(x - m) for x in z)
                for i in range(n):
                    ref[i] += math.exp(z[i] - m) / Z
    got = O.total_score_fp32(st.S_part[0])[: n0 + steps].astype(np.float64)
    assert np.allclose(got, ref, rtol=1e-6, atol=0)
    assert abs(sum(ref) - steps * L * 4) < 1e-9


def test_t2_variant_rows_and_codec():                           # AMB-11/12 stores
    st, outs, _, (K, V, Q) = _tiny_run(t2_bp=5000, interval=8, steps=32)
    cnt = O.census(st, 0)
    assert cnt[2] > 0
    Kf = S.bf16_bits_to_f32(K)
    for p in O.export_index(st, 0, 2):
        for g in range(2):
            c, s = O.quantize_int8(st.rowK[0, 0, g, p])
            assert np.array_equal(c, st.codeK[0, 0, g, p]) and s == st.scaleK[0, 0, g, p]
    # T0/T1 rows: the original generator bytes, or (token passed through T2) the
    # bf16 of a dequantised row -- one to three codec round trips (AMB-12)
    for tier in (0, 1):
        for p in O.export_index(st, 0, tier):
            for g in range(2):
                x, ok = Kf[0, 0, g, p], False
                for _ in range(4):
                    if np.array_equal(st.rowK[0, 0, g, p], x):
                        ok = True
                        break
                    x = O.f32_to_bf16_value(O.dequantize_int8(*O.quantize_int8(x)))
                assert ok, (tier, p, g)
    assert np.isfinite(outs[-1]).all()


def test_migration_rows_equal_generator_when_f2_zero():         # "migration is a copy"
    st, _, _, (K, V, Q) = _tiny_run(interval=8, steps=32)
    Kf, Vf = S.bf16_bits_to_f32(K), S.bf16_bits_to_f32(V)
    for tier in (0, 1):
        idx = O.export_index(st, 0, tier)
        assert np.array_equal(st.rowK[:, 0, :, idx], Kf[:, 0, :, idx])
        assert np.array_equal(st.rowV[:, 0, :, idx], Vf[:, 0, :, idx])


def test_generator_long_tail_calibration():                     # P:76 (top-20% -> 56.5%)
    """Recipe calibration: 7B head shapes, 2 layers, 64 steps, r=0."""
    L, steps, n0 = 2, 24, 1999
    K = S.gen_kv(2, "k", L, 1, 4, 128, 0, n0 + steps, 64, 4)
    V = S.gen_kv(2, "v", L, 1, 4, 128, 0, n0 + steps, 64, 4)
    Q = S.gen_q(2, 0, steps, L, 1, 28, 4, 128)
    cfg = O.OracleConfig(B=1, L=L, Hq=28, Hkv=4, d=128, prompt_len=64, evict_bp=0)
    st = O.init_state(cfg, K, V, n0)
    for t in range(steps):
        O.decode_step(st, Q[t], manage=False)
    s = np.sort(O.total_score_fp32(st.S_part[0][:, :st.n]))[::-1]
    share = s[: len(s) // 5].sum() / s.sum()
    assert 0.50 < share < 0.66, share


# --------------------------------------------------------------------- tier policies
def _pol_cfg(policy, budget=0, seed=0, P=4, ks=2, kw=3):
    return O.OracleConfig(B=1, L=1, Hq=1, Hkv=1, d=2, prompt_len=P, sink_size=ks, window_size=kw,
                          policy=policy, budget=budget, policy_seed=seed)


def test_splitmix64_reference_value():
    # first output of SplitMix64 from state 0 (the published reference value)
    assert O.splitmix64(0) == 0xE220A8397B1DCDAF


def test_streaming_keeps_exactly_the_protected_set():
    # StreamingLLM: sinks + window (+ prompt) survive, everything else is evicted
    n = 30
    cfg = _pol_cfg(O.POLICY_STREAMING)
    S = np.random.default_rng(1).random((1, n)).astype(np.float32)
    new = O.classify_request(S, np.zeros(n, np.uint8), n, cfg)
    prot = O.protected_mask(n, cfg.prompt_len, cfg.sink_size, cfg.window_size)
    assert np.array_equal(new == O.T0, prot) and np.array_equal(new == O.T3, ~prot)


def test_h2o_uniform_scores_reduce_to_recency():
    # uniform scores -> the tie-break keeps the newest tokens
    n, budget = 40, 15
    cfg = _pol_cfg(O.POLICY_H2O, budget=budget)
    new = O.classify_request(np.ones((1, n), np.float32), np.zeros(n, np.uint8), n, cfg)
    prot = O.protected_mask(n, cfg.prompt_len, cfg.sink_size, cfg.window_size)
    live = [p for p in range(n) if not prot[p]]
    keep = budget - int(prot.sum())
    assert [p for p in live if new[p] == O.T0] == live[-keep:]
    assert int((new == O.T0).sum()) == budget and set(np.unique(new)) <= {O.T0, O.T3}


def test_h2o_sort_and_take_brute_force():
    # distinct scores -> keep P plus the top budget - |P| live tokens by score
    rng = np.random.default_rng(7)
    for trial in range(20):
        n = int(rng.integers(12, 60))
        budget = int(rng.integers(1, n + 5))
        cfg = _pol_cfg(O.POLICY_H2O, budget=budget, P=int(rng.integers(0, 5)))
        S = rng.permutation(n).astype(np.float32)[None] * 0.25
        new = O.classify_request(S, np.zeros(n, np.uint8), n, cfg)
        prot = O.protected_mask(n, cfg.prompt_len, cfg.sink_size, cfg.window_size)
        live = [p for p in range(n) if not prot[p]]
        keep = min(len(live), max(0, budget - int(prot.sum())))
        top = sorted(live, key=lambda p: -S[0, p])[:keep]
        want = set(np.nonzero(prot)[0]) | set(top)
        assert set(np.nonzero(new == O.T0)[0]) == want and int((new == O.T3).sum()) == n - len(want)


def test_random_policy_determinism_and_uniformity():
    # deterministic given the seed; every live position kept with frequency keep/|U|
    n, budget = 40, 20
    cfg = _pol_cfg(O.POLICY_RANDOM, budget=budget, seed=3)
    S = np.zeros((1, n), np.float32)
    a = O.classify_request(S, np.zeros(n, np.uint8), n, cfg)
    b = O.classify_request(S, np.zeros(n, np.uint8), n, cfg)
    assert np.array_equal(a, b)
    prot = O.protected_mask(n, cfg.prompt_len, cfg.sink_size, cfg.window_size)
    live = np.nonzero(~prot)[0]
    keep = budget - int(prot.sum())
    freq = np.zeros(n)
    trials = 600
    for seed in range(trials):
        c = _pol_cfg(O.POLICY_RANDOM, budget=budget, seed=seed)
        freq += O.classify_request(S, np.zeros(n, np.uint8), n, c) == O.T0
    f = freq[live] / trials
    assert np.all(freq[prot] == trials)
    assert abs(f.mean() - keep / len(live)) < 1e-9                 # exactly `keep` per draw
    assert np.all(np.abs(f - keep / len(live)) < 0.1)              # uniform over positions


def test_policy_budget_covers_everything():
    # budget >= n keeps all
    n = 25
    for pol in (O.POLICY_H2O, O.POLICY_RANDOM):
        new = O.classify_request(np.random.default_rng(2).random((1, n)).astype(np.float32),
                                 np.zeros(n, np.uint8), n, _pol_cfg(pol, budget=n + 3, seed=1))
        assert np.all(new == O.T0)


# --------------------------------------------------------------------- VATP scorer
def _vatp_run(scale_v):
    from tests.oracle_runner import OracleRun
    from paper_2605_09490_b200 import harness as Hh
    w = Hh.workload("tiny", L=2, steps=4, interval=2, scorer=O.SCORER_VATP)
    r = OracleRun(w)
    if scale_v != 1.0:                       # scale every V row exactly (power of two)
        r.st.rowV *= scale_v
        r.st.vnorm *= scale_v
    outs = [r.step() for _ in range(w["steps"])]
    return r, outs


def test_vatp_scales_with_value_norms():
    # property pin: doubling every value row (exact in bf16/fp32) doubles every VATP increment
    # and the attention output, and leaves the tiers unchanged; a wrong weight (K norm, no
    # weight, squared norm) breaks it
    r1, o1 = _vatp_run(1.0)
    r2, o2 = _vatp_run(2.0)
    assert np.array_equal(r2.st.S_part, 2 * r1.st.S_part)
    assert np.array_equal(r2.st.tier, r1.st.tier)
    for a, b in zip(o1, o2):
        assert np.allclose(b, 2 * a, rtol=1e-12, atol=0)


def test_vatp_weights_are_value_row_norms():
    # one layer, one kv head, unit probability mass on a single token: the increment is that
    # token's ||v|| (brute force on a hand-built state)
    V = np.array([[3.0, 4.0], [0.0, 1.0], [6.0, 8.0]], np.float32)
    vn = O.value_norms(V)
    assert vn.tolist() == [5.0, 1.0, 10.0]
    class St:
        vnorm = vn[None, None, None, :]
    inc = O.score_increment(np.array([0.25, 0.5, 0.25]), St, 0, 0, 0, np.arange(3))
    assert inc.tolist() == [1.25, 0.5, 2.5]


# ------------------------------------------------ redundancy / combined scorers
def test_ordered_bits_sorts_like_the_values():
    # order pin: ranking by ordered_bits equals ranking by value for mixed signs, and equals
    # the raw-bit order of AMB-7 on non-negative values
    rng = np.random.default_rng(5)
    f = np.concatenate([rng.standard_normal(500), [0.0, 1e-40, -1e-40, 3.4e38, -3.4e38]]).astype(np.float32)
    ob = O.ordered_bits(f)
    assert np.array_equal(np.argsort(ob, kind="stable"), np.argsort(f, kind="stable"))
    pos = np.abs(f)
    assert np.array_equal(np.argsort(O.ordered_bits(pos), kind="stable"),
                          np.argsort(pos.view(np.uint32), kind="stable"))


def test_key_redundancy_bruteforce_and_closed_forms():
    # brute force in plain Python (math.fsum / math.sqrt) on a tiny random K, plus closed forms:
    # a scaled copy of the previous key has cosine 1, its negation -1, a zero row 0, position 0 is 0
    rng = np.random.default_rng(9)
    L, B, Hkv, N, d = 3, 2, 2, 7, 5
    K = rng.standard_normal((L, B, Hkv, N, d)).astype(np.float32)
    K[:, 0, 0, 3] = 2.0 * K[:, 0, 0, 2]          # cos = 1 at i = 3
    K[:, 0, 1, 4] = -K[:, 0, 1, 3]               # cos = -1 at i = 4
    K[:, 1, 0, 5] = 0.0                          # zero row: cos(k5, k4) = cos(k6, k5) = 0
    R = O.key_redundancy(K)
    for b in range(B):
        for g in range(Hkv):
            for i in range(N):
                acc = np.float32(0)
                for l in range(L):
                    c = 0.0
                    if i > 0:
                        a = [float(x) for x in K[l, b, g, i]]
                        p = [float(x) for x in K[l, b, g, i - 1]]
                        na, nb = math.fsum(x * x for x in a), math.fsum(x * x for x in p)
                        if na > 0 and nb > 0:
                            c = math.fsum(x * y for x, y in zip(a, p)) / math.sqrt(na * nb)
                    acc = np.float32(acc + np.float32(c))
                assert abs(float(R[b, g, i]) - float(acc)) <= 2e-6 * L, (b, g, i)
    assert R[0, 0, 3] == pytest.approx(L, abs=1e-5)
    assert R[0, 1, 4] == pytest.approx(-L, abs=1e-5)
    assert R[1, 0, 5] == 0.0 and R[1, 0, 6] == 0.0
    assert np.all(R[:, :, 0] == 0.0)


def _red_cfg(scorer, L=2, Hkv=2, P=2, ks=1, kw=2, hbm_bp=5000, evict_bp=2500):
    return O.OracleConfig(B=1, L=L, Hq=Hkv, Hkv=Hkv, d=4, prompt_len=P, sink_size=ks, window_size=kw,
                          hbm_bp=hbm_bp, evict_bp=evict_bp, scorer=scorer)


def test_redundancy_evicts_the_most_redundant_tokens_first():
    # P:713 "penalizes tokens with high cosine similarity to neighbors": with equal attention
    # scores the evicted tokens are exactly the live ones with the largest mean neighbour cosine
    n, Hkv = 13, 2
    cfg = _red_cfg(O.SCORER_REDUNDANCY, Hkv=Hkv)
    S = np.full((Hkv, n), 0.5, np.float32)
    rng = np.random.default_rng(3)
    R = rng.uniform(-2, 2, size=(Hkv, n)).astype(np.float32)
    new = O.classify_request(S, np.zeros(n, np.uint8), n, cfg, R_part_b=R)
    prot = O.protected_mask(n, cfg.prompt_len, cfg.sink_size, cfg.window_size)
    live = np.nonzero(~prot)[0]
    rho = [float(np.float32(np.float32(R[0, i] + R[1, i]) / np.float32(cfg.L * Hkv))) for i in live]
    order = [p for _, p in sorted(zip([-r for r in rho], live), key=lambda x: (x[0], x[1]))]
    n3 = int(len(live) * cfg.evict_bp // 10000)
    assert n3 >= 1
    assert sorted(np.nonzero(new == O.T3)[0].tolist()) == sorted(order[:n3])


def test_redundancy_reduces_to_attention_when_rho_is_constant():
    # special case: a constant redundancy shifts every key by the same amount, and S/S_max is
    # monotone in S, so the tiers equal the attention scorer's; the combined scorer likewise
    # reduces to VATP (same S input -> same tiers as the attention ranking of that S)
    n, Hkv = 40, 2
    rng = np.random.default_rng(11)
    S = rng.uniform(0.1, 3.0, size=(Hkv, n)).astype(np.float32)
    R = np.full((Hkv, n), 0.25, np.float32)
    base = O.classify_request(S, np.zeros(n, np.uint8), n, _red_cfg(O.SCORER_ATTENTION, hbm_bp=4000, evict_bp=1500))
    for sc in (O.SCORER_REDUNDANCY, O.SCORER_COMBINED):
        got = O.classify_request(S, np.zeros(n, np.uint8), n, _red_cfg(sc, hbm_bp=4000, evict_bp=1500), R_part_b=R)
        assert np.array_equal(got, base)


def test_classify_scores_closed_form():
    # I = S / S_max over the live set (protected positions excluded from the max), rho = mean
    # of R over layers x kv heads; a position whose S equals S_max and rho = 0 keys to 1
    cfg = _red_cfg(O.SCORER_REDUNDANCY, L=2, Hkv=2)
    S = np.array([100.0, 2.0, 4.0, 1.0], np.float32)
    live = np.array([False, True, True, True])
    R = np.array([[0.0, 0.5, 0.0, -1.0], [0.0, 0.5, 0.0, -1.0]], np.float32)
    k = O.classify_scores(S, R, live, cfg)
    assert k[2] == 1.0
    assert k[1] == np.float32(0.5) - np.float32(0.25)
    assert k[3] == np.float32(0.25) + np.float32(0.5)
    assert k[0] == np.float32(25.0)


def test_combined_increments_are_vatp_weighted():
    # the combined scorer accumulates the VATP increment (attention x ||v||); r = 0 so
    # the different rankings cannot change the visible set
    from paper_2605_09490_b200 import harness as Hh
    from tests.oracle_runner import OracleRun
    outs = {}
    for sc in (O.SCORER_VATP, O.SCORER_COMBINED):
        w = Hh.workload("tiny", L=2, steps=3, interval=64, scorer=sc, evict_bp=0)
        r = OracleRun(w)
        for _ in range(3):
            r.step()
        outs[sc] = r.st.S_part.copy()
    assert np.array_equal(outs[O.SCORER_VATP], outs[O.SCORER_COMBINED])


# --------------------------------------------------------------------- the decode loop at r > 0, T2, external
# update, lossy T2 exit (round-2 pins: each kills a plausible mutation of the oracle)
def _sdpa_masked(q, k, v, keep, G):
    """torch SDPA in float64 with a boolean mask: q [Hq][d], k/v [Hkv][n][d], keep [n]."""
    q = torch.as_tensor(q, dtype=torch.float64)
    k = torch.as_tensor(k, dtype=torch.float64).repeat_interleave(G, 0)
    v = torch.as_tensor(v, dtype=torch.float64).repeat_interleave(G, 0)
    mask = torch.as_tensor(keep)[None, None, :].expand(q.shape[0], 1, keep.shape[0])
    return torch.nn.functional.scaled_dot_product_attention(q[:, None, :], k, v, attn_mask=mask)[:, 0].numpy()


def test_decode_loop_masks_t3_at_r_gt_0():                    # Eq. 3 P:233-236 inside Alg. 1's loop
    """At r = 10 % the loop's o equals float64 SDPA over ALL positions with only the oracle's T3
    set masked (original generator rows: f2 = 0), and differs from full attention -- so an
    oracle that attends every position, or drops a live one, fails.  Brute force on one head."""
    st, outs, t3s, (K, V, Q) = _tiny_run(hbm_bp=3000, evict_bp=1000, interval=8, steps=20)
    Kf, Vf, Qf = (S.bf16_bits_to_f32(x).astype(np.float64) for x in (K, V, Q))
    n0, checked = 255, 0
    for t in (1, 8, 9, 16, 19):                                # steps after (and at) events
        n = n0 + t + 1
        ev = set(int(i) for i in t3s[t - 1])                   # T3 as the step's attention saw it
        assert len(ev) > 0
        keep = np.ones(n, dtype=bool)
        keep[list(ev)] = False
        ref = _sdpa_masked(Qf[t, 0, 0], Kf[0, 0, :, :n], Vf[0, 0, :, :n], keep, G=2)
        assert np.allclose(outs[t][0, 0], ref, rtol=0, atol=1e-12), t
        full = _sdpa_masked(Qf[t, 0, 0], Kf[0, 0, :, :n], Vf[0, 0, :, :n], np.ones(n, bool), G=2)
        assert np.abs(full - ref).max() > 1e-6                  # the mask matters at this step
        h = 3
        bf = _brute_attention(list(Qf[t, 0, 0, h]), Kf[0, 0, h // 2, :n].tolist(), Vf[0, 0, h // 2, :n].tolist(),
                              skip=ev)
        assert np.allclose(outs[t][0, 0, h], bf, rtol=0, atol=1e-12)
        checked += 1
    assert checked == 5


def test_decode_loop_attends_t2_as_code_times_scale():        # P:151, AMB-12
    """With f2 = 50 % the loop's o equals float64 SDPA over rows in which every T2 token is
    fp32(code x scale) of its stored codes (the codec is pinned above), T3 masked; and it
    differs measurably from SDPA over the full-precision rows."""
    w = S.WORKLOADS["tiny"]
    n0, steps = w["N"] - 1, 10
    K = S.gen_kv(w["seed"], "k", 1, 1, 2, 64, 0, n0 + steps, w["P"], 4)
    V = S.gen_kv(w["seed"], "v", 1, 1, 2, 64, 0, n0 + steps, w["P"], 4)
    Q = S.gen_q(w["seed"], 0, steps, 1, 1, 4, 2, 64)
    cfg = O.OracleConfig(B=1, L=1, Hq=4, Hkv=2, d=64, prompt_len=w["P"], manage_interval=8,
                         hbm_bp=5000, evict_bp=500, t2_bp=5000)
    st = O.init_state(cfg, K, V, n0)
    for t in range(9):                                         # events at t = 0 and 8
        O.decode_step(st, Q[t])
    t, n_att = 9, st.n + 1                                     # step 9 appends position st.n (T0)
    tier = st.tier[0, :n_att].copy()
    t2 = np.nonzero(tier == 2)[0]
    assert t2.size > 0 and tier[-1] == 0
    Kr = st.rowK[0, 0, :, :n_att].astype(np.float64)           # [Hkv][n][d] full-precision rows
    Vr = st.rowV[0, 0, :, :n_att].astype(np.float64)
    Kq, Vq = Kr.copy(), Vr.copy()
    for g in range(2):
        ck = torch.from_numpy(st.codeK[0, 0, g, t2].astype(np.float32))
        cv = torch.from_numpy(st.codeV[0, 0, g, t2].astype(np.float32))
        Kq[g, t2] = (ck * torch.from_numpy(st.scaleK[0, 0, g, t2])[:, None]).double().numpy()
        Vq[g, t2] = (cv * torch.from_numpy(st.scaleV[0, 0, g, t2])[:, None]).double().numpy()
    keep = tier != 3
    o = O.decode_step(st, Q[t])
    Qf = S.bf16_bits_to_f32(Q).astype(np.float64)
    ref = _sdpa_masked(Qf[t, 0, 0], Kq, Vq, keep, G=2)
    assert np.allclose(o[0, 0], ref, rtol=0, atol=1e-12)
    hi = _sdpa_masked(Qf[t, 0, 0], Kr, Vr, keep, G=2)
    assert np.abs(hi - ref).max() > 1e-5                      # dequantisation changes the output


def test_score_update_external_nested_loop():                 # Eq. 1, AMB-14
    rng = np.random.default_rng(11)
    Hkv, G, N = 3, 4, 40
    vis = np.array(sorted(rng.choice(N, size=25, replace=False)))
    probs = rng.random((Hkv * G, vis.size))
    S0 = rng.random((Hkv, N)).astype(np.float32)
    got = O.score_update_external(S0.copy(), vis, probs, G)
    want = S0.copy()
    for g in range(Hkv):
        for j, p in enumerate(vis):
            acc = 0.0
            for h in range(g * G, g * G + G):                  # every head of the group
                acc += float(probs[h, j])
            want[g, p] = np.float32(np.float32(want[g, p]) + np.float32(acc))
    assert np.array_equal(got, want)
    untouched = np.setdiff1d(np.arange(N), vis)
    assert np.array_equal(got[:, untouched], S0[:, untouched])


def test_row_leaving_t2_keeps_bf16_of_dequant():              # AMB-12 (lossy T2 exit)
    """Two crafted events: positions 3..6 go to T2 at the first, 3..5 return to T0 at the
    second.  Their stored rows must be bf16(code x scale) of the first quantisation
    (torch's bf16 rounding) -- not the original rows, which they differ from."""
    L, Hkv, d, n = 2, 1, 8, 12
    g = torch.Generator().manual_seed(3)
    Kb = (torch.randn((L, 1, Hkv, n, d), generator=g) * 1.7).to(torch.bfloat16)
    Vb = (torch.randn((L, 1, Hkv, n, d), generator=g) * 0.9).to(torch.bfloat16)
    bits = lambda x: x.view(torch.int16).numpy().view(np.uint16)
    cfg = O.OracleConfig(B=1, L=L, Hq=2, Hkv=Hkv, d=d, prompt_len=2, sink_size=1, window_size=2,
                         hbm_bp=5000, evict_bp=0, t2_bp=10000)
    st = O.init_state(cfg, bits(Kb), bits(Vb), n)
    st.S_part[0, 0, :n] = np.arange(n, dtype=np.float32)       # ascending: 3..6 lowest -> T2
    O.manage_event(st)
    assert np.nonzero(st.tier[0, :n] == 2)[0].tolist() == [3, 4, 5, 6]
    st.S_part[0, 0, :n] = np.arange(n, 0, -1, dtype=np.float32)   # descending: 3..5 highest -> T0
    O.manage_event(st)
    assert st.tier[0, 3:6].tolist() == [0, 0, 0]
    Kf, Vf = Kb.float().numpy(), Vb.float().numpy()
    for src, row in ((Kf, st.rowK), (Vf, st.rowV)):
        for p in (3, 4, 5):
            for l in range(L):
                c, s = O.quantize_int8(src[l, 0, 0, p])
                want = (torch.from_numpy(c.astype(np.float32)) * float(s)).to(torch.bfloat16).float().numpy()
                assert np.array_equal(row[l, 0, 0, p], want), (p, l)
        assert not np.array_equal(row[:, 0, 0, 3:6], src[:, 0, 0, 3:6])


# --------------------------------------------------------------------- windowed / R-KV scorers
# P:137 (R-KV's "last alpha = 8 observation tokens"), App. E P:972-978 (Z = lambda I - (1 - lambda) R,
# softmax of the last 8 observation tokens max-pooled with kernel 7, lambda = 0.07); AMB-32/33.
def test_max_pool_visible_matches_torch_max_pool1d():          # library routine on the compacted cache
    rng = np.random.default_rng(21)
    n = 60
    W = rng.random(n).astype(np.float32)
    tier = rng.integers(0, 4, size=n).astype(np.uint8)
    vis = np.nonzero(tier != O.T3)[0]
    got = O.max_pool_visible(W, vis)
    ref = torch.nn.functional.max_pool1d(torch.from_numpy(W[vis])[None, None], kernel_size=7, stride=1,
                                         padding=3)[0, 0].numpy()
    assert np.array_equal(got[vis], ref)
    # a T3 position is not a neighbour: the pool spans 3 non-T3 positions on each side
    W2 = np.zeros(12, np.float32)
    W2[5] = 9.0
    t2 = np.zeros(12, np.uint8)
    t2[[6, 7, 8]] = O.T3
    v2 = np.nonzero(t2 != O.T3)[0]
    p2 = O.max_pool_visible(W2, v2)
    assert [int(i) for i in v2 if p2[i] == 9.0] == [2, 3, 4, 5, 9, 10, 11]


def _event_inputs(scorer, interval, events, evict_bp=1000, L=2):
    """Runs the tiny oracle through ``events`` manage events (t = 0, Delta, ...) and captures
    (t, S_part, S_snap, tiers, n) of request 0 right before each classify (after the event
    step's score update).  Returns (run, captures)."""
    from paper_2605_09490_b200 import harness as Hh
    from tests.oracle_runner import OracleRun
    w = Hh.workload("tiny", L=L, steps=interval * (events - 1) + 1, interval=interval, scorer=scorer,
                    evict_bp=evict_bp)
    r = OracleRun(w)
    caps = []
    orig = O.manage_event

    def spy(st):
        caps.append((st.t, st.S_part[0].copy(), None if st.S_snap is None else st.S_snap[0].copy(),
                     st.tier[0, :st.n].copy(), st.n))
        orig(st)
    O.manage_event = spy
    try:
        for _ in range(w["steps"]):
            r.step()
    finally:
        O.manage_event = orig
    return r, caps


@pytest.mark.parametrize("interval", [4, 8, 16])
def test_windowed_score_is_brute_force_sum_over_the_last_w_steps(interval):
    """At an event t_e the windowed score of position i is the sum, over the last
    w = min(8, Delta) steps t_e-w+1 .. t_e, over layers and q heads, of the softmax probability
    of i (brute-force fp64 softmax over that step's visible set, original rows: f2 = 0), then
    max-pooled (kernel 7) over the non-T3 positions in position order (AMB-32).
    An off-by-one window moves every value by a whole step's mass and fails."""
    r, caps = _event_inputs(O.SCORER_WINDOW, interval, events=3)
    cfg = r.cfg
    w = O.observation_window(cfg)
    assert w == min(8, interval)
    Kf = S.bf16_bits_to_f32(r.K).astype(np.float64)
    inv = 1.0 / math.sqrt(cfg.d)
    n0 = r.w["N"] - 1
    for t_e, S_now, S_sn, tier, n in caps[1:]:
        assert n == n0 + t_e + 1
        keep = tier != O.T3                                     # T3 fixed since the last event (w <= Delta)
        Wb = np.zeros(n)
        for t in range(t_e - w + 1, t_e + 1):
            n_t = n0 + t + 1
            vis = np.nonzero(keep[:n_t])[0]
            Qf = S.bf16_bits_to_f32(r.Q[t]).astype(np.float64)
            for l in range(cfg.L):
                for h in range(cfg.Hq):
                    z = (Kf[l, 0, h // cfg.G, vis] @ Qf[l, 0, h]) * inv
                    e = np.exp(z - z.max())
                    Wb[vis] += e / e.sum()
        vis = np.nonzero(keep)[0]
        ref = np.zeros(n)
        for j in range(len(vis)):
            ref[vis[j]] = max(Wb[vis[x]] for x in range(max(0, j - 3), min(len(vis), j + 4)))
        got = O.windowed_scores(S_now, S_sn, tier, n)
        tol = 8 * np.finfo(np.float32).eps * float(S_now[:, :n].sum(0).max()) + 1e-6
        assert np.abs(got[vis] - ref[vis]).max() <= tol, (t_e, np.abs(got[vis] - ref[vis]).max(), tol)
        step_mass = cfg.L * cfg.Hq / n                          # mean mass of one step per position
        assert step_mass > 50 * tol


def test_windowed_score_at_the_first_event_is_the_cumulative_score():
    # the window cannot reach back before step 0: at t = 0 the snapshot is the initial S = 0
    _, caps = _event_inputs(O.SCORER_WINDOW, 16, events=1)
    t_e, S_now, S_sn, tier, n = caps[0]
    assert t_e == 0 and not S_sn.any()
    vis = np.nonzero(tier != O.T3)[0]
    assert np.array_equal(O.windowed_scores(S_now, S_sn, tier, n),
                          O.max_pool_visible(O.total_score_fp32(S_now[:, :n]), vis))


def test_rkv_closed_form():
    # Z = fp32(lambda * I) - fp32((1 - lambda) * rho), I = pooled / max over the live set, rho the
    # mean neighbour cosine over layers x kv heads (App. E; AMB-33)
    cfg = _red_cfg(O.SCORER_RKV, L=2, Hkv=2)
    S = np.array([100.0, 2.0, 4.0, 1.0], np.float32)
    live = np.array([False, True, True, True])
    R = np.array([[0.0, 0.5, 0.0, -1.0], [0.0, 0.5, 0.0, -1.0]], np.float32)
    k = O.classify_scores(S, R, live, cfg)
    lam, lam1 = np.float32(0.07), np.float32(0.93)
    assert k[2] == lam                                        # I = 1, rho = 0
    assert k[1] == np.float32(lam * np.float32(0.5)) - np.float32(lam1 * np.float32(0.25))
    assert k[3] == np.float32(lam * np.float32(0.25)) + np.float32(lam1 * np.float32(0.5))
    assert k[0] == np.float32(lam * np.float32(25.0))


def test_rkv_reduces_to_window_with_constant_redundancy_and_penalises_redundancy():
    """Special cases of Z = lambda I - (1 - lambda) R: a constant R shifts every key equally, so
    R-KV's tiers equal the windowed scorer's; a constant I leaves only -R, so the evicted tokens
    are the most redundant live ones."""
    n, Hkv = 40, 2
    rng = np.random.default_rng(13)
    S_now = rng.uniform(0.5, 3.0, size=(Hkv, n)).astype(np.float32)
    S_sn = (S_now * rng.uniform(0.0, 0.9, size=(Hkv, n))).astype(np.float32)
    tier = np.zeros(n, np.uint8)
    tier[[7, 19]] = O.T3
    Rc = np.full((Hkv, n), 0.3, np.float32)
    base = O.classify_request(S_now, tier, n, _red_cfg(O.SCORER_WINDOW, hbm_bp=4000, evict_bp=1500),
                              S_snap_b=S_sn)
    got = O.classify_request(S_now, tier, n, _red_cfg(O.SCORER_RKV, hbm_bp=4000, evict_bp=1500),
                             R_part_b=Rc, S_snap_b=S_sn)
    assert np.array_equal(got, base)
    # constant window mass: S_snap = S_now - c
    S_sn2 = (S_now - np.float32(0.25)).astype(np.float32)
    S_now2 = S_now.copy()
    S_now2[:] = np.float32(1.0)
    S_sn2[:] = np.float32(0.5)
    R = rng.uniform(-2, 2, size=(Hkv, n)).astype(np.float32)
    cfg = _red_cfg(O.SCORER_RKV, hbm_bp=4000, evict_bp=1500)
    new = O.classify_request(S_now2, np.zeros(n, np.uint8), n, cfg, R_part_b=R, S_snap_b=S_sn2)
    prot = O.protected_mask(n, cfg.prompt_len, cfg.sink_size, cfg.window_size)
    live = np.nonzero(~prot)[0]
    rho = {int(i): float(np.float32(np.float32(R[0, i] + R[1, i]) / np.float32(cfg.L * Hkv))) for i in live}
    order = sorted(live.tolist(), key=lambda i: (-rho[i], i))
    n3 = int(len(live) * cfg.evict_bp // 10000)
    assert n3 >= 1
    assert sorted(np.nonzero(new == O.T3)[0].tolist()) == sorted(order[:n3])


def test_window_scorer_tiers_differ_from_cumulative():
    """The windowed scorer is a different ranking from Eq. 1's cumulative one on the same run
    (P:137-140 contrasts them): at the second event the two tier arrays differ."""
    r_w, _ = _event_inputs(O.SCORER_WINDOW, 16, events=2, evict_bp=2000)
    r_a, _ = _event_inputs(O.SCORER_ATTENTION, 16, events=2, evict_bp=2000)
    assert not np.array_equal(r_w.st.tier, r_a.st.tier)
