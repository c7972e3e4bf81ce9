"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on identical seeded inputs.

Bars (BASELINE.json north star, DESIGN.md AMB-17/18): tiers, index lists and migrated
T0/T1 bytes and T2 codes bit-exact; attention o within |g-o| <= 2e-3 + 1e-2|o|;
scores within 1e-5 relative.
"""
import numpy as np
import pytest
import torch

from oracle import kvtier_oracle as O
from paper_2605_09490_b200 import harness as H
from paper_2605_09490_b200 import kvtier as kt
from paper_2605_09490_b200.synth import synth as S
from tests.oracle_runner import OracleRun, o_close, s_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests (no CPU fallback exists)")
    import __graft_entry__
    __graft_entry__.build()


def _bf16_bits(a):
    return np.asarray(a, dtype=np.float32).view(np.uint32) >> 16


def _check_event_state(run, orc, reqs_gpu, layers=(0,)):
    """Tiers, index lists, census and store bytes after a manage event (store rows of the
    ctx's own kv heads when it holds a KV-head shard)."""
    kv = run.kv
    h0, hl = getattr(run, "heads", (0, run.w["Hkv"]))
    hs = slice(h0, h0 + hl)
    st = orc.st
    n = st.n
    tiers = kv.export(kt.X_TIERS)
    idx = [kv.export(w) for w in (kt.X_IDX_T0, kt.X_IDX_T1, kt.X_IDX_T2)]
    counts, _ = kv.census()
    for bo, bg in enumerate(reqs_gpu):
        want = st.tier[bo, :n]
        assert np.array_equal(tiers[bg], want), f"tiers differ for request {bg}"
        for T in range(3):
            assert np.array_equal(idx[T][bg], O.export_index(st, bo, T)), f"idx T{T} request {bg}"
        assert counts[bg].tolist() == O.census(st, bo).tolist()
    for l in layers:
        t0 = kv.export(kt.X_T0_ROWS, l)
        t1 = kv.export(kt.X_T1_ROWS, l)
        stg = kv.export(kt.X_STAGING, l) if run.w["staging"] != 0 else None
        for bo, bg in enumerate(reqs_gpu):
            for T, rows in ((0, t0), (1, t1)):
                pos = O.export_index(st, bo, T)
                wk = _bf16_bits(st.rowK[l, bo, hs][:, pos])            # [H_l][npos][d]
                wv = _bf16_bits(st.rowV[l, bo, hs][:, pos])
                assert np.array_equal(rows[bg][:, :, 0, :], wk), f"T{T} K rows layer {l} req {bg}"
                assert np.array_equal(rows[bg][:, :, 1, :], wv), f"T{T} V rows layer {l} req {bg}"
            if stg is not None:
                assert np.array_equal(stg[bg], t1[bg]), "HBM staging != pinned host T1 store"
        if run.w["t2_bp"]:
            codes = kv.export(kt.X_T2_CODES, l)
            scales = kv.export(kt.X_T2_SCALES, l)
            for bo, bg in enumerate(reqs_gpu):
                pos = O.export_index(st, bo, 2)
                assert np.array_equal(codes[bg][:, :, 0, :], st.codeK[l, bo, hs][:, pos])
                assert np.array_equal(codes[bg][:, :, 1, :], st.codeV[l, bo, hs][:, pos])
                assert np.array_equal(scales[bg][:, :, 0], st.scaleK[l, bo, hs][:, pos])
                assert np.array_equal(scales[bg][:, :, 1], st.scaleV[l, bo, hs][:, pos])


def _run_pair(w, reqs=None, graph=False, check_every=1, layers_api=False, split=0, variant=0, out_fp32=True,
              **run_kw):
    run = H.TieredDecode(w, split=split, variant=variant, out_fp32=out_fp32, **run_kw)
    orc = OracleRun(w, reqs=reqs)
    reqs_gpu = orc.reqs
    if graph:
        run.capture()
    worst = 0.0
    for t in range(w["steps"]):
        (run.step_layers() if layers_api else run.step())
        o_gpu = run.output()
        o_ref = orc.step()
        if t % check_every == 0 or run.is_event(t) or t == w["steps"] - 1:
            run.sync()
            ok, mabs, _ = o_close(o_gpu[:, reqs_gpu], o_ref)
            worst = max(worst, mabs)
            assert ok, f"attention o mismatch at step {t}: max abs {mabs}"
            S_gpu = run.kv.export(kt.X_SCORES)
            ok, mrel = s_close(S_gpu[reqs_gpu], orc.st.S_part[:, :, :orc.st.n])
            assert ok, f"scores mismatch at step {t}: max rel {mrel}"
            if orc.st.R_part is not None:          # redundancy partials (AMB-30): fp32 cosines
                R_gpu = run.kv.export(kt.X_REDUNDANCY)[reqs_gpu]
                err = np.abs(R_gpu - orc.st.R_part[:, :, :orc.st.n]).max()
                assert err <= 2e-6 * w["L"], f"redundancy mismatch at step {t}: {err}"
            if orc.st.S_snap is not None:          # windowed scorers: the window's start snapshot (AMB-32)
                ok, mrel = s_close(run.kv.export(kt.X_SNAPSHOT)[reqs_gpu], orc.st.S_snap[:, :, :orc.st.n])
                assert ok, f"snapshot mismatch at step {t}: max rel {mrel}"
            if run.is_event(t):
                _check_event_state(run, orc, reqs_gpu)
    run.close()
    return worst


# --------------------------------------------------------------------- generator
def test_synth_gpu_matches_cpu():
    from paper_2605_09490_b200.synth import synth_gpu as SG
    import __graft_entry__
    __graft_entry__.build()
    dev = torch.device("cuda:0")
    for which in ("k", "v"):
        g = SG.gen_kv(7, which, 3, 2, 2, 64, 100, 40, 16, 4, dev).view(torch.int16).cpu().numpy().view(np.uint16)
        c = S.gen_kv(7, which, 3, 2, 2, 64, 100, 40, 16, 4)
        assert np.array_equal(g, c)
    g = SG.gen_q(9, 5, 3, 2, 2, 8, 2, 128, dev).view(torch.int16).cpu().numpy().view(np.uint16)
    assert np.array_equal(g, S.gen_q(9, 5, 3, 2, 2, 8, 2, 128))
    full = SG.gen_kv(7, "k", 3, 2, 2, 64, 100, 40, 16, 4, dev)
    for l in range(3):                          # one layer at a time: the same bytes
        assert torch.equal(SG.gen_kv_layer(7, "k", l, 2, 2, 64, 100, 40, 16, 4, dev), full[l])


# --------------------------------------------------------------------- tiny end to end
def test_tiny_32_steps():                     # BASELINE.json configs[0]
    _run_pair(H.workload("tiny"))


def test_tiny_delta8_events():                # events at t = 0, 8, 16, 24
    _run_pair(H.workload("tiny", interval=8))


def test_tiny_t2_half():                      # f2 = 50 %: int8 T2 rows in attention + codec bytes
    _run_pair(H.workload("tiny", interval=8, t2_bp=5000))


@pytest.mark.parametrize("mchunk", ["1", "3", "0"])
def test_tiny_migrate_paths(mchunk, monkeypatch):   # in-place migrate in chunks of (layer, kv head) pairs
    monkeypatch.setenv("KVTIER_MCHUNK", mchunk)
    _run_pair(H.workload("tiny", interval=8, t2_bp=3000, B=2, L=2, Hkv=2, Hq=4), graph=True)


def test_tiny_per_event_mode():               # AMB-9 literal Alg. 1
    _run_pair(H.workload("tiny", interval=8, evict_mode=kt.EVICT_PER_EVENT, evict_bp=1000))


def test_tiny_stream_mode_layers_api():       # S = 0: T1 re-fetched from pinned host every step
    _run_pair(H.workload("tiny", interval=8, staging=0, L=3), layers_api=True)


def test_tiny_graph_stream_mode():
    _run_pair(H.workload("tiny", interval=8, staging=0, L=3, t2_bp=3000), graph=True)


@pytest.mark.parametrize("split", [1, 3, 8])
def test_tiny_layer_kernel_splits(split):     # per-layer kernel: CTAs per unit, PDL merge
    _run_pair(H.workload("tiny", interval=8, B=3, L=2, steps=17), split=split, layers_api=True)


@pytest.mark.parametrize("variant", range(6))
def test_multi_request_multi_layer_variants(variant):   # per-layer kernel variants: tiles, ragged tails, d = 128
    w = H.workload("tiny", B=3, L=2, Hq=12, Hkv=2, d=128, N=700, P=40, interval=16, steps=40,
                   hbm_bp=3000, evict_bp=1000, t2_bp=0 if variant == 3 else 2500)
    _run_pair(w, layers_api=True, check_every=7, variant=variant, split=(0, 4, 2, 3, 1, 16)[variant])


@pytest.mark.parametrize("variant", [0, 2, 5])
def test_tiny_variants(variant):                      # d = 64 kernels
    _run_pair(H.workload("tiny", interval=8, t2_bp=3000, B=2, L=2, steps=20), layers_api=True, variant=variant)


# --------------------------------------------------------------------- 7B-shaped, sampled
def test_7b_sampled_requests():               # BASELINE.json configs[1], bench launch configuration
    w = H.workload("7b", steps=66)
    _run_pair(w, reqs=[0, 5], graph=True, check_every=16)


def test_7b_sampled_requests_bf16_out():      # the bench's exact launch configuration: o stored as bf16
    w = H.workload("7b", steps=66)
    _run_pair(w, reqs=[2, 7], graph=True, check_every=16, out_fp32=False)


# --------------------------------------------------------------------- larger BASELINE shapes, sampled
@pytest.mark.parametrize("name,B,req,steps", [("14b", 2, 1, 2), ("32b", 1, 0, 2), ("70b", 1, 0, 1)])
def test_large_shapes_sampled_requests(name, B, req, steps):
    # BASELINE.json configs[2..4] per-request shapes (all layers, heads and tokens; fewer
    # requests so one GPU and the CPU oracle fit): the t = 0 event (+ one step) through the
    # bench's launch configuration (step graph, PDL chain), one request checked
    w = H.workload(name, B=B, steps=steps)
    _run_pair(w, reqs=[req], graph=True, check_every=1)


# --------------------------------------------------------------------- classify cross-fed
@pytest.mark.parametrize("kind", ["ties", "cont"])
def test_classify_crossfed_bit_exact(kind):   # AMB-18 (i): identical S -> identical tiers
    w = H.workload("tiny", B=4, L=1, N=3000, P=64, steps=3, interval=1, hbm_bp=3000, evict_bp=700,
                   t2_bp=4000)
    run = H.TieredDecode(w)
    cfg = O.OracleConfig(B=4, L=1, Hq=4, Hkv=2, d=64, prompt_len=64, hbm_bp=3000, evict_bp=700, t2_bp=4000)
    tier = np.zeros((4, 3002), np.uint8)
    for t in range(3):
        with torch.cuda.stream(run.main):
            run.kv.step(run.Q[t], run.Kn[t], run.Vn[t], run.O, 1, stream=run.main, side=run.side)
        run.sync()
        n = run.kv.position()[0]
        Sp = S.gen_scores(100 + t, 4, 2, n, kind)
        run.kv.import_scores(Sp)
        run.kv.classify(stream=run.main)
        run.kv.migrate(stream=run.main, side=run.side)
        run.sync()
        got = run.kv.export(kt.X_TIERS)
        tier[:, n - 1] = 0
        for b in range(4):
            want = O.classify_request(Sp[b], tier[b], n, cfg)
            assert np.array_equal(got[b], want), (t, b)
            tier[b, :n] = want
    run.close()


# --------------------------------------------------------------------- Prop. 1 on the GPU
def test_prop1_gpu_outputs_independent_of_beta():
    outs, t3 = [], []
    for beta in (3000, 5000, 7000):
        w = H.workload("tiny", interval=8, hbm_bp=beta, B=2, L=2)
        run = H.TieredDecode(w)
        run.capture()
        seq = []
        for t in range(w["steps"]):
            run.step()
            seq.append(run.output().copy())
        run.sync()
        outs.append(np.stack(seq))
        t3.append(run.kv.export(kt.X_TIERS) == 3)
        run.close()
    for k in (1, 2):
        assert np.array_equal(t3[k], t3[0])
        # bitwise equality holds in the oracle (ascending-position sums); on the GPU the
        # T0/T1 split changes the chunking and so the fp32 summation order (p enters the P.V
        # MMA as hi + lo bf16 terms): equal to fp32 rounding, far inside the parity tolerance
        mabs = float(np.abs(outs[k] - outs[0]).max())
        assert mabs < 1e-4, mabs


def test_graph_equals_step_calls_bitwise():
    # the step graph and kv_tier_step run the same whole-step kernel with the same work split:
    # identical bits
    w = H.workload("tiny", interval=8, B=2, L=2, t2_bp=3000)
    a = H.TieredDecode(w)
    b = H.TieredDecode(w)
    b.capture()
    for t in range(w["steps"]):
        a.step()
        b.step()
        oa, ob = a.output(), b.output()
        assert np.array_equal(oa, ob), t
    a.sync(); b.sync()
    assert np.array_equal(a.kv.export(kt.X_SCORES), b.kv.export(kt.X_SCORES))
    a.close(); b.close()


def test_step_kernel_matches_layer_kernel():
    # whole-step kernel (kv_tier_step) vs the per-layer kernels (decode_attention per layer): the
    # same softmax summed in a different order -> fp32 rounding apart; T0 rows byte-equal
    w = H.workload("tiny", interval=8, B=3, L=3, t2_bp=3000, Hq=12, Hkv=2, d=128, N=700, P=40)
    a = H.TieredDecode(w)
    b = H.TieredDecode(w)
    b.capture()
    for t in range(w["steps"]):
        a.step_layers()
        b.step()
        oa, ob = a.output(), b.output()
        assert np.abs(oa - ob).max() <= 2e-6 + 1e-5 * np.abs(oa).max(), t
    a.sync(); b.sync()
    ok, mrel = s_close(b.kv.export(kt.X_SCORES), a.kv.export(kt.X_SCORES))
    assert ok, mrel
    assert np.array_equal(a.kv.export(kt.X_T0_ROWS, 2)[1], b.kv.export(kt.X_T0_ROWS, 2)[1])
    a.close(); b.close()


def test_step_kernel_none_runs_the_layer_kernels():
    # step_kernel = 3: kv_tier_step / the step graph run the per-layer kernels -> bit-identical to
    # driving decode_attention layer by layer (same kernels, same split, same order)
    w = H.workload("tiny", interval=8, B=3, L=3, t2_bp=3000, Hq=12, Hkv=2, d=128, N=700, P=40)
    a = H.TieredDecode(w)
    b = H.TieredDecode(w, step_kernel=3)
    assert b.kv.layout()[1][0] == 0            # no whole-step kernel shape
    b.capture()
    for t in range(w["steps"]):
        a.step_layers()
        b.step()
        assert np.array_equal(a.output(), b.output()), t
    a.sync(); b.sync()
    assert np.array_equal(a.kv.export(kt.X_SCORES), b.kv.export(kt.X_SCORES))
    a.close(); b.close()


def test_stream_mode_equals_differential_bitwise():   # same rows, same order -> same bits
    # both through the per-layer kernels (stream mode always runs them; the differential run
    # uses the per-layer ABI so the work split is the same)
    outs = []
    for staging in (kt.STAGING_ALL, 0):
        w = H.workload("tiny", interval=8, B=2, L=3, staging=staging)
        run = H.TieredDecode(w)
        seq = []
        for _ in range(w["steps"]):
            run.step_layers()
            seq.append(run.output().copy())
        outs.append(np.stack(seq))
        run.close()
    assert np.array_equal(outs[0], outs[1])


# --------------------------------------------------------------------- standalone score update
def test_score_update_external_matches_oracle():
    w = H.workload("tiny", interval=8, B=2, L=1, steps=12)
    run = H.TieredDecode(w)
    cfg_G = w["Hq"] // w["Hkv"]
    for t in range(12):
        run.step()
    run.sync()
    S_before = run.kv.export(kt.X_SCORES).copy()
    tiers = run.kv.export(kt.X_TIERS)
    nvis = run.kv.visible_count()
    rng = np.random.default_rng(0)
    probs = rng.random((2, w["Hq"], nvis)).astype(np.float32)
    run.kv.score_update(0, torch.from_numpy(probs).cuda(), stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    got = run.kv.export(kt.X_SCORES)
    for b in range(2):
        vis = np.nonzero(tiers[b] != 3)[0]
        assert len(vis) == nvis
        want = O.score_update_external(S_before[b].copy(), vis, probs[b], cfg_G)
        assert np.array_equal(got[b], want) or s_close(got[b], want)[0]
    run.close()


# --------------------------------------------------------------------- error behaviour
def test_abi_errors():
    w = H.workload("tiny", steps=2)
    run = H.TieredDecode(w)
    with pytest.raises(kt.KvTierError) as e:
        run.kv.migrate(stream=run.main, side=run.side)
    assert e.value.status == -4                       # E_STATE: migrate without classify
    with pytest.raises(kt.KvTierError) as e:
        run.kv.decode_attention(5, run.Q[0, 0], run.O[0], 1, stream=run.main)
    assert e.value.status == -1                       # E_INVAL: layer out of range
    run.step()
    run.step()
    with pytest.raises(kt.KvTierError) as e:          # E_CAPACITY: N_max reached
        run.kv.step(run.Q[1], run.Kn[1], run.Vn[1], run.O, 1, stream=run.main, side=run.side)
    assert e.value.status == -5
    run.close()


# --------------------------------------------------------------------- whole-step kernel shapes
# kv_tier_step picks (slices per kv head s, heads per CTA m, warps per CTA) from the config;
# these shapes drive its extremes: one head cut into 16 slices, many heads per CTA, d = 64,
# G = 1 and G = 8, a ragged T2 segment, events every 4 steps.
@pytest.mark.parametrize("shape", [
    dict(B=1, Hq=8, Hkv=1, d=128, N=900, P=16),         # 1 kv head over a 16-CTA cluster
    dict(B=24, Hq=16, Hkv=8, d=64, N=120, P=16),        # 192 heads: several heads per CTA
    dict(B=3, Hq=3, Hkv=3, d=128, N=333, P=20),         # G = 1
    dict(B=2, Hq=16, Hkv=2, d=64, N=701, P=64)])        # G = 8, d = 64
def test_step_kernel_shapes(shape):
    w = H.workload("tiny", L=3, interval=4, steps=13, hbm_bp=4000, evict_bp=800, t2_bp=3000, **shape)
    _run_pair(w, graph=True, check_every=2)


@pytest.mark.parametrize("G,Hkv,s", [(7, 4, 4), (5, 4, 2), (8, 2, 3), (1, 4, 9), (2, 2, 16)])
def test_umma_step_kernel_parity(G, Hkv, s):
    # the tcgen05 / TMEM consumer of the whole-step kernel (d = 128, no T2 rows): S = K q^T and
    # O = V^T P^T on the 5th-generation tensor cores, online softmax on the CUDA cores; every
    # event's tiers / rows and o / scores against the oracle, across head ratios and cluster sizes
    w = H.workload("tiny", B=2, L=3, Hq=G * Hkv, Hkv=Hkv, d=128, N=900, P=64, interval=8, steps=18,
                   hbm_bp=4000, evict_bp=800, t2_bp=0)
    run = H.TieredDecode(w, split=s, step_kernel=2)
    shape = run.kv.layout()[1]
    run.close()
    assert shape[0] > 0 and shape[1] == s and shape[3] == 5, shape      # the tcgen05 consumer
    _run_pair(w, graph=True, check_every=2, split=s, step_kernel=2)


def test_umma_step_kernel_equals_mma_sync_consumer():
    # the two consumers of the whole-step kernel compute the same softmax in a different
    # summation order: fp32 rounding apart, T0 rows byte-equal
    w = H.workload("tiny", B=3, L=4, Hq=28, Hkv=4, d=128, N=1500, P=64, interval=8, steps=20, hbm_bp=5000,
                   evict_bp=500, t2_bp=0)
    a = H.TieredDecode(w, step_kernel=1)
    b = H.TieredDecode(w, step_kernel=2)
    assert a.kv.layout()[1][3] == 8 and b.kv.layout()[1][3] == 5
    a.capture()
    b.capture()
    for t in range(w["steps"]):
        a.step()
        b.step()
        oa, ob = a.output(), b.output()
        assert np.abs(oa - ob).max() <= 2e-6 + 1e-5 * np.abs(oa).max(), t
    a.sync(); b.sync()
    assert np.array_equal(a.kv.export(kt.X_TIERS), b.kv.export(kt.X_TIERS))
    assert np.array_equal(a.kv.export(kt.X_T0_ROWS, 1), b.kv.export(kt.X_T0_ROWS, 1))
    a.close(); b.close()


@pytest.mark.parametrize("s", [1, 2, 3, 5, 9, 16])
def test_step_kernel_slices_per_head(s):
    # the config's split fixes the cluster size (row slices per kv head): odd sizes, a 9-CTA and a
    # 16-CTA cluster, G = 5 (14B/32B head ratio), a ragged T2 segment
    w = H.workload("tiny", B=2, L=2, Hq=20, Hkv=4, d=128, N=900, P=64, interval=4, steps=9, hbm_bp=5000,
                   evict_bp=300, t2_bp=2500)
    run = H.TieredDecode(w, split=s)
    shape = run.kv.layout()[1]
    run.close()
    assert shape[1] == s or shape[0] == 0
    _run_pair(w, graph=True, check_every=2, split=s)


# --------------------------------------------------------------------- KV-head sharding (§8e row 2)
@pytest.mark.parametrize("world", [2, 4])
def test_kvhead_sharding_matches_unsharded_oracle(world):
    # world ctxs on one GPU, each owning H_kv/world kv heads; gathered scores at events
    w = H.workload("tiny", B=2, L=2, Hq=16, Hkv=4, d=64, N=400, P=16, interval=8, steps=26,
                   hbm_bp=4000, evict_bp=800, t2_bp=3000)
    sh = H.KvHeadShardedDecode(w, world)
    orc = OracleRun(w)
    sh.capture()
    for t in range(w["steps"]):
        sh.step()
        o_ref = orc.step()
        ok, mabs, _ = o_close(sh.output()[:, orc.reqs], o_ref)
        assert ok, (t, mabs)
        if sh.is_event(t) or t == w["steps"] - 1:
            S_gpu = sh.scores()
            ok, mrel = s_close(S_gpu[orc.reqs], orc.st.S_part[:, :, :orc.st.n])
            assert ok, (t, mrel)
            tiers = [r.kv.export(kt.X_TIERS) for r in sh.runs]
            for x in tiers[1:]:
                assert np.array_equal(x, tiers[0])            # every shard holds the same tiers
            for r in sh.runs:
                _check_event_state(r, orc, orc.reqs, layers=(0, 1))
    sh.close()


def test_redundancy_scorer_refused_in_classify_gathered():
    # R_part lives per shard, and the gathered classify would rank without it (AMB-31): refused
    w = H.workload("tiny", Hq=4, Hkv=2, steps=2, scorer=kt.SCORER_REDUNDANCY)
    sh = H.KvHeadShardedDecode(w, 2)
    with pytest.raises(kt.KvTierError):
        sh.step()                                    # t = 0 is an event
    sh.close()


def test_kvhead_plain_classify_refused():
    w = H.workload("tiny", Hq=4, Hkv=2, steps=2)
    run = H.TieredDecode(w, heads=(0, 1), shard=kt.SHARD_KVHEAD, rank=0, world=2)
    run.step(manage=False)
    with pytest.raises(RuntimeError):
        run.kv.classify(stream=run.main)
    run.close()


# --------------------------------------------------------------------- sequence sharding (§8e row 3)
def _check_seq_event_state(sh, orc, layers=(0, 1)):
    """Every shard holds the global tiers; its index lists, census and T0/T1 rows (and T2
    codes) are exactly the oracle's restricted to the positions it owns."""
    from paper_2605_09490_b200 import dist as D
    st = orc.st
    n = st.n
    for r, run in enumerate(sh.runs):
        kv = run.kv
        own = set(D.seq_owned_positions(n, sh.world, r))
        tiers = kv.export(kt.X_TIERS)
        idx = [kv.export(x) for x in (kt.X_IDX_T0, kt.X_IDX_T1, kt.X_IDX_T2)]
        counts, _ = kv.census()
        for bo, bg in enumerate(orc.reqs):
            assert np.array_equal(tiers[bg], st.tier[bo, :n]), f"shard {r}: tiers differ"
            want = [[p for p in O.export_index(st, bo, T) if p in own] for T in range(3)]
            for T in range(3):
                assert idx[T][bg].tolist() == want[T], f"shard {r}: idx T{T}"
            n_own = sum(1 for p in range(n) if p in own)
            assert counts[bg].tolist() == [len(want[0]), len(want[1]), len(want[2]),
                                           n_own - len(want[0]) - len(want[1]) - len(want[2])]
        for l in layers:
            for T, x in ((0, kt.X_T0_ROWS), (1, kt.X_T1_ROWS)):
                rows = kv.export(x, l)
                for bo, bg in enumerate(orc.reqs):
                    pos = [p for p in O.export_index(st, bo, T) if p in own]
                    assert np.array_equal(rows[bg][:, :, 0, :], _bf16_bits(st.rowK[l, bo][:, pos]))
                    assert np.array_equal(rows[bg][:, :, 1, :], _bf16_bits(st.rowV[l, bo][:, pos]))
            if run.w["t2_bp"]:
                codes = kv.export(kt.X_T2_CODES, l)
                for bo, bg in enumerate(orc.reqs):
                    pos = [p for p in O.export_index(st, bo, 2) if p in own]
                    assert np.array_equal(codes[bg][:, :, 0, :], st.codeK[l, bo][:, pos])


@pytest.mark.parametrize("world,staging,scorer", [(2, kt.STAGING_ALL, 0), (3, kt.STAGING_ALL, 0), (2, 0, 0),
                                                  (2, kt.STAGING_ALL, kt.SCORER_REDUNDANCY),
                                                  (3, kt.STAGING_ALL, kt.SCORER_COMBINED)])
def test_sequence_sharding_matches_unsharded_oracle(world, staging, scorer):
    # world ctxs on one GPU, block-cyclic 64-position ownership; per-layer LSE combine of the
    # ranks' partials, global (M, L) back into the fused score update, summed scores at events;
    # staging 0: each shard re-fetches its own T1 rows from pinned host memory every step
    # redundancy / combined: every shard appends every new key to its previous-key state, so R_part
    # is complete on each shard and the gathered classify ranks I - rho exactly as unsharded
    w = H.workload("tiny", B=2, L=2, Hq=8, Hkv=2, d=64, N=400, P=16, interval=8, steps=26,
                   hbm_bp=4000, evict_bp=800, t2_bp=3000, staging=staging, scorer=scorer)
    sh = H.SeqShardedDecode(w, world)
    orc = OracleRun(w)
    for t in range(w["steps"]):
        sh.step()
        o = sh.output()
        ref = orc.step()
        ok, mabs, _ = o_close(o[:, orc.reqs], ref)
        assert ok, (t, mabs)
        if sh.is_event(t) or t == w["steps"] - 1:
            ok, mrel = s_close(sh.scores()[orc.reqs], orc.st.S_part[:, :, :orc.st.n])
            assert ok, (t, mrel)
            if sh.is_event(t):
                _check_seq_event_state(sh, orc)
    sh.close()


def test_sequence_shard_without_visible_tokens():
    # a shard owning no position yet (n < 64 * rank) contributes an empty partial (m = -inf, l = 0)
    w = H.workload("tiny", B=1, L=1, Hq=4, Hkv=2, d=64, N=60, P=8, interval=4, steps=6,
                   hbm_bp=5000, evict_bp=500, t2_bp=0)
    sh = H.SeqShardedDecode(w, 2)
    orc = OracleRun(w)
    for t in range(w["steps"]):
        sh.step()
        ok, mabs, _ = o_close(sh.output()[:, orc.reqs], orc.step())
        assert ok, (t, mabs)
    ok, mrel = s_close(sh.scores()[orc.reqs], orc.st.S_part[:, :, :orc.st.n])
    assert ok, mrel
    sh.close()


def test_sequence_shard_refuses_plain_paths():
    w = H.workload("tiny", steps=2)
    run = H.TieredDecode(w, shard=kt.SHARD_SEQUENCE, rank=1, world=2)
    with pytest.raises(kt.KvTierError):
        run.kv.step(run.Q[0], run.Kn[0], run.Vn[0], run.O, 1, stream=run.main, side=run.side)
    run.kv.begin_step(stream=run.main)
    with pytest.raises(kt.KvTierError):
        run.kv.decode_attention(0, run.Q[0, 0], run.O[0], 1, stream=run.main, k_new=run.Kn[0, 0], v_new=run.Vn[0, 0])
    run.close()


@pytest.mark.parametrize("graph,staging,scorer", [(True, kt.STAGING_ALL, 0), (False, kt.STAGING_ALL, 0), (True, 0, 0),
                                                  (True, kt.STAGING_ALL, kt.SCORER_WINDOW),
                                                  (True, kt.STAGING_ALL, kt.SCORER_RKV)])
def test_sequence_shard_library_communicator(graph, staging, scorer):
    # kv_tier_init with an nccl_unique_id: kv_tier_step runs every layer's all-gather of (o, m, l)
    # on the library's NCCL communicator, the LSE combine and the rescaled score update -- the
    # whole step captured as ONE CUDA graph -- and kv_tier_classify all-gathers S_part itself.
    # world = 1 (one GPU): the collective is the identity, the path and its state machine are
    # the multi-rank ones
    w = H.workload("tiny", B=2, L=3, Hq=8, Hkv=2, d=64, N=400, P=16, interval=8, steps=26,
                   hbm_bp=4000, evict_bp=800, t2_bp=3000, staging=staging, scorer=scorer)
    _run_pair(w, graph=graph, check_every=4, shard=kt.SHARD_SEQUENCE, rank=0, world=1,
              nccl_id=kt.nccl_unique_id())


def test_sequence_shard_library_communicator_7b_sampled():
    # 7B-shaped (28 layers, G = 7, d = 128) through the communicator path, requests 2 and 7
    w = H.workload("7b", steps=10, interval=4)
    _run_pair(w, reqs=[2, 7], graph=True, check_every=3, shard=kt.SHARD_SEQUENCE, rank=0, world=1,
              nccl_id=kt.nccl_unique_id())


def _seq_proc_worker(rank, world, port, q):
    import os
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)   # one GPU: gloo via host memory
    try:
        w = H.workload("tiny", B=2, L=2, Hq=8, Hkv=2, d=64, N=400, P=16, interval=8, steps=18,
                       hbm_bp=4000, evict_bp=800, t2_bp=3000)
        sr = H.SeqShardRank(w, rank, world)
        orc = OracleRun(w)
        worst_o, worst_s = 0.0, 0.0
        for t in range(w["steps"]):
            sr.step()
            ok, mabs, _ = o_close(sr.output()[:, orc.reqs], orc.step())
            worst_o = max(worst_o, mabs)
            assert ok, (rank, t, mabs)
            if sr.is_event(t) or t == w["steps"] - 1:
                ok, mrel = s_close(sr.scores()[orc.reqs], orc.st.S_part[:, :, :orc.st.n])
                worst_s = max(worst_s, mrel)
                assert ok, (rank, t, mrel)
                assert np.array_equal(sr.run.kv.export(kt.X_TIERS)[orc.reqs], orc.st.tier[:, :orc.st.n])
        sr.close()
        q.put((rank, "ok", worst_o, worst_s))
    except Exception as e:                      # report to the parent
        q.put((rank, repr(e), 0.0, 0.0))
    finally:
        tdist.destroy_process_group()


def test_sequence_sharding_two_processes():
    # the multi-process driver (one ctx per process, per-layer all-gather of (o, m, l) over a
    # process group) against the unsharded oracle; two processes share the one GPU of this box
    import socket
    import torch.multiprocessing as mp
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_seq_proc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for rank, status, wo, ws in res:
        assert status == "ok", (rank, status)


# --------------------------------------------------------------------- negative controls,
# determinism (item 6): the parity checks must fail on an injected fault
def test_negative_control_flipped_tier_is_caught():
    # one live token's score is raised on the GPU side only (kv_tier_import_scores): at the next
    # event it lands in T0 on the GPU but not in the oracle, and the event-state check must fail
    w = H.workload("tiny", interval=8, steps=9)
    run = H.TieredDecode(w)
    orc = OracleRun(w)
    for t in range(8):
        run.step()
        orc.step()
    run.sync()
    S = run.kv.export(kt.X_SCORES).copy()
    t1 = O.export_index(orc.st, 0, O.T1)
    assert t1.size > 0
    S[0, :, t1[0]] += 1e3                                   # a T1 token becomes the heaviest hitter
    run.kv.import_scores(S)
    run.step()
    orc.step()
    run.sync()
    with pytest.raises(AssertionError):
        _check_event_state(run, orc, orc.reqs)
    run.close()


def test_negative_control_missing_token_is_caught():
    # the GPU evicts one token more than the oracle (r one step higher at the first event): the
    # tier / index / census checks must fail even when the attention outputs stay within tolerance
    w = H.workload("tiny", interval=8, steps=1)
    run = H.TieredDecode(dict(w, evict_bp=w["evict_bp"] + 100))      # floor(6.48) = 6 vs floor(5.4) = 5 of |U| = 108
    orc = OracleRun(w)
    run.step()
    orc.step()
    run.sync()
    assert run.kv.census()[0][0][3] == O.census(orc.st, 0)[3] + 1
    with pytest.raises(AssertionError):
        _check_event_state(run, orc, orc.reqs)
    run.close()


def test_two_runs_export_identical_bytes():
    # determinism: two runs of the same seeded workload give byte-identical outputs and exports
    w = H.workload("tiny", B=2, L=2, interval=8, steps=20, t2_bp=3000, evict_bp=800)
    res = []
    for _ in range(2):
        run = H.TieredDecode(w)
        run.capture()
        outs = []
        for _ in range(w["steps"]):
            run.step()
            outs.append(run.output())
        run.sync()
        res.append((np.stack(outs), [run.kv.export(x) for x in (kt.X_SCORES, kt.X_TIERS, kt.X_IDX_T1)],
                    run.kv.export(kt.X_T0_ROWS, 1), run.kv.export(kt.X_T2_CODES, 0)))
        run.close()
    a, b = res
    assert np.array_equal(a[0], b[0])
    for x, y in zip(a[1], b[1]):
        assert np.array_equal(x, y)
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])


# --------------------------------------------------------------------- tier policies (§8f N3)
@pytest.mark.parametrize("policy,budget", [(kt.POLICY_STREAMING, 0), (kt.POLICY_H2O, 300), (kt.POLICY_RANDOM, 300)])
def test_tier_policy_parity(policy, budget):
    # the paper's pure-eviction baselines on the same classify/migrate/decode path
    w = H.workload("tiny", B=3, L=2, Hq=8, Hkv=2, d=128, N=640, P=32, interval=8, steps=26,
                   hbm_bp=5000, evict_bp=500, t2_bp=0, policy=policy, budget=budget, policy_seed=11)
    _run_pair(w, graph=True, check_every=4)


def test_random_policy_request_keys_sampled_requests():
    # RANDOM keys depend on the request index: the oracle runs only requests 1 and 3
    w = H.workload("tiny", B=4, L=1, Hq=4, Hkv=2, d=64, N=500, P=16, interval=8, steps=18,
                   hbm_bp=5000, evict_bp=500, t2_bp=0, policy=kt.POLICY_RANDOM, budget=250, policy_seed=5)
    _run_pair(w, reqs=[1, 3], graph=True, check_every=8)


# --------------------------------------------------------------------- VATP scorer (§8f N2)
@pytest.mark.parametrize("api", ["graph", "layers"])
def test_vatp_scorer_parity(api):
    # value-aware scores: S += fp32(sum_h p) * ||v|| with the norms of the appended rows
    w = H.workload("tiny", B=3, L=2, Hq=8, Hkv=2, d=128, N=600, P=32, interval=8, steps=26,
                   hbm_bp=4000, evict_bp=800, t2_bp=3000, scorer=kt.SCORER_VATP)
    _run_pair(w, graph=api == "graph", layers_api=api == "layers", check_every=4)


@pytest.mark.parametrize("scorer", ["redundancy", "combined"])
@pytest.mark.parametrize("api", ["graph", "layers"])
def test_redundancy_scorer_parity(scorer, api):
    # "attn - redundancy" / "attn x val - redundancy": R_part from the loaded and
    # appended keys, signed classify keys I - rho (AMB-30/31); T2 on so keys leave / re-enter HBM
    sc = kt.SCORER_REDUNDANCY if scorer == "redundancy" else kt.SCORER_COMBINED
    w = H.workload("tiny", B=3, L=3, Hq=8, Hkv=2, d=128, N=600, P=32, interval=8, steps=26,
                   hbm_bp=4000, evict_bp=1200, t2_bp=3000, scorer=sc)
    _run_pair(w, graph=api == "graph", layers_api=api == "layers", check_every=4)


@pytest.mark.parametrize("scorer", ["window", "rkv"])
@pytest.mark.parametrize("api,interval", [("graph", 16), ("layers", 8), ("step", 4)])
def test_window_scorer_parity(scorer, api, interval):
    # windowed attention (last w = min(8, Delta) steps, max-pooled over the cache) and
    # R-KV's Z = 0.07 I - 0.93 R (App. E): S_part, the window snapshot, tiers, index
    # lists and rows at every event equal the oracle's (AMB-32/33); T2 on
    sc = kt.SCORER_WINDOW if scorer == "window" else kt.SCORER_RKV
    w = H.workload("tiny", B=3, L=3, Hq=8, Hkv=2, d=128, N=600, P=32, interval=interval, steps=2 * interval + 10,
                   hbm_bp=4000, evict_bp=1200, t2_bp=3000, scorer=sc)
    _run_pair(w, graph=api == "graph", layers_api=api == "layers", check_every=4)


def test_window_scorer_refused_in_classify_gathered():
    w = H.workload("tiny", Hq=4, Hkv=2, steps=2, scorer=kt.SCORER_WINDOW)
    sh = H.KvHeadShardedDecode(w, 2)
    with pytest.raises(kt.KvTierError):
        sh.step()                                    # t = 0 is an event
    sh.close()


def test_rkv_scorer_sampled_7b_requests():
    # the 7B-shaped config (d = 128, 28 layers, G = 7) with R-KV's scorer, requests 1 and 6
    w = H.workload("7b", steps=18, interval=8, scorer=kt.SCORER_RKV)
    _run_pair(w, reqs=[1, 6], check_every=4)


def test_redundancy_scorer_sampled_7b_requests():
    # the 7B-shaped config (d = 128, 28 layers) with the combined scorer, requests 0 and 5
    w = H.workload("7b", steps=10, interval=4, scorer=kt.SCORER_COMBINED)
    _run_pair(w, reqs=[0, 5], check_every=3)


# --------------------------------------------------------------------- N1: host-side T1 attention
@pytest.mark.parametrize("staging,d,fused", [(kt.STAGING_ALL, 128, False), (kt.STAGING_ALL, 128, True),
                                              (0, 128, True), (0, 64, False)])
def test_host_t1_attention_matches_oracle(staging, d, fused):
    # T1 attended on the host cores, T0 ∪ T2 on the GPU, combined by LSE (Eq. 3):
    # o, scores and every event's tiers / rows equal the oracle's full-attention run
    w = H.workload("tiny", B=3, L=2, Hq=8, Hkv=2, d=d, N=600, P=32, interval=8, steps=26,
                   hbm_bp=4000, evict_bp=800, t2_bp=3000, staging=staging)
    h = H.HostT1Decode(w, fused=fused)
    orc = OracleRun(w)
    for t in range(w["steps"]):
        h.step()
        ok, mabs, _ = o_close(h.output()[:, orc.reqs], orc.step())
        assert ok, (t, mabs)
        if t % 4 == 0 or h.is_event(t):
            h.sync()
            ok, mrel = s_close(h.run.kv.export(kt.X_SCORES)[orc.reqs], orc.st.S_part[:, :, :orc.st.n])
            assert ok, (t, mrel)
            if h.is_event(t):
                _check_event_state(h.run, orc, orc.reqs, layers=(0, 1))
    h.close()


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVT_FUZZ_SEEDS_H1", "16"))))
def test_randomized_host_t1(seed):
    # seeded draws incl. the degenerate ratios: beta = 100 % (no T1: the host partial is empty,
    # m = -inf) and beta = 0 (every live token in T1), T2 on/off, both staging modes, d = 64/128
    rng = np.random.default_rng(7000 + seed)
    Hkv = int(rng.choice([1, 2, 4]))
    w = H.workload("tiny", B=int(rng.integers(1, 4)), L=int(rng.integers(1, 4)), Hq=Hkv * int(rng.choice([1, 3, 8])),
                   Hkv=Hkv, d=int(rng.choice([64, 128])), N=int(rng.integers(150, 800)), P=int(rng.integers(0, 40)),
                   interval=int(rng.choice([4, 8])), steps=int(rng.integers(8, 18)),
                   hbm_bp=int(rng.choice([0, 10000, int(rng.integers(0, 10001))])), evict_bp=int(rng.integers(0, 2001)),
                   t2_bp=int(rng.choice([0, 3000])), staging=int(rng.choice([kt.STAGING_ALL, 0])),
                   evict_mode=int(rng.choice([kt.EVICT_TOTAL, kt.EVICT_PER_EVENT])))
    h = H.HostT1Decode(w, fused=bool(rng.integers(0, 2)))
    orc = OracleRun(w)
    for t in range(w["steps"]):
        h.step()
        ok, mabs, _ = o_close(h.output()[:, orc.reqs], orc.step())
        assert ok, (t, mabs)
        if h.is_event(t) or t == w["steps"] - 1:
            h.sync()
            ok, mrel = s_close(h.run.kv.export(kt.X_SCORES)[orc.reqs], orc.st.S_part[:, :, :orc.st.n])
            assert ok, (t, mrel)
            if h.is_event(t):
                _check_event_state(h.run, orc, orc.reqs, layers=tuple(range(w["L"])))
    h.close()


def test_host_t1_sampled_7b_requests():
    w = H.workload("7b", steps=6, interval=4, staging=0)
    h = H.HostT1Decode(w)
    orc = OracleRun(w, reqs=[0, 5])
    for t in range(w["steps"]):
        h.step()
        ok, mabs, _ = o_close(h.output()[:, orc.reqs], orc.step())
        assert ok, (t, mabs)
    h.sync()
    ok, mrel = s_close(h.run.kv.export(kt.X_SCORES)[orc.reqs], orc.st.S_part[:, :, :orc.st.n])
    assert ok, mrel
    h.close()


def test_host_t1_mode_guards():
    w = H.workload("tiny", steps=2)
    run = H.TieredDecode(w)
    run.kv.set_host_t1(True)
    with torch.cuda.stream(run.main):
        run.kv.begin_step(stream=run.main)
        with pytest.raises(kt.KvTierError):      # the GPU result alone would miss T1
            run.kv.decode_attention(0, run.Q[0, 0], run.O[0], 1, stream=run.main, k_new=run.Kn[0, 0], v_new=run.Vn[0, 0])
    run.close()
    r2 = H.TieredDecode(H.workload("tiny", steps=2, scorer=kt.SCORER_VATP))
    with pytest.raises(kt.KvTierError):
        r2.kv.set_host_t1(True)
    r2.close()


# --------------------------------------------------------------------- N4 (partial): inside a decoder
def test_model_decode_stream_mode_equals_differential_and_prop1():
    # the tiered attention inside a random-weight decoder (q/k/v from the layer's projections):
    # strict DDR residency (stream mode) gives bit-identical hidden states to differential
    # staging, and at r = 0 the HBM ratio changes nothing beyond rounding (Prop. 1)
    base = dict(B=2, L=3, Hq=8, Hkv=2, d=64, N=400, P=16, interval=4, steps=10, evict_bp=0)
    xs = {}
    for name, extra in (("diff50", dict(hbm_bp=5000)), ("stream50", dict(hbm_bp=5000, staging=0)),
                        ("hbm100", dict(hbm_bp=10000))):
        m = H.ModelDecode(H.workload("tiny", **base, **extra), hidden=256, inter=512)
        seq = []
        for _ in range(base["steps"]):
            seq.append(m.step().float().cpu().numpy())
        m.sync()
        xs[name] = np.stack(seq)
        m.close()
    assert np.array_equal(xs["diff50"], xs["stream50"])
    assert np.all(np.isfinite(xs["hbm100"]))
    # bf16 hidden states fed back through 3 layers x 10 steps: rounding differences of the
    # T0/T1 chunking grow to a few bf16 ulps (measured max 0.09 at |x| ~ 3), so compare in norm
    a, b = xs["diff50"].astype(np.float64), xs["hbm100"].astype(np.float64)
    rel = np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel <= 2e-2, rel


def _ref_decoder_step(m, x, caches):
    """Plain torch decoder step over whole K/V caches (no tiers): the model's own prefill K/V
    plus every appended row, fp32 softmax over all positions (Eq. 3 with nothing evicted)."""
    w = m.w
    B, Hq, Hkv, d = w["B"], w["Hq"], w["Hkv"], w["d"]
    G = Hq // Hkv
    for l, p in enumerate(m.layers):
        qkv = m._rms(x) @ p["wqkv"]
        q = qkv[:, :Hq * d].reshape(B, Hq, d).float()
        k = qkv[:, Hq * d:(Hq + Hkv) * d].reshape(B, Hkv, 1, d)
        v = qkv[:, (Hq + Hkv) * d:].reshape(B, Hkv, 1, d)
        K = torch.cat([caches[l][0], k], dim=2)
        V = torch.cat([caches[l][1], v], dim=2)
        caches[l] = (K, V)
        Kq = K.float().repeat_interleave(G, dim=1)                  # [B][Hq][n][d]
        Vq = V.float().repeat_interleave(G, dim=1)
        a = torch.softmax(torch.einsum("bhd,bhnd->bhn", q, Kq) / np.sqrt(d), dim=-1)
        o = torch.einsum("bhn,bhnd->bhd", a, Vq).to(torch.bfloat16)
        x = x + o.reshape(B, Hq * d) @ p["wo"]
        gu = m._rms(x) @ p["wgu"]
        x = x + (torch.nn.functional.silu(gu[:, :m.inter]) * gu[:, m.inter:]) @ p["wd"]
    return m._rms(x)


def test_model_prefill_initial_tiers_and_decode():
    # Alg. 1 line 1: C <- Prefill(M, x_1:P).  The decoder's own causal prefill produces
    # every layer's prefix K/V, the library loads them as the initial cache, and the decode
    # continues from the last prompt position.  With beta = 100 %, r = 0 (nothing leaves T0, Prop. 1)
    # the tiered decoder equals a plain torch decoder over the whole caches, step after step,
    # across the manage events; the t = 0 event classifies exactly the prefill's positions.
    base = dict(B=2, L=3, Hq=8, Hkv=2, d=64, N=300, P=16, interval=4, steps=9, evict_bp=0, hbm_bp=10000)
    m = H.ModelDecode(H.workload("tiny", **base), hidden=256, inter=512, prefill=True, keep_prefill=True)
    caches = list(m.prefill_kv)
    assert len(caches) == base["L"] and caches[0][0].shape == (2, 2, base["N"] - 1, 64)
    x = m.x.clone()
    for t in range(base["steps"]):
        got = m.step()
        x = _ref_decoder_step(m, x, caches)
        a, b = got.float().cpu().numpy().astype(np.float64), x.float().cpu().numpy().astype(np.float64)
        rel = np.linalg.norm(a - b) / np.linalg.norm(b)
        assert rel <= 2e-2, (t, rel)
        x = got.clone()                      # both continue from the library's hidden state
    m.sync()
    counts, _ = m.run.kv.layout()
    assert counts[3] == 0 and counts[0] == base["N"] - 1 + base["steps"]
    m.close()


def test_model_prefill_tiers_with_eviction():
    # the same prefill at beta 50 %, r 5 %: the t = 0 event splits the prefill's positions by
    # their step-0 scores (Alg. 1 lines 17-25); the census adds up and the decode stays finite
    base = dict(B=2, L=3, Hq=8, Hkv=2, d=64, N=300, P=16, interval=4, steps=6, evict_bp=500, hbm_bp=5000)
    m = H.ModelDecode(H.workload("tiny", **base), hidden=256, inter=512, prefill=True)
    outs = [m.step().float().cpu().numpy() for _ in range(base["steps"])]
    m.sync()
    counts, _ = m.run.kv.layout()
    assert sum(counts) == base["N"] - 1 + base["steps"] and counts[1] > 0 and counts[3] > 0
    assert np.all(np.isfinite(np.stack(outs)))
    m.close()


@pytest.mark.parametrize("staging", [kt.STAGING_ALL, 0])
def test_model_decode_graph_equals_eager(staging):
    # the whole decoder step as one CUDA graph (torch.cuda.graph around kv_tier_capture_begin /
    # _end, kv_tier_graph_advance per replay; events eager between replays) runs the same kernels
    # on the same data as the eager step: identical hidden states, scores and tiers
    base = dict(B=2, L=3, Hq=8, Hkv=2, d=64, N=400, P=16, interval=4, steps=14, evict_bp=800, hbm_bp=5000,
                staging=staging)
    outs, tiers, scores = [], [], []
    for graph in (False, True):
        m = H.ModelDecode(H.workload("tiny", **base), hidden=256, inter=512)
        seq = []
        for t in range(base["steps"]):
            if graph and t == 2:
                m.capture()
            seq.append(m.step().float().cpu().numpy())
        m.sync()
        outs.append(np.stack(seq))
        tiers.append(m.run.kv.export(kt.X_TIERS))
        scores.append(m.run.kv.export(kt.X_SCORES))
        m.close()
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(tiers[0], tiers[1])
    assert np.array_equal(scores[0], scores[1])


def test_lse_combine_kernel_matches_full_softmax():
    # kv_tier_lse_combine: shards of a softmax-weighted sum, combined in rank order, equal the
    # float64 softmax over the concatenation; an empty shard (m = -inf, l = 0) contributes nothing
    g = torch.Generator().manual_seed(3)
    W, rows, n, d = 4, 37, 90, 64
    z = torch.randn(rows, n, generator=g, dtype=torch.float64) * 3
    V = torch.randn(n, d, generator=g, dtype=torch.float64)
    ref = torch.softmax(z * np.log(2), dim=-1) @ V
    cuts = [0, 30, 30, 61, 90]                        # rank 1 owns nothing
    o_parts, lse_parts = [], []
    for r in range(W):
        zz, vv = z[:, cuts[r]:cuts[r + 1]], V[cuts[r]:cuts[r + 1]]
        if zz.shape[1] == 0:
            o_parts.append(torch.zeros(rows, d, dtype=torch.float64))
            lse_parts.append(torch.tensor([[-float("inf"), 0.0]] * rows, dtype=torch.float64))
            continue
        m = zz.max(dim=-1).values
        p = torch.exp2(zz - m[:, None])
        l = p.sum(dim=-1)
        o_parts.append(p @ vv / l[:, None])
        lse_parts.append(torch.stack([m, l], dim=-1))
    op = torch.stack(o_parts).float().cuda()
    lp = torch.stack(lse_parts).float().cuda()
    o, lse = kt.lse_combine(op, lp)
    torch.cuda.synchronize()
    assert (o.double().cpu() - ref).abs().max() < 1e-5
    M = z.max(dim=-1).values
    assert torch.equal(lse[:, 0].double().cpu(), M.float().double())
    L = torch.exp2(z - M[:, None]).sum(dim=-1)
    assert ((lse[:, 1].double().cpu() - L) / L).abs().max() < 1e-5


# --------------------------------------------------------------------- randomized configurations
@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVT_FUZZ_SEEDS", "64"))))
def test_randomized_configs(seed):
    # seeded draws over the configuration space (shapes, ratios, T2, eviction mode, interval,
    # staging, tier policy, scorer) against the oracle: catches interactions no fixed test covers
    rng = np.random.default_rng(1000 + seed)
    Hkv = int(rng.choice([1, 2, 4]))
    G = int(rng.choice([1, 2, 5, 7, 8]))
    d = int(rng.choice([64, 128]))
    N = int(rng.integers(150, 900))
    P = int(rng.integers(0, 48))
    pol = int(rng.choice([kt.POLICY_HIERARCHY] * 4 + [kt.POLICY_STREAMING, kt.POLICY_H2O, kt.POLICY_RANDOM]))
    w = H.workload("tiny", B=int(rng.integers(1, 5)), L=int(rng.integers(1, 4)), Hq=Hkv * G, Hkv=Hkv, d=d, N=N, P=P,
                   interval=int(rng.choice([4, 8, 16])), steps=int(rng.integers(10, 22)),
                   hbm_bp=int(rng.integers(0, 10001)), evict_bp=int(rng.integers(0, 2001)),
                   t2_bp=int(rng.choice([0, 0, 2500, 10000])),
                   evict_mode=int(rng.choice([kt.EVICT_TOTAL, kt.EVICT_PER_EVENT])),
                   staging=int(rng.choice([kt.STAGING_ALL, kt.STAGING_ALL, 0])),
                   policy=pol, budget=int(rng.integers(P + 140, N + 50)) if pol in (2, 3) else 0,
                   policy_seed=seed, scorer=int(rng.choice([0, 0, kt.SCORER_VATP, kt.SCORER_REDUNDANCY,
                                                             kt.SCORER_COMBINED, kt.SCORER_WINDOW,
                                                             kt.SCORER_RKV])))
    api = int(rng.integers(0, 3))             # step graph / kv_tier_step (whole-step kernel) / per-layer ABI
    sk = int(rng.choice([0, 2, 3]))           # whole-step consumer: mma.sync / tcgen05 (where it applies) / none
    _run_pair(w, graph=api == 0, layers_api=api == 2, check_every=3, step_kernel=sk)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("KVT_FUZZ_SEEDS_SEQ", "24"))))
def test_randomized_sequence_shards(seed):
    rng = np.random.default_rng(5000 + seed)
    Hkv = int(rng.choice([1, 2]))
    w = H.workload("tiny", B=int(rng.integers(1, 4)), L=int(rng.integers(1, 3)), Hq=Hkv * int(rng.choice([2, 4, 7])),
                   Hkv=Hkv, d=int(rng.choice([64, 128])), N=int(rng.integers(100, 700)), P=int(rng.integers(0, 40)),
                   interval=int(rng.choice([4, 8])), steps=int(rng.integers(8, 18)), hbm_bp=int(rng.integers(0, 10001)),
                   evict_bp=int(rng.integers(0, 1500)), t2_bp=int(rng.choice([0, 3000])),
                   staging=int(rng.choice([kt.STAGING_ALL, 0])),
                   scorer=int(rng.choice([0, 0, kt.SCORER_VATP, kt.SCORER_REDUNDANCY, kt.SCORER_COMBINED])))
    sh = H.SeqShardedDecode(w, int(rng.integers(2, 5)))
    orc = OracleRun(w)
    for t in range(w["steps"]):
        sh.step()
        ok, mabs, _ = o_close(sh.output()[:, orc.reqs], orc.step())
        assert ok, (t, mabs)
        if sh.is_event(t):
            ok, mrel = s_close(sh.scores()[orc.reqs], orc.st.S_part[:, :, :orc.st.n])
            assert ok, (t, mrel)
            _check_seq_event_state(sh, orc, layers=tuple(range(w["L"])))
    sh.close()
