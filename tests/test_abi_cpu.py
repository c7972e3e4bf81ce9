"""CPU-side checks of the C ABI (-m "not gpu"): the library builds for sm_100a, loads,
exports every symbol include/*.h declares, and validates configs without a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest
import torch

import __graft_entry__
from paper_2605_09490_b200 import kvtier as kt

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    __graft_entry__.build()


def _declared(header, api):
    src = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(api + r"\s+[\w\s\*]+?\b(kv_\w+)\s*\(", src)))


def _exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_every_declared_symbol_is_exported():
    for header, api, lib in (("kv_tier.h", "KV_TIER_API", "libkvtier.so"), ("kv_synth.h", "KV_SYNTH_API", "libkvsynth.so")):
        decl = _declared(header, api)
        assert len(decl) >= 3
        exp = _exported(kt.lib_path(lib))
        missing = [d for d in decl if d not in exp]
        assert not missing, (lib, missing)
    assert sorted(_declared("kv_tier.h", "KV_TIER_API")) == kt.EXPORTED


def test_sass_is_sm100a_and_uses_tensor_cores():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", kt.lib_path()], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out
    assert "HMMA" in out                 # mma.sync bf16 tiles in the decode kernel
    assert "UBLKCP" in out               # cp.async.bulk ring (TMA bulk copy engine)
    assert "SYNCS" in out                # mbarrier full/empty pipeline
    assert "UTCHMMA" in out              # tcgen05.mma (step kernel, step_kernel = 2)
    assert "LDTM" in out                 # tcgen05.ld: TMEM accumulators -> registers
    assert "UTCBAR" in out               # tcgen05.commit -> mbarrier


def test_library_loads_and_versions():
    assert "sm_100a" in kt.version()


def _cfg(**kw):
    base = dict(B=8, L=28, Hq=28, Hkv=4, d=128, max_tokens=2255, prompt_len=64)
    base.update(kw)
    return kt.make_config(**base)


def test_query_sizes_7b():
    # T0 holds the steady state (Alg. 1): |P| + top n_hbm + Delta appends, not the chain
    N, P, ks, kw, delta = 2255, 64, 4, 128, 64
    s = kt.query_sizes(_cfg())
    keep = (5000 * (N - (P + ks + kw)) + 9999) // 10000
    slack = max(16, delta) + 16
    assert s.cap_t0 == (P + ks + kw + keep + slack + 15) // 16 * 16
    assert s.cap_t0 < 0.62 * N
    assert s.cap_t1 >= N - (s.cap_t0 - slack)                   # a long prefix starts partly in T1 (AMB-26)
    # single-buffered K/V stores: L*B*Hkv*cap0*d*2 bytes each
    assert s.t0_store >= 2 * 28 * 8 * 4 * s.cap_t0 * 128 * 2
    assert s.t0_store < 2 * 2 * 28 * 8 * 4 * s.cap_t0 * 128 * 2
    assert s.host_t1 == 28 * 8 * 4 * N * 128 * 2 * 2
    assert s.device_arena >= s.t0_store + s.t1_staging + s.scores
    plain = 28 * 8 * N * 4 * 4 * 128
    assert s.device_arena < 1.25 * plain                        # T0 + all of T1 staged + metadata
    st = kt.query_sizes(_cfg(staging=0))                        # strict DDR residency
    assert st.device_arena < 0.8 * plain


@pytest.mark.parametrize("bad", [dict(d=96), dict(Hq=30), dict(Hq=36, Hkv=4), dict(hbm_bp=10001),
                                 dict(window_size=0), dict(staging=5)])
def test_invalid_configs_rejected(bad):
    with pytest.raises(kt.KvTierError) as e:
        kt.query_sizes(_cfg(**bad))
    assert e.value.status == -1


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_init_without_gpu_fails_loudly():
    cfg = _cfg(B=1, L=1, max_tokens=300)
    buf = kt.Buffers(device_arena=C.c_void_p(4096))
    h = C.c_void_p()
    st = kt.load().kv_tier_init(C.byref(cfg), C.byref(buf), None, C.byref(h))
    assert st == -2                      # E_CUDA: there is no CPU fallback


# --------------------------------------------------------------------- host logic without a GPU
def test_sequence_shard_store_sizing():
    # a sequence shard's stores hold its own positions only: T0 = owned rows
    # (+ one block), T1 = 1.25x its share + one block, host stores by owned row
    from paper_2605_09490_b200 import dist as D
    N, W = 16640, 8
    full = kt.query_sizes(kt.make_config(64, 80, 64, 8, 128, N, 64))
    for r in (0, 3, 7):
        s = kt.query_sizes(kt.make_config(64, 80, 64, 8, 128, N, 64, shard=kt.SHARD_SEQUENCE, rank=r, world=W))
        own = len(D.seq_owned_positions(N, W, r))
        assert own + 64 >= s.cap_t0 >= own and s.cap_t0 % 16 == 0
        assert s.cap_t1 < full.cap_t1 and s.cap_t1 >= 1.25 * full.cap_t1 / W
        assert s.host_t1 * W < 1.2 * full.host_t1
        assert s.device_arena < 180e9 < full.device_arena          # 70B fits one B200 per shard


def test_lse_combine_rejects_bad_arguments():
    # argument errors are detected synchronously, before any launch
    for args in ((None, None, 1, 1, 4, None, None), (1 << 20, 1 << 20, 1, 1, 6, 1 << 20, 1 << 20),
                 (1 << 20, 1 << 20, 0, 1, 4, 1 << 20, 1 << 20), (0x10008, 1 << 20, 1, 1, 4, 1 << 20, 1 << 20)):
        st = kt.load().kv_tier_lse_combine(*(C.c_void_p(a) if i in (0, 1, 5, 6) and a is not None else a
                                             for i, a in enumerate(args)), None)
        assert st == -1                                            # E_INVAL


@pytest.mark.parametrize("field,value", [("policy", 9), ("scorer", 6), ("scorer", -1), ("budget", 0),
                                         ("step_kernel", 4), ("step_kernel", -1)])
def test_policy_and_scorer_validation(field, value):
    kw = dict(policy=kt.POLICY_H2O, budget=100)
    kw[field] = value
    cfg = kt.make_config(2, 1, 4, 2, 64, 300, 16, **kw)
    s = kt.Sizes()
    assert kt.load().kv_tier_query_sizes(C.byref(cfg), C.byref(s)) == -1


def test_scorers_accepted_under_sequence_sharding():
    # every shard tracks the global previous key (R_part complete on each): accepted; the windowed
    # scorers are checked at kv_tier_init (they need the library's communicator)
    for sc, want in ((kt.SCORER_REDUNDANCY, 0), (kt.SCORER_COMBINED, 0), (kt.SCORER_VATP, 0),
                     (kt.SCORER_WINDOW, 0), (kt.SCORER_RKV, 0)):
        cfg = kt.make_config(2, 1, 4, 2, 64, 300, 16, scorer=sc, shard=kt.SHARD_SEQUENCE, world=2, rank=0)
        s = kt.Sizes()
        assert kt.load().kv_tier_query_sizes(C.byref(cfg), C.byref(s)) == want


def test_redundancy_scorers_size_their_buffers():
    # R_part [B][H_kv][N] fp32 + the previous key [L][B][H_kv][d] bf16 on top of the attention arena
    sz = {}
    for sc in (kt.SCORER_ATTENTION, kt.SCORER_REDUNDANCY):
        cfg = kt.make_config(2, 3, 4, 2, 64, 300, 16, scorer=sc)
        s = kt.Sizes()
        assert kt.load().kv_tier_query_sizes(C.byref(cfg), C.byref(s)) == 0
        sz[sc] = s.device_arena
    extra = sz[kt.SCORER_REDUNDANCY] - sz[kt.SCORER_ATTENTION]
    assert 2 * 2 * 300 * 4 + 3 * 2 * 2 * 64 * 2 <= extra <= 2 * 2 * 300 * 4 + 3 * 2 * 2 * 64 * 2 + 2 * 256


def test_window_scorers_size_their_buffers():
    # windowed: the snapshot [B][H_kv][N] + the pool scratch [B][N] fp32 + [B][N] int32; R-KV adds
    # R-KV's redundancy buffers on top (R_part + previous keys)
    sz = {}
    for sc in (kt.SCORER_ATTENTION, kt.SCORER_WINDOW, kt.SCORER_RKV, kt.SCORER_REDUNDANCY):
        cfg = kt.make_config(2, 3, 4, 2, 64, 300, 16, scorer=sc)
        s = kt.Sizes()
        assert kt.load().kv_tier_query_sizes(C.byref(cfg), C.byref(s)) == 0
        sz[sc] = s.device_arena
    win = 2 * 2 * 300 * 4 + 2 * 2 * 300 * 4
    assert win <= sz[kt.SCORER_WINDOW] - sz[kt.SCORER_ATTENTION] <= win + 2 * 256
    red = sz[kt.SCORER_REDUNDANCY] - sz[kt.SCORER_ATTENTION]
    assert win + red <= sz[kt.SCORER_RKV] - sz[kt.SCORER_ATTENTION] <= win + red + 4 * 256
    cfg = kt.make_config(2, 3, 4, 2, 64, 300, 16, scorer=kt.SCORER_WINDOW, manage_interval=0)
    assert kt.load().kv_tier_query_sizes(C.byref(cfg), C.byref(kt.Sizes())) == -1


def test_nccl_unique_id_and_init_guards():
    # the library resolves NCCL at run time: an id is 128 bytes and differs per call; an id is
    # refused for shard modes without a collective, and for bf16 o (the combine is fp32)
    a, b = kt.nccl_unique_id(), kt.nccl_unique_id()
    assert len(a) == kt.NCCL_ID_BYTES and a != b
    lib = kt.load()
    assert lib.kv_tier_nccl_unique_id(None, 128) == -1
    idb = C.create_string_buffer(a, kt.NCCL_ID_BYTES)
    h = C.c_void_p()
    buf = kt.Buffers(device_arena=C.c_void_p(1 << 20))
    for kw in (dict(shard=kt.SHARD_REQUEST), dict(shard=kt.SHARD_KVHEAD, world=2),
               dict(shard=kt.SHARD_SEQUENCE, world=2, out_fp32=0)):
        cfg = kt.make_config(2, 1, 4, 2, 64, 300, 16, **kw)
        assert lib.kv_tier_init(C.byref(cfg), C.byref(buf), idb, C.byref(h)) == -1


def test_window_scorer_on_sequence_shards_needs_the_communicator():
    # WINDOW pools over the global cache order: a sequence shard without the library's
    # communicator cannot see the other shards' scores, so kv_tier_init refuses it (before any GPU use)
    for sc in (kt.SCORER_WINDOW, kt.SCORER_RKV):
        cfg = kt.make_config(2, 1, 4, 2, 64, 300, 16, scorer=sc, shard=kt.SHARD_SEQUENCE, world=2, rank=0)
        buf = kt.Buffers(device_arena=C.c_void_p(1 << 20))
        h = C.c_void_p()
        assert kt.load().kv_tier_init(C.byref(cfg), C.byref(buf), None, C.byref(h)) == -1


def test_capture_entry_points_reject_null_ctx():
    lib = kt.load()
    assert lib.kv_tier_capture_begin(None) == -1
    assert lib.kv_tier_capture_end(None) == -1
    assert lib.kv_tier_graph_advance(None) == -1


def test_host_t1_entry_points_reject_null_ctx():
    # N1 entry points check their arguments before touching a device
    lib = kt.load()
    assert lib.kv_tier_set_host_t1(None, 1) == -1
    assert lib.kv_tier_host_t1_attention(None, 0, None, None, None) == -1
    assert lib.kv_tier_host_t1_score_update(None, 0, None, None) == -1
    assert lib.kv_tier_host_t1_layer(None, 0, None, None, None, None, None) == -1
