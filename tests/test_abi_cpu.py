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


def test_library_loads_and_versions():
    assert "sm_100a" in kt.version()


def _cfg(**kw):
    base = dict(B=8, L=28, Hq=28, Hkv=4, d=128, max_tokens=2255, prompt_len=64)
    base.update(kw)
    return kt.make_config(**base)


def test_query_sizes_7b():
    s = kt.query_sizes(_cfg())
    assert s.cap_t0 >= 2255 and s.cap_t1 >= 1128
    # T0 ping-pong: 2 x K/V x L*B*Hkv*cap0*d*2 bytes
    assert s.t0_store >= 2 * 2 * 28 * 8 * 4 * s.cap_t0 * 128 * 2
    assert s.host_t1 == 28 * 8 * 4 * 2255 * 128 * 2 * 2
    assert s.device_arena >= s.t0_store + s.t1_staging + s.scores


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
