"""ctypes binding of libkvsynth.so (GPU twin of synth.py; include/kv_synth.h)."""
import ctypes as C
import os

from .synth import SIG_A_DEFAULT

_lib = None


def load():
    global _lib
    if _lib is None:
        p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "lib", "libkvsynth.so")
        if not os.path.exists(p):
            raise FileNotFoundError(f"{p} missing: build first")
        lib = C.CDLL(p)
        lib.kv_synth_kv.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_void_p]
        lib.kv_synth_q.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_void_p, C.c_void_p]
        lib.kv_synth_kv.restype = C.c_int
        lib.kv_synth_kv_layer.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_void_p]
        lib.kv_synth_kv_layer.restype = C.c_int
        lib.kv_synth_q.restype = C.c_int
        _lib = lib
    return _lib


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def gen_kv(seed, which, L, B, Hkv, d, pos0, npos, prompt_len, sink_size, device, sig_a=SIG_A_DEFAULT, stream=None):
    """torch.bfloat16 [L][B][Hkv][npos][d] on `device` (same bytes as synth.gen_kv)."""
    import torch
    out = torch.empty((L, B, Hkv, npos, d), dtype=torch.bfloat16, device=device)
    rc = load().kv_synth_kv(seed, 0 if which == "k" else 1, L, B, Hkv, d, pos0, npos, prompt_len, sink_size,
                            float(sig_a), C.c_void_p(out.data_ptr()), _stream(stream))
    if rc:
        raise RuntimeError(f"kv_synth_kv failed: cuda error {rc}")
    return out


def gen_kv_layer(seed, which, layer, B, Hkv, d, pos0, npos, prompt_len, sink_size, device, sig_a=SIG_A_DEFAULT,
                 stream=None):
    """torch.bfloat16 [B][Hkv][npos][d]: layer `layer` of gen_kv's tensor (same bytes)."""
    import torch
    out = torch.empty((B, Hkv, npos, d), dtype=torch.bfloat16, device=device)
    rc = load().kv_synth_kv_layer(seed, 0 if which == "k" else 1, layer, B, Hkv, d, pos0, npos, prompt_len,
                                  sink_size, float(sig_a), C.c_void_p(out.data_ptr()), _stream(stream))
    if rc:
        raise RuntimeError(f"kv_synth_kv_layer failed: cuda error {rc}")
    return out


def gen_q(seed, t0, T, L, B, Hq, Hkv, d, device, stream=None):
    """torch.bfloat16 [T][L][B][Hq][d] on `device` (same bytes as synth.gen_q)."""
    import torch
    out = torch.empty((T, L, B, Hq, d), dtype=torch.bfloat16, device=device)
    rc = load().kv_synth_q(seed, t0, T, L, B, Hq, Hkv, d, C.c_void_p(out.data_ptr()), _stream(stream))
    if rc:
        raise RuntimeError(f"kv_synth_q failed: cuda error {rc}")
    return out
