"""Build the in-tree CUDA libraries for sm_100a (called by __graft_entry__.build()).

    libkvtier.so  -- the product: C-ABI tiered-KV decode path (include/kv_tier.h)
    libkvsynth.so -- seeded synthetic-input generator (include/kv_synth.h), test plumbing
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(HERE, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xcompiler", "-fvisibility=hidden",
         "-Xcompiler", "-fopenmp", "-lgomp"]     # OpenMP: host-T1 attention (N1) on the host cores
if os.environ.get("KVT_TRACE_LOOP"):        # debug: per-stage wait/busy accounting in the trace
    FLAGS += ["-DKVT_TRACE_LOOP=1"]
if os.environ.get("KVT_NO_RED_DECODE"):     # experiment: no redundancy code in the decode kernel
    FLAGS += ["-DKVT_NO_RED_DECODE=1"]
if os.environ.get("KVT_FLAT_TRACE"):        # debug: per-unit epilogue timing in the flat kernel's trace
    FLAGS += ["-DKVT_FLAT_TRACE=1"]

TARGETS = {
    "libkvtier.so": ["csrc/ctx.cu", "csrc/attn.cu", "csrc/attn_flat.cu", "csrc/tiers.cu", "csrc/step.cu"],
    "libkvsynth.so": ["synth/synth.cu"],
}
DEPS = ["csrc/kv_internal.cuh", "csrc/decode_common.cuh", "../include/kv_tier.h", "../include/kv_synth.h"]


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(os.path.join(HERE, s)) > t for s in srcs + DEPS)


def build(force=False, verbose=False):
    os.makedirs(LIB_DIR, exist_ok=True)
    for name, srcs in TARGETS.items():
        out = os.path.join(LIB_DIR, name)
        if not force and not _stale(out, srcs):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, "-o", out, *[os.path.join(HERE, s) for s in srcs]]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB_DIR


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
