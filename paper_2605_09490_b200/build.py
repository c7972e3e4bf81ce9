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
if os.environ.get("KVT_TRACE"):             # debug builds: per-(layer, CTA) timeline buffer
    FLAGS += ["-DKVT_TRACE=1"]
if os.environ.get("KVT_INLINE_OFFLOAD"):    # A/B builds: the event's host offload inside the migrate kernel
    FLAGS += ["-DKVT_INLINE_OFFLOAD=1"]
if os.environ.get("KVT_SLEEP_CHAIN"):       # A/B builds: suspend (not spin) on the step kernel's layer chain
    FLAGS += ["-DKVT_SPIN_CHAIN=0"]

TARGETS = {
    "libkvtier.so": ["csrc/ctx.cu", "csrc/attn.cu", "csrc/tiers.cu", "csrc/step.cu"],
    "libkvsynth.so": ["synth/synth.cu"],
}
DEPS = ["csrc/kv_internal.cuh", "csrc/decode_common.cuh", "../include/kv_tier.h", "../include/kv_synth.h"]


def _stamp(cmd):
    """The nvcc command without absolute paths (the repo is checked out elsewhere on GPU boxes)."""
    return " ".join(os.path.relpath(x, HERE) if os.path.isabs(x) and x.startswith(os.path.dirname(HERE)) else x
                    for x in cmd[1:])


def _stale(out, srcs, cmd):
    """Out of date when missing, older than a source, or built with another nvcc command (the
    flags stamp next to the library: a debug build never silently stands in for the product)."""
    if not os.path.exists(out):
        return True
    stamp = out + ".cmd"
    if not os.path.exists(stamp) or open(stamp).read() != _stamp(cmd):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(os.path.join(HERE, s)) > t for s in srcs + DEPS)


def build(force=False, verbose=False):
    os.makedirs(LIB_DIR, exist_ok=True)
    for name, srcs in TARGETS.items():
        out = os.path.join(LIB_DIR, name)
        cmd = [NVCC, *ARCH, *FLAGS, "-o", out, *[os.path.join(HERE, s) for s in srcs]]
        if not force and not _stale(out, srcs, cmd):
            continue
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        with open(out + ".cmd", "w") as f:
            f.write(_stamp(cmd))
    return LIB_DIR


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
