"""Decode-loop driver over the C ABI (Alg. 1), used by tests and bench.py.

Inputs are the seeded synthetic workloads of synth.py, generated directly in HBM by
libkvsynth.so.  Every step of the method runs inside libkvtier.so; this module only
allocates buffers, orders the calls and times them.
"""
from __future__ import annotations

import torch

from . import kvtier as kt
from .synth import synth as S
from .synth import synth_gpu as SG


def workload(name, **over):
    w = dict(S.WORKLOADS[name])
    w.setdefault("interval", S.MANAGE_INTERVAL)
    w.setdefault("t2_bp", 0)
    w.setdefault("evict_mode", kt.EVICT_TOTAL)
    w.setdefault("staging", kt.STAGING_ALL)
    w.update(over)
    return w


class TieredDecode:
    """One ctx running workload `w` for w['steps'] decode steps on `device`.

    The chain holds n0 = N - 1 prefix tokens; step 0 appends position N - 1, so the
    first manage event (t = 0) sees exactly N tokens (reading AMB-22)."""

    def __init__(self, w, device="cuda:0", out_fp32=True, split=0, seed_offset=0, keep_inputs=False, variant=0):
        self.w = w
        self.dev = torch.device(device)
        torch.cuda.set_device(self.dev)
        B, L, Hq, Hkv, d, N, P, T = (w[k] for k in ("B", "L", "Hq", "Hkv", "d", "N", "P", "steps"))
        self.seed = w["seed"] + seed_offset
        self.n0 = N - 1
        self.T = T
        self.cfg = kt.make_config(B, L, Hq, Hkv, d, self.n0 + T, P, hbm_bp=w["hbm_bp"], evict_bp=w["evict_bp"],
                                  t2_bp=w["t2_bp"], manage_interval=w["interval"], evict_mode=w["evict_mode"],
                                  staging=w["staging"], device=self.dev.index or 0, out_fp32=int(out_fp32),
                                  split=split, variant=variant)
        self.kv = kt.KvTier(self.cfg)
        self.main = torch.cuda.Stream(self.dev)
        self.side = torch.cuda.Stream(self.dev)
        with torch.cuda.stream(self.main):
            K = SG.gen_kv(self.seed, "k", L, B, Hkv, d, 0, self.n0, P, S.SINK_SIZE, self.dev, stream=self.main)
            V = SG.gen_kv(self.seed, "v", L, B, Hkv, d, 0, self.n0, P, S.SINK_SIZE, self.dev, stream=self.main)
            for l in range(L):
                self.kv.load_prefix(l, K[l], V[l], self.n0, stream=self.main)
            self.main.synchronize()
            if keep_inputs:
                self.K0, self.V0 = K, V
            del K, V
            kn = SG.gen_kv(self.seed, "k", L, B, Hkv, d, self.n0, T, P, S.SINK_SIZE, self.dev, stream=self.main)
            vn = SG.gen_kv(self.seed, "v", L, B, Hkv, d, self.n0, T, P, S.SINK_SIZE, self.dev, stream=self.main)
            # [L][B][Hkv][T][d] -> [T][L][B][Hkv][d] (per-step append rows)
            self.Kn = kn.permute(3, 0, 1, 2, 4).contiguous()
            self.Vn = vn.permute(3, 0, 1, 2, 4).contiguous()
            del kn, vn
            self.Q = SG.gen_q(self.seed, 0, T, L, B, Hq, Hkv, d, self.dev, stream=self.main)
            odt = torch.float32 if out_fp32 else torch.bfloat16
            self.O = torch.empty((L, B, Hq, d), dtype=odt, device=self.dev)
            # fixed buffers for the captured step graph
            self.qbuf = torch.empty_like(self.Q[0])
            self.kbuf = torch.empty_like(self.Kn[0])
            self.vbuf = torch.empty_like(self.Vn[0])
        self.main.synchronize()
        self.t = 0
        self.graph = False

    # ---------------------------------------------------------------- steps
    def capture(self):
        with torch.cuda.stream(self.main):
            self.kv.step_graph_capture(self.qbuf, self.kbuf, self.vbuf, self.O, 1, stream=self.main, side=self.side)
        self.graph = True

    def is_event(self, t):
        return t % self.w["interval"] == 0

    def output(self):
        """Host copy of the last step's o [L][B][Hq][d] (waits for the main stream)."""
        self.main.synchronize()
        return self.O.cpu().numpy()

    def step(self):
        """One decode step t (+ manage event when t mod Delta == 0).  Asynchronous on
        self.main: read results through output()."""
        t = self.t
        with torch.cuda.stream(self.main):
            if self.graph:
                self.qbuf.copy_(self.Q[t], non_blocking=True)
                self.kbuf.copy_(self.Kn[t], non_blocking=True)
                self.vbuf.copy_(self.Vn[t], non_blocking=True)
                self.kv.step_graph_launch(stream=self.main)
            else:
                self.kv.step(self.Q[t], self.Kn[t], self.Vn[t], self.O, 1, stream=self.main, side=self.side)
            if self.is_event(t):
                self.kv.classify(stream=self.main)
                self.kv.migrate(stream=self.main, side=self.side)
        self.t += 1
        return self.O

    def step_layers(self):
        """Same step through the per-layer ABI calls (append / prefetch / decode_attention)."""
        t = self.t
        L = self.w["L"]
        stream_mode = self.w["staging"] == 0
        with torch.cuda.stream(self.main):
            self.kv.begin_step(stream=self.main)
            if stream_mode:
                for l in range(min(2, L)):
                    self.kv.prefetch(l, side=self.side)
            for l in range(L):
                self.kv.append(l, self.Kn[t, l], self.Vn[t, l], stream=self.main)
                self.kv.decode_attention(l, self.Q[t, l], self.O[l], 1, stream=self.main)
                if stream_mode and l + 2 < L:
                    self.kv.prefetch(l + 2, side=self.side)
            self.kv.end_step(stream=self.main)
            if self.is_event(t):
                self.kv.classify(stream=self.main)
                self.kv.migrate(stream=self.main, side=self.side)
        self.t += 1
        return self.O

    def sync(self):
        self.main.synchronize()
        self.side.synchronize()
        self.kv.sync()

    def close(self):
        self.sync()
        self.kv.close()
