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

    def __init__(self, w, device="cuda:0", out_fp32=True, split=0, seed_offset=0, keep_inputs=False, variant=0,
                 heads=None, classify_fn=None, shard=kt.SHARD_REQUEST, rank=0, world=1, nccl_id=None,
                 step_kernel=0, prefix_fn=None):
        """heads = (first kv head, count): this ctx holds only those kv heads and their q
        heads (KV-head sharding); classify_fn(run, stream) replaces kv.classify at events
        (e.g. dist.kvhead_classify, or a single-process gather over several ctxs); nccl_id:
        sequence sharding on the library's own communicator (kv_tier_step / the step graph
        run the per-layer exchange, kv_tier_classify the event's all-gather); prefix_fn(l) ->
        (K, V) [B][H_kv][N-1][d] bf16 on the device: the prefix of layer l from a prefill (called
        in layer order) instead of the synthetic generator."""
        self.w = w
        self.dev = torch.device(device)
        torch.cuda.set_device(self.dev)
        B, L, Hq, Hkv, d, N, P, T = (w[k] for k in ("B", "L", "Hq", "Hkv", "d", "N", "P", "steps"))
        G = Hq // Hkv
        h0, hl = heads if heads is not None else (0, Hkv)
        self.heads = (h0, hl)
        self.classify_fn = classify_fn
        self.seed = w["seed"] + seed_offset
        self.n0 = N - 1
        self.T = T
        self.cfg = kt.make_config(B, L, hl * G, hl, d, self.n0 + T, P, hbm_bp=w["hbm_bp"], evict_bp=w["evict_bp"],
                                  t2_bp=w["t2_bp"], manage_interval=w["interval"], evict_mode=w["evict_mode"],
                                  staging=w["staging"], device=self.dev.index or 0, out_fp32=int(out_fp32),
                                  split=split, variant=variant, shard=shard, rank=rank, world=world,
                                  policy=w.get("policy", 0), budget=w.get("budget", 0),
                                  policy_seed=w.get("policy_seed", 0), scorer=w.get("scorer", 0),
                                  step_kernel=step_kernel)
        hs = slice(h0, h0 + hl)
        qs = slice(h0 * G, (h0 + hl) * G)
        self.kv = kt.KvTier(self.cfg, nccl_id=nccl_id)
        self.main = torch.cuda.Stream(self.dev)
        self.side = torch.cuda.Stream(self.dev)
        with torch.cuda.stream(self.main):
            if prefix_fn is not None:        # Alg. 1 line 1: C <- Prefill(M, x_1:P), layer by layer
                assert heads is None and not keep_inputs
                for l in range(L):
                    Kl, Vl = prefix_fn(l)
                    self.kv.load_prefix(l, Kl, Vl, self.n0, stream=self.main)
                    self.main.synchronize()
                    del Kl, Vl
            elif keep_inputs:
                K = SG.gen_kv(self.seed, "k", L, B, Hkv, d, 0, self.n0, P, S.SINK_SIZE, self.dev, stream=self.main)
                V = SG.gen_kv(self.seed, "v", L, B, Hkv, d, 0, self.n0, P, S.SINK_SIZE, self.dev, stream=self.main)
                if heads is not None:
                    K, V = K[:, :, hs].contiguous(), V[:, :, hs].contiguous()
                for l in range(L):
                    self.kv.load_prefix(l, K[l], V[l], self.n0, stream=self.main)
                self.K0, self.V0 = K, V
            else:                       # one layer at a time: the full prefix of a large config never sits in HBM
                for l in range(L):
                    Kl = SG.gen_kv_layer(self.seed, "k", l, B, Hkv, d, 0, self.n0, P, S.SINK_SIZE, self.dev,
                                         stream=self.main)
                    Vl = SG.gen_kv_layer(self.seed, "v", l, B, Hkv, d, 0, self.n0, P, S.SINK_SIZE, self.dev,
                                         stream=self.main)
                    if heads is not None:
                        Kl, Vl = Kl[:, hs].contiguous(), Vl[:, hs].contiguous()
                    self.kv.load_prefix(l, Kl, Vl, self.n0, stream=self.main)
                    self.main.synchronize()     # the layer's buffers are freed before the next is drawn
                    del Kl, Vl
            self.main.synchronize()
            kn = SG.gen_kv(self.seed, "k", L, B, Hkv, d, self.n0, T, P, S.SINK_SIZE, self.dev, stream=self.main)
            vn = SG.gen_kv(self.seed, "v", L, B, Hkv, d, self.n0, T, P, S.SINK_SIZE, self.dev, stream=self.main)
            # [L][B][Hkv][T][d] -> [T][L][B][Hkv][d] (per-step append rows)
            self.Kn = kn[:, :, hs].permute(3, 0, 1, 2, 4).contiguous()
            self.Vn = vn[:, :, hs].permute(3, 0, 1, 2, 4).contiguous()
            del kn, vn
            self.Q = SG.gen_q(self.seed, 0, T, L, B, Hq, Hkv, d, self.dev, stream=self.main)[:, :, :, qs].contiguous()
            odt = torch.float32 if out_fp32 else torch.bfloat16
            self.O = torch.empty((L, B, hl * G, d), dtype=odt, device=self.dev)
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
        """Host copy of the last step's o [L][B][Hq][d] as fp32 (waits for the main stream)."""
        self.main.synchronize()
        return self.O.float().cpu().numpy()

    def step(self, manage=True):
        """One decode step t (+ manage event when t mod Delta == 0 unless manage=False).
        Asynchronous on self.main: read results through output()."""
        t = self.t
        with torch.cuda.stream(self.main):
            if self.graph:
                torch._foreach_copy_([self.qbuf, self.kbuf, self.vbuf], [self.Q[t], self.Kn[t], self.Vn[t]],
                                     non_blocking=True)          # one multi-tensor copy launch
                self.kv.step_graph_launch(stream=self.main)
            else:
                self.kv.step(self.Q[t], self.Kn[t], self.Vn[t], self.O, 1, stream=self.main, side=self.side)
            if manage and self.is_event(t):
                self.classify()
                self.kv.migrate(stream=self.main, side=self.side)
        self.t += 1
        return self.O

    def classify(self):
        if self.classify_fn is not None:
            self.classify_fn(self, self.main)
        else:
            self.kv.classify(stream=self.main)

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
                self.classify()
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


class ModelDecode:
    """the tiered attention inside a decoder of the 7B model's shape
    (Qwen2-7B dims) with random bf16 weights, so the path runs with its real
    per-layer dependency: q/k/v come from this layer's projections of the previous layer's
    output, and the T1 prefetch of layer l+2 (stream mode) overlaps layer l's MLP.
    Non-attention layers are plain torch/cuBLAS (RMSNorm, GEMMs, SiLU; no RoPE, no LM head):
    they are the context, not the product.  The prefix K/V are the synthetic generator's, or with
    prefill=True the model's own: Alg. 1 line 1, C <- Prefill(M, x_1:P) -- a causal
    forward (torch SDPA, GQA) over N-1 random prompt embeddings, each layer's K/V loaded as that
    layer's prefix, and the last prompt position's output is the first decode input."""

    def __init__(self, w, hidden=3584, inter=18944, device="cuda:0", prefill=False, keep_prefill=False, **kw):
        import math
        self.w, self.hidden, self.inter = w, hidden, inter
        B, L, Hq, Hkv, d = w["B"], w["L"], w["Hq"], w["Hkv"], w["d"]
        dev = torch.device(device)
        torch.cuda.set_device(dev)
        g = torch.Generator(device=dev).manual_seed(w["seed"] + 17)

        def W(i, o):
            return (torch.randn(i, o, generator=g, device=dev) / math.sqrt(i)).to(torch.bfloat16)

        self.layers = [dict(wqkv=W(hidden, (Hq + 2 * Hkv) * d), wo=W(Hq * d, hidden), wgu=W(hidden, 2 * inter),
                            wd=W(inter, hidden)) for _ in range(L)]
        self.x = torch.randn(B, hidden, generator=g, device=dev).to(torch.bfloat16)
        self.prefill_kv = [] if keep_prefill else None
        if prefill:
            self._H = torch.randn(B, w["N"] - 1, hidden, generator=g, device=dev).to(torch.bfloat16)
            torch.cuda.synchronize(dev)              # weights and prompt drawn on torch's stream
            self.run = TieredDecode(w, device=device, out_fp32=False, prefix_fn=self._prefill_layer, **kw)
            self.x = self._rms(self._H[:, -1])
            self._H = None
        else:
            self.run = TieredDecode(w, device=device, out_fp32=False, **kw)
        self.O = torch.empty((B, Hq, d), dtype=torch.bfloat16, device=dev)
        # the weights were drawn on torch's current stream; the steps run on the ctx's main
        # stream (non-blocking w.r.t. it): order them
        self.run.main.wait_stream(torch.cuda.current_stream(dev))

    def _prefill_layer(self, l):
        """Layer l of the prefill over the prompt's hidden states (causal attention over the
        prompt); returns the layer's K, V [B][H_kv][n][d] and advances the hidden states."""
        w, p, Hs = self.w, self.layers[l], self._H
        B, n = Hs.shape[0], Hs.shape[1]
        Hq, Hkv, d = w["Hq"], w["Hkv"], w["d"]
        qkv = self._rms(Hs) @ p["wqkv"]
        q = qkv[..., :Hq * d].reshape(B, n, Hq, d).transpose(1, 2)
        k = qkv[..., Hq * d:(Hq + Hkv) * d].reshape(B, n, Hkv, d).transpose(1, 2).contiguous()
        v = qkv[..., (Hq + Hkv) * d:].reshape(B, n, Hkv, d).transpose(1, 2).contiguous()
        a = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        Hs = Hs + a.transpose(1, 2).reshape(B, n, Hq * d) @ p["wo"]
        gu = self._rms(Hs) @ p["wgu"]
        self._H = Hs + (torch.nn.functional.silu(gu[..., :self.inter]) * gu[..., self.inter:]) @ p["wd"]
        if self.prefill_kv is not None:
            self.prefill_kv.append((k.clone(), v.clone()))
        return k, v

    @staticmethod
    def _rms(x):
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-6)).to(torch.bfloat16)

    def capture(self):
        """The whole decoder step -- RMSNorm, GEMMs, the library's begin_step / prefetch /
        decode_attention per layer / end_step -- as ONE CUDA graph (torch.cuda.graph around the
        library's kv_tier_capture_begin / _end); step() then replays it and advances the
        library's host state (kv_tier_graph_advance).  Manage events stay eager between replays."""
        r = self.run
        self.xin = self.x.clone()
        torch.cuda.synchronize(self.run.dev)
        self.graph = torch.cuda.CUDAGraph()
        r.kv.capture_begin()
        try:
            with torch.cuda.graph(self.graph, stream=r.main):
                self.xout = self._body(self.xin)
        finally:
            r.kv.capture_end()

    def _body(self, x):
        r, w = self.run, self.w
        kv, s = r.kv, torch.cuda.current_stream(r.dev)
        B, L, Hq, Hkv, d = w["B"], w["L"], w["Hq"], w["Hkv"], w["d"]
        stream_mode = w["staging"] == 0
        kv.begin_step(stream=s)
        if stream_mode:
            for l in range(min(2, L)):
                kv.prefetch(l, side=r.side)
        for l, p in enumerate(self.layers):
            qkv = self._rms(x) @ p["wqkv"]
            q = qkv[:, :Hq * d].reshape(B, Hq, d).contiguous()
            k = qkv[:, Hq * d:(Hq + Hkv) * d].reshape(B, Hkv, d).contiguous()
            v = qkv[:, (Hq + Hkv) * d:].reshape(B, Hkv, d).contiguous()
            kv.decode_attention(l, q, self.O, 1, stream=s, k_new=k, v_new=v)
            if stream_mode and l + 2 < L:
                kv.prefetch(l + 2, side=r.side)
            x = x + self.O.reshape(B, Hq * d) @ p["wo"]
            gu = self._rms(x) @ p["wgu"]
            x = x + (torch.nn.functional.silu(gu[:, :self.inter]) * gu[:, self.inter:]) @ p["wd"]
        kv.end_step(stream=s)
        return self._rms(x)

    def step(self):
        r, w = self.run, self.w
        kv, s, t = r.kv, r.main, r.t
        if getattr(self, "graph", None) is not None:
            with torch.cuda.stream(s):
                self.xin.copy_(self.x)
                self.graph.replay()
                kv.graph_advance()
                if r.is_event(t):
                    r.classify()
                    kv.migrate(stream=s, side=r.side)
                self.x = self.xout.clone()
            r.t += 1
            torch.cuda.current_stream(r.dev).wait_stream(s)   # the caller reads x on its own stream
            return self.x
        B, L, Hq, Hkv, d = w["B"], w["L"], w["Hq"], w["Hkv"], w["d"]
        stream_mode = w["staging"] == 0
        with torch.cuda.stream(s):
            kv.begin_step(stream=s)
            if stream_mode:
                for l in range(min(2, L)):
                    kv.prefetch(l, side=r.side)
            x = self.x
            for l, p in enumerate(self.layers):
                qkv = self._rms(x) @ p["wqkv"]
                q = qkv[:, :Hq * d].reshape(B, Hq, d).contiguous()
                k = qkv[:, Hq * d:(Hq + Hkv) * d].reshape(B, Hkv, d).contiguous()
                v = qkv[:, (Hq + Hkv) * d:].reshape(B, Hkv, d).contiguous()
                kv.decode_attention(l, q, self.O, 1, stream=s, k_new=k, v_new=v)
                if stream_mode and l + 2 < L:
                    kv.prefetch(l + 2, side=r.side)
                x = x + self.O.reshape(B, Hq * d) @ p["wo"]
                gu = self._rms(x) @ p["wgu"]
                x = x + (torch.nn.functional.silu(gu[:, :self.inter]) * gu[:, self.inter:]) @ p["wd"]
            kv.end_step(stream=s)
            if r.is_event(t):
                r.classify()
                kv.migrate(stream=s, side=r.side)
            self.x = self._rms(x)
        r.t += 1
        torch.cuda.current_stream(r.dev).wait_stream(s)       # the caller reads x on its own stream
        return self.x

    def sync(self):
        self.run.sync()

    def close(self):
        self.run.close()
        self.layers = None


class KvHeadShardedDecode:
    """KV-head sharding simulated in one process: `world` ctxs on one
    device, ctx r holding kv heads [r*H_l, (r+1)*H_l).  At an event the ctxs' S_part are
    gathered in rank order (the bytes an NCCL all-gather moves) and every ctx classifies the
    same gathered scores.  Outputs are concatenated over q heads."""

    def __init__(self, w, world, device="cuda:0", **kw):
        Hkv = w["Hkv"]
        assert Hkv % world == 0
        hl = Hkv // world
        self.world = world
        self.runs = []
        for r in range(world):
            self.runs.append(TieredDecode(w, device=device, heads=(r * hl, hl), shard=kt.SHARD_KVHEAD,
                                          rank=r, world=world, **kw))
        self.w = w

    def is_event(self, t):
        return t % self.w["interval"] == 0

    @property
    def t(self):
        return self.runs[0].t

    def capture(self):
        for r in self.runs:
            r.capture()

    def step(self):
        t = self.t
        for r in self.runs:
            r.step(manage=False)
        if self.is_event(t):
            for r in self.runs:
                r.main.synchronize()
            gathered = torch.stack([r.kv.scores_tensor() for r in self.runs]).contiguous()   # the all-gather
            torch.cuda.current_stream(self.runs[0].dev).synchronize()
            for r in self.runs:
                with torch.cuda.stream(r.main):
                    r.kv.classify_gathered(gathered, self.world, stream=r.main)
                    r.kv.migrate(stream=r.main, side=r.side)
            for r in self.runs:
                r.main.synchronize()

    def output(self):
        import numpy as np
        return np.concatenate([r.output() for r in self.runs], axis=2)

    def scores(self):
        import numpy as np
        for r in self.runs:
            r.sync()
        return np.concatenate([r.kv.export(kt.X_SCORES) for r in self.runs], axis=1)

    def sync(self):
        for r in self.runs:
            r.sync()

    def close(self):
        for r in self.runs:
            r.close()


class HostT1Decode:
    """T1 attended on the host cores where it lives (kv_tier_set_host_t1).
    Per layer: q goes down (D2H), the GPU attends T0 ∪ T2 ∪ {new} (decode_attention_lse) while
    the host attends T1 (host_t1_attention, OpenMP), the two partials are combined on the GPU
    (lse_combine, Eq. 3 split by tier), and the score update runs for the GPU's tokens
    (score_update_lse) and for T1 on the host (host_t1_score_update) with the global (M, L)."""

    def __init__(self, w, device="cuda:0", fused=True, **kw):
        """fused: one kv_tier_host_t1_layer call per layer (the library sequences the copies,
        the host loop and both score updates); else the same sequence from Python."""
        self.w, self.fused = w, fused
        self.run = TieredDecode(w, device=device, out_fp32=True, **kw)
        self.run.kv.set_host_t1(True)
        B, L, Hq, d = w["B"], w["L"], w["Hq"], w["d"]
        dev = self.run.dev
        self.parts_o = torch.empty((2, B, Hq, d), dtype=torch.float32, device=dev)
        self.parts_l = torch.empty((2, B, Hq, 2), dtype=torch.float32, device=dev)
        self.q_host = torch.empty((B, Hq, d), dtype=torch.bfloat16).pin_memory()
        self.o_host = torch.empty((B, Hq, d), dtype=torch.float32).pin_memory()
        self.l_host = torch.empty((B, Hq, 2), dtype=torch.float32).pin_memory()
        self.lse_host = torch.empty((L, B, Hq, 2), dtype=torch.float32).pin_memory()
        self.O = torch.empty((L, B, Hq, d), dtype=torch.float32, device=dev)
        self.LSE = torch.empty((L, B, Hq, 2), dtype=torch.float32, device=dev)
        self.t = 0

    def is_event(self, t):
        return t % self.w["interval"] == 0

    def step(self, q=None):
        """One decode step; q: optional [L][B][H_q][d] bf16 (default: the generated queries)."""
        r, t = self.run, self.t
        kv, s = r.kv, r.main
        Q = r.Q[t] if q is None else q
        with torch.cuda.stream(s):
            kv.begin_step(stream=s)
            for l in range(self.w["L"]):
                if self.fused:
                    kv.host_t1_layer(l, Q[l], self.O[l], stream=s, k_new=r.Kn[t, l], v_new=r.Vn[t, l])
                    continue
                self.q_host.copy_(Q[l], non_blocking=True)                  # q down
                q_ready = torch.cuda.Event()
                q_ready.record(s)
                kv.decode_attention_lse(l, Q[l], self.parts_o[0], self.parts_l[0], 1, stream=s,
                                        k_new=r.Kn[t, l], v_new=r.Vn[t, l])
                q_ready.synchronize()
                kv.host_t1_attention(l, self.q_host, self.o_host, self.l_host)   # overlaps the GPU partial
                self.parts_o[1].copy_(self.o_host, non_blocking=True)            # (o, m, l) up
                self.parts_l[1].copy_(self.l_host, non_blocking=True)
                o, lse = kt.lse_combine(self.parts_o, self.parts_l)
                self.O[l].copy_(o)
                self.LSE[l].copy_(lse)
                kv.score_update_lse(self.LSE[l], stream=s)
                self.lse_host[l].copy_(self.LSE[l], non_blocking=True)
                done = torch.cuda.Event()
                done.record(s)
                done.synchronize()
                kv.host_t1_score_update(l, self.lse_host[l], stream=s)
            kv.end_step(stream=s)
            if self.is_event(t):
                kv.classify(stream=s)
                kv.migrate(stream=s, side=r.side)
        self.t += 1
        r.t = self.t
        return self.O

    def output(self):
        self.run.main.synchronize()
        return self.O.cpu().numpy()

    def sync(self):
        self.run.sync()

    def close(self):
        self.run.close()


class SeqShardedDecode:
    """Sequence sharding simulated in one process: `world` ctxs on one
    device, ctx r owning the 64-position blocks k with k % world == r.  Every layer: each ctx
    attends its own tokens (decode_attention_lse), the partials are combined in rank order
    (dist.lse_combine -- the bytes an NCCL all-gather moves), and each ctx finishes its
    score update with the global (M, L).  Events: summed S_part -> classify_gathered."""

    def __init__(self, w, world, device="cuda:0", out_fp32=True, **kw):
        self.w, self.world = w, world
        self.runs = [TieredDecode(w, device=device, out_fp32=out_fp32, shard=kt.SHARD_SEQUENCE, rank=r,
                                  world=world, **kw) for r in range(world)]
        r0 = self.runs[0]
        self.dev = r0.dev
        self.stream = r0.main
        B, L, Hq, d = w["B"], w["L"], w["Hq"], w["d"]
        self.Ol = [torch.empty((L, B, Hq, d), dtype=torch.float32, device=self.dev) for _ in range(world)]
        self.LSE = [torch.empty((L, B, Hq, 2), dtype=torch.float32, device=self.dev) for _ in range(world)]
        self.O = torch.empty((L, B, Hq, d), dtype=torch.float32, device=self.dev)
        self.LSEg = torch.empty((L, B, Hq, 2), dtype=torch.float32, device=self.dev)
        self.t = 0

    def is_event(self, t):
        return t % self.w["interval"] == 0

    def step(self):
        from . import dist as D
        t, s = self.t, self.stream
        r0 = self.runs[0]
        stream_mode = self.w["staging"] == 0
        L = self.w["L"]
        with torch.cuda.stream(s):
            for r in self.runs:
                r.kv.begin_step(stream=s)
                if stream_mode:                      # T1 rows of the first layers, layer-ahead
                    for l in range(min(2, L)):
                        r.kv.prefetch(l, side=r.side)
            for l in range(L):
                for i, r in enumerate(self.runs):
                    r.kv.decode_attention_lse(l, r0.Q[t, l], self.Ol[i][l], self.LSE[i][l], 1, stream=s,
                                              k_new=r0.Kn[t, l], v_new=r0.Vn[t, l])
                    if stream_mode and l + 2 < L:
                        r.kv.prefetch(l + 2, side=r.side)
                o, lse = D.lse_combine(torch.stack([x[l] for x in self.Ol]), torch.stack([x[l] for x in self.LSE]))
                self.O[l].copy_(o)
                self.LSEg[l].copy_(lse)
                for r in self.runs:
                    r.kv.score_update_lse(self.LSEg[l], stream=s)
            for r in self.runs:
                r.kv.end_step(stream=s)
            if self.is_event(t):
                S_all = torch.stack([r.kv.scores_tensor() for r in self.runs]).contiguous()   # the all-gather
                for r in self.runs:
                    r.kv.classify_gathered(S_all, self.world, stream=s)
                    r.kv.migrate(stream=s, side=r.side)
                s.synchronize()
        self.t += 1
        for r in self.runs:
            r.t = self.t
        return self.O

    def output(self):
        self.stream.synchronize()
        return self.O.cpu().numpy()

    def scores(self):
        """Summed S_part [B][H_kv][n] (every position has exactly one owner)."""
        import numpy as np
        self.sync()
        return np.sum([r.kv.export(kt.X_SCORES) for r in self.runs], axis=0)

    def sync(self):
        self.stream.synchronize()
        for r in self.runs:
            r.sync()

    def close(self):
        for r in self.runs:
            r.close()


class SeqShardRank:
    """One rank of a sequence-sharded decode in its own process: the ctx
    owns the 64-position blocks k with k % world == rank; every layer the ranks all-gather
    (o, m, l) over the process group (NCCL, or gloo staged through host memory) and combine
    them in rank order; events classify the all-gathered scores.  Every rank ends each step
    with the full o of all layers."""

    def __init__(self, w, rank, world, device="cuda:0", group=None, **kw):
        self.w, self.rank, self.world, self.group = w, rank, world, group
        self.run = TieredDecode(w, device=device, out_fp32=True, shard=kt.SHARD_SEQUENCE, rank=rank, world=world, **kw)
        B, L, Hq, d = w["B"], w["L"], w["Hq"], w["d"]
        dev = self.run.dev
        self.Ol = torch.empty((L, B, Hq, d), dtype=torch.float32, device=dev)
        self.LSE = torch.empty((L, B, Hq, 2), dtype=torch.float32, device=dev)
        self.O = torch.empty((L, B, Hq, d), dtype=torch.float32, device=dev)
        self.LSEg = torch.empty((L, B, Hq, 2), dtype=torch.float32, device=dev)
        self.t = 0

    def is_event(self, t):
        return t % self.w["interval"] == 0

    def step(self):
        from . import dist as D
        r, t = self.run, self.t
        s = r.main
        stream_mode = self.w["staging"] == 0
        L = self.w["L"]
        with torch.cuda.stream(s):
            r.kv.begin_step(stream=s)
            if stream_mode:                          # T1 rows of the first layers, layer-ahead
                for l in range(min(2, L)):
                    r.kv.prefetch(l, side=r.side)
            for l in range(L):
                r.kv.decode_attention_lse(l, r.Q[t, l], self.Ol[l], self.LSE[l], 1, stream=s,
                                          k_new=r.Kn[t, l], v_new=r.Vn[t, l])
                if stream_mode and l + 2 < L:
                    r.kv.prefetch(l + 2, side=r.side)
                o, lse = D.seq_combine(self.Ol[l], self.LSE[l], self.group)
                self.O[l].copy_(o)
                self.LSEg[l].copy_(lse)
                r.kv.score_update_lse(self.LSEg[l], stream=s)
            r.kv.end_step(stream=s)
            if self.is_event(t):
                D.seq_classify(r.kv, stream=s, group=self.group)
                r.kv.migrate(stream=s, side=r.side)
        self.t += 1
        r.t = self.t
        return self.O

    def output(self):
        self.run.main.synchronize()
        return self.O.cpu().numpy()

    def scores(self):
        """Summed S_part over the ranks [B][H_kv][n] (exact: one owner per position)."""
        from . import dist as D
        self.run.sync()
        S = torch.from_numpy(self.run.kv.export(kt.X_SCORES).copy())
        return D.gather_scores(S, self.group).sum(dim=0).numpy()

    def close(self):
        self.run.close()
