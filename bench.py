#!/usr/bin/env python
"""Benchmark of the tiered-KV decode hot path (BASELINE.json metric):
tiered decode steps/s, HBM GB/s vs roofline, T1 prefetch overhead % of step time.

A step = one decode step of the whole path over one batch: the new token of every layer is
appended (a1), T1 is readable from HBM staging (a2, differential mode, paper §3.4), GQA decode
attention + the fused cumulative score update for every layer (a3 + a4), and every Delta = 64
steps classify + migrate (a5 + a6).  Default workload: BASELINE.json configs[1], 7B-shaped,
beta 50 % / r 5 %, differential staging.  Inputs are synthetic (synth.py recipe); the per-step
K/V traffic (~0.9 GB) exceeds the 126 MB L2, so no L2 flush is needed between steps.

Headline `value`: steps/s with the manage event amortised at its natural rate, 1 / (t_step +
t_event / Delta), both MEASURED in this run (t_step over the timed window's event-free steps,
t_event = the mean classify + migrate time, CUDA events on the launching stream).  The raw window
rate K / elapsed is reported beside it with the number of events the window happened to contain.

    python bench.py [--gpus N --steps K --warmup W]          # our CUDA path (N > 1 spawns N ranks)
    python bench.py --impl reference ...                      # the CPU oracle (reference arm)
Multi-GPU: one process per GPU, requests sharded across ranks (weak scaling, no collective in
the step), time = max over ranks.  `--shard sequence`: one batch's positions split over the ranks.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "src": "fallback (B200_PROFILING.md)"}
STEP_KERNELS = {"auto": 0, "mma": 1, "tcgen05": 2, "layers": 3}                      # kv_tier_config::step_kernel
CONFIG_INDEX = {"tiny": 0, "7b": 1, "14b": 2, "32b": 3, "70b": 4}      # BASELINE.json configs[i]
POLICIES = {"hierarchy": 0, "streaming": 1, "h2o": 2, "random": 3}       # kv_tier_policy
SCORERS = {"attention": 0, "vatp": 1, "redundancy": 2, "combined": 3, "window": 4, "rkv": 5}   # kv_tier_scorer
MODEL_DIMS = {"tiny": (256, 512), "7b": (3584, 18944)}                    # (hidden, intermediate): Qwen2-7B
EVENT_LAUNCHES = 5          # classify, plan, cooperative migrate, commit, offload (side stream)


def _metric():
    """The BASELINE.json metric string, shared by both arms (the driver pairs them by it)."""
    try:
        with open(os.path.join(ROOT, "BASELINE.json")) as f:
            return json.load(f)["metric"]
    except Exception:
        return "tiered decode steps/sec & HBM GB/s vs roofline; T1 prefetch overhead % of step time"


METRIC = _metric()


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured (MEASURED_PEAKS.json)"}
    return PEAKS_FALLBACK


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=192)
    ap.add_argument("--warmup", type=int, default=64)
    ap.add_argument("--impl", default="kvtier", choices=["kvtier", "reference"])
    ap.add_argument("--config", default="7b")
    ap.add_argument("--hbm", type=int, default=5000, help="beta in basis points")
    ap.add_argument("--evict", type=int, default=500, help="r in basis points")
    ap.add_argument("--split", type=int, default=0)
    ap.add_argument("--batch", type=int, default=0,
                    help="requests per GPU (0: the config's B); e.g. 16 = the 32B config's share on 2 GPUs")
    ap.add_argument("--policy", default="hierarchy", choices=list(POLICIES),
                    help="tier policy: the paper's hierarchy or a pure-eviction baseline (P:276-280)")
    ap.add_argument("--budget", type=int, default=1024, help="kept tokens per request (h2o / random)")
    ap.add_argument("--shard", default="request", choices=["request", "sequence"],
                    help="N>1 partitioning: requests per rank (weak scaling, default) or one batch's "
                         "positions split over the ranks with a per-layer LSE combine (strong scaling)")
    ap.add_argument("--scorer", default="attention", choices=list(SCORERS),
                    help="token scorer: Eq. 1 attention, VATP (P:712), redundancy (P:713), combined (P:714), "
                         "windowed attention (P:137, P:976), R-KV's 0.07 I - 0.93 R (P:972-978)")
    ap.add_argument("--positions", type=int, default=0,
                    help="chain length N per request (0: the config's); e.g. --config 70b --positions 2048 = "
                         "the positions ONE rank of configs[4]'s 8-way sequence split attends")
    ap.add_argument("--step-kernel", default="auto", choices=list(STEP_KERNELS),
                    help="whole-step kernel consumer: auto (= mma), mma (mma.sync), tcgen05 (TMEM accumulators)")
    ap.add_argument("--no-extras", action="store_true", help="skip control/e2e/stream/N1/N4/cpu legs")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    return ap.parse_args()


class ClockSampler:
    """NVML clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index, self.samples, self.reasons, self._stop = index, [], set(), threading.Event()
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:           # no NVML: report it
            self.nv = None
            self.err = str(e)
        return self

    def _run(self):
        nv = self.nv
        names = {getattr(nv, k): k.replace("nvmlClocksThrottleReason", "").replace("nvmlClocksEventReason", "")
                 for k in dir(nv) if k.startswith(("nvmlClocksThrottleReason", "nvmlClocksEventReason"))
                 and isinstance(getattr(nv, k), int)}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in names.items():
                    if bit and (mask & bit) == bit and name not in ("None", "All", "GpuIdle"):
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join(timeout=1)

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "err", "")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ byte accounting
def attn_bytes(w, counts, n_vis, out_bytes=2):
    """Algorithmic HBM bytes of one layer of a3 + a4: every visible K/V row once
    (4*d B per bf16 token per kv head; 2*(d+4) B per int8 T2 token), q and o, and the 8 B fp32
    read + write of the score per visible token per kv head."""
    B, Hq, Hkv, d = w["B"], w["Hq"], w["Hkv"], w["d"]
    n01, n2 = counts[0] + counts[1], counts[2]
    kv = B * Hkv * (n01 * 4 * d + n2 * 2 * (d + 4))
    return kv + B * Hq * d * (2 + out_bytes) + 8 * B * Hkv * n_vis


def host_link_peak_gbs(nbytes=256 << 20, reps=10):
    """Measured pinned host -> device copy bandwidth of this box (the stream-mode roofline)."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    d.copy_(h)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            d.copy_(h, non_blocking=True)
            b.record(s)
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
    del h, d
    return best


def timed(fn, stream, n):
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / 1e3


def _max_over_ranks(x):
    from paper_2605_09490_b200.dist import max_over_ranks
    return max_over_ranks(x)


def _sum_over_ranks(x):
    from paper_2605_09490_b200.dist import sum_over_ranks
    return sum_over_ranks(x)


def _barrier_sync():
    from paper_2605_09490_b200.dist import barrier_sync
    barrier_sync()


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


# ------------------------------------------------------------------ CPU oracle leg
def cpu_oracle_sample(w, budget_s, threads=None):
    """Time the CPU oracle (as it stands) on 1 request of the workload, all layers, decode steps
    from t = 0 (the first includes the t = 0 manage event) until budget_s; returns full-batch
    steps/s (per-request time x B requests).  threads: BLAS threads (None = all cores)."""
    import contextlib
    from tests.oracle_runner import OracleRun
    from threadpoolctl import threadpool_limits, threadpool_info
    with (threadpool_limits(limits=threads) if threads else contextlib.nullcontext()):
        used = threads or max([p.get("num_threads", 1) for p in threadpool_info()] or [1])
        orc = OracleRun(dict(w, steps=64), reqs=[0])
        t0 = time.perf_counter()
        k = 0
        while k < 64 and (k == 0 or time.perf_counter() - t0 < budget_s):
            orc.step()
            k += 1
        el = time.perf_counter() - t0
    return {"value": 1.0 / (el / k * w["B"]), "unit": "steps/s", "cores": int(used), "kind": "oracle",
            "steps_run": k, "requests_run": 1,
            "sample": f"1 of {w['B']} requests x {w['L']} layers x {k} decode steps from t=0 (t=0 event incl.), "
                      f"{el:.1f} s; per-request time x {w['B']} requests = one full-batch step"}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (rank 0 only; other ranks exit 0)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from paper_2605_09490_b200.synth import synth as S
    w = dict(S.WORKLOADS[args.config], hbm_bp=args.hbm, evict_bp=args.evict, interval=64, t2_bp=0, evict_mode=0)
    budget = max(5.0, min(60.0, args.cpu_seconds * (args.steps + args.warmup) / 256))
    cb = cpu_oracle_sample(w, budget)
    val = cb["value"]
    cb["cpu_model"] = _cpu_model()
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val,
        "unit": "steps/s", "n_gpus": args.gpus, "steps": cb["steps_run"], "warmup": 0,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": 1e3 / val, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}-shaped (BASELINE.json configs[{CONFIG_INDEX.get(args.config, '?')}]) "
                               f"B={w['B']} L={w['L']} Hq/Hkv={w['Hq']}/{w['Hkv']} d={w['d']} N={w['N']} "
                               f"beta={args.hbm}bp r={args.evict}bp Delta=64"},
        "cpu_baseline": cb,
        "e2e": {"value": val, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the CPU oracle (numpy fp64, tests/ infrastructure) on this box's host cores: one request of "
                "the batch for as many steps as the budget allows, scaled to the full batch",
    }), flush=True)


# ------------------------------------------------------------------ GPU legs
def _event_step(run, timing):
    """One step through the captured step graph; at a manage event, classify + migrate with CUDA
    events around them (timing: list collecting the event's device time in s)."""
    import torch
    t = run.t
    with torch.cuda.stream(run.main):
        # the step's inputs into the graph's fixed buffers: one multi-tensor copy launch
        torch._foreach_copy_([run.qbuf, run.kbuf, run.vbuf], [run.Q[t], run.Kn[t], run.Vn[t]], non_blocking=True)
        run.kv.step_graph_launch(stream=run.main)
        if run.is_event(t):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(run.main)
            run.classify()
            run.kv.migrate(stream=run.main, side=run.side)
            b.record(run.main)
            timing.append((a, b))
    run.t += 1


def measure_tiered(run, W, K, w, local, with_clocks=True):
    """Warm up W steps, time K steps; returns the step/event split and the per-step bytes."""
    import torch
    L, itv = w["L"], w["interval"]
    scratch = []
    for _ in range(W):
        _event_step(run, scratch)
    run.sync()
    ev_times, bytes_steps = [], []
    n_events = 0
    _barrier_sync()
    clk = ClockSampler(local) if with_clocks else None
    if clk:
        clk.__enter__()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(run.main)
    for _ in range(K):
        counts, _ = run.kv.layout()                       # host mirror: the layout this step reads
        n_vis = sum(counts[:3]) + 1
        bytes_steps.append(L * attn_bytes(w, counts, n_vis))
        n_events += 1 if run.is_event(run.t) else 0
        _event_step(run, ev_times)
    b.record(run.main)
    b.synchronize()
    if clk:
        clk.__exit__()
    el = a.elapsed_time(b) / 1e3
    t_ev = [x.elapsed_time(y) / 1e3 for x, y in ev_times]
    # the event cost when the window held none: step on to the next event and time it
    while not t_ev:
        extra = []
        _event_step(run, extra)
        run.sync()
        t_ev = [x.elapsed_time(y) / 1e3 for x, y in extra]
    t_event = statistics.mean(t_ev)
    t_step = (el - sum(x.elapsed_time(y) / 1e3 for x, y in ev_times)) / K     # event-free step
    return {"el": el, "t_step": t_step, "t_event": t_event, "n_events": n_events,
            "t_amortized": t_step + t_event / itv, "bytes_per_step": statistics.mean(bytes_steps),
            "clocks": clk.summary() if clk else None}


def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    world_env = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and world_env is None:            # spawn one rank per GPU on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000), *sys.argv]
        sys.exit(subprocess.call(cmd))
    world = int(world_env or "1")
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    import torch
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2605_09490_b200 import harness as H
    from paper_2605_09490_b200 import kvtier as kt

    W, K = args.warmup, args.steps
    E = 0 if args.no_extras else 64                    # e2e window: exactly one Delta (one event)
    pol = POLICIES[args.policy]
    over = {"B": args.batch} if args.batch else {}
    if args.positions:
        over["N"] = args.positions
    # steps the longest leg needs (+ the event chase after the window)
    w = H.workload(args.config, hbm_bp=args.hbm, evict_bp=args.evict, steps=W + K + E + 66, policy=pol, **over,
                   budget=args.budget if pol in (2, 3) else 0, policy_seed=7, scorer=SCORERS[args.scorer])
    dev = f"cuda:{local}"
    peaks = _peaks()
    if args.shard == "sequence":
        return run_sequence_sharded(args, w, world, rank, local, dev, peaks)
    from paper_2605_09490_b200.dist import shard_plan
    seed_off, _ = shard_plan(world, rank, 1)
    L, B, Hkv, d, itv = w["L"], w["B"], w["Hkv"], w["d"], w["interval"]

    # ---- headline: tiered step (whole-step kernel via the step graph), device-resident inputs
    run = H.TieredDecode(w, device=dev, out_fp32=False, split=args.split, seed_offset=seed_off,
                         step_kernel=STEP_KERNELS[args.step_kernel])
    run.capture()
    m = measure_tiered(run, W, K, w, local)
    t_amort = _max_over_ranks(m["t_amortized"])
    el_max = _max_over_ranks(m["el"])
    sps = world / t_amort
    step_bytes = m["bytes_per_step"]
    counts, shape = run.kv.layout()
    n_vis = sum(counts[:3])

    # ---- e2e: the same step through the public API, pinned host inputs/outputs, one Delta window
    e2e = None
    if E:
        qh = run.Q[run.t:run.t + E].cpu().pin_memory()
        kh = run.Kn[run.t:run.t + E].cpu().pin_memory()
        vh = run.Vn[run.t:run.t + E].cpu().pin_memory()
        oh = [torch.empty(run.O.shape, dtype=run.O.dtype).pin_memory() for _ in range(2)]
        # double-buffered landing zones: step i+1's H2D and step i-1's D2H run on a copy stream
        # while step i computes (every byte still crosses the host link every step)
        cs = torch.cuda.Stream()
        land = [(torch.empty_like(run.qbuf), torch.empty_like(run.kbuf), torch.empty_like(run.vbuf)) for _ in range(2)]
        oland = [torch.empty_like(run.O) for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_used = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        ev_drained = [torch.cuda.Event() for _ in range(2)]
        e_events = sum(1 for t in range(run.t, run.t + E) if run.is_event(t))

        def h2d(i):
            sl = i % 2
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(ev_used[sl])
                land[sl][0].copy_(qh[i], non_blocking=True)
                land[sl][1].copy_(kh[i], non_blocking=True)
                land[sl][2].copy_(vh[i], non_blocking=True)
                ev_in[sl].record(cs)

        j = [0]

        def e2e_step():
            i = j[0]
            sl = i % 2
            if i == 0:
                h2d(0)                         # inside the timed region
            if i + 1 < E:
                h2d(i + 1)
            with torch.cuda.stream(run.main):
                run.main.wait_event(ev_in[sl])
                run.qbuf.copy_(land[sl][0], non_blocking=True)
                run.kbuf.copy_(land[sl][1], non_blocking=True)
                run.vbuf.copy_(land[sl][2], non_blocking=True)
                ev_used[sl].record(run.main)
                run.kv.step_graph_launch(stream=run.main)
                if run.is_event(run.t):
                    run.classify()
                    run.kv.migrate(stream=run.main, side=run.side)
                if i >= 2:
                    run.main.wait_event(ev_drained[sl])
                oland[sl].copy_(run.O, non_blocking=True)
                ev_out[sl].record(run.main)
            with torch.cuda.stream(cs):
                cs.wait_event(ev_out[sl])
                oh[sl].copy_(oland[sl], non_blocking=True)
                ev_drained[sl].record(cs)
            if i == E - 1:                     # the timed region ends when the last output is on the host
                run.main.wait_event(ev_drained[sl])
            run.t += 1
            j[0] += 1

        _barrier_sync()
        el_e = _max_over_ranks(timed(e2e_step, run.main, E))
        run.sync()
        cs.synchronize()
        h2d_bytes = qh[0].numel() * 2 + kh[0].numel() * 2 + vh[0].numel() * 2
        e2e = {"value": world * E / el_e, "unit": "steps/s", "h2d_bytes_per_step": int(h2d_bytes),
               "d2h_bytes_per_step": int(oh[0].numel() * oh[0].element_size()), "steps": E,
               "events_in_window": e_events,
               "note": "pinned host q/k_new/v_new -> HBM and o -> host every step (double-buffered on a copy "
                       "stream); a window of exactly Delta steps, so the manage event is amortised as in the "
                       "headline"}
    run.close()
    del run
    torch.cuda.empty_cache()

    # ---- HBM-resident bytes per mode (kv_tier_query_sizes of this config, per GPU)
    plain_kv = L * B * w["N"] * 4 * Hkv * d
    resident = {}
    for name, extra in (("differential_staging", {}), ("stream_mode", dict(staging=0)),
                        ("all_hbm_beta100", dict(hbm_bp=10000, evict_bp=0))):
        wx = dict(w, **extra)
        cfg = kt.make_config(B, L, w["Hq"], Hkv, d, w["N"] - 1 + w["steps"], w["P"], hbm_bp=wx["hbm_bp"],
                             evict_bp=wx["evict_bp"], t2_bp=wx["t2_bp"], manage_interval=itv,
                             staging=wx.get("staging", kt.STAGING_ALL))
        sz = kt.query_sizes(cfg)
        resident[name] = {"device_arena": int(sz.device_arena), "t0_store": int(sz.t0_store),
                          "t1_staging": int(sz.t1_staging), "host_pinned": int(sz.host_t1 + sz.host_t2),
                          "device_x_plain_kv": sz.device_arena / plain_kv}
    resident["plain_kv_bytes"] = int(plain_kv)

    control = stream_leg = host_t1_leg = model_leg = None
    if not args.no_extras:
        # ---- control: the same r and event schedule with beta = 100 % (every survivor in T0): the
        # visible sets match the tiered run's, so the difference is the hierarchy's own cost
        ctl = H.TieredDecode(dict(w, hbm_bp=10000), device=dev, out_fp32=False, split=args.split, seed_offset=seed_off,
                             step_kernel=STEP_KERNELS[args.step_kernel])
        ctl.capture()
        mc = measure_tiered(ctl, W, K, dict(w, hbm_bp=10000), local, with_clocks=False)
        ctl.close()
        del ctl
        torch.cuda.empty_cache()
        tc = _max_over_ranks(mc["t_amortized"])
        control = {"steps_per_s": world / tc, "ms_per_step": 1e3 * tc,
                   "hierarchy_overhead_pct": 100.0 * (1.0 - tc / t_amort),
                   "note": "beta = 100 %, same r, same events: identical visible sets, every survivor in T0"}

        # ---- stream mode (S = 0): T1 rows cross the host link every step (AMB-13)
        Ks, Ws = 8, 2
        sr = H.TieredDecode(dict(w, staging=0), device=dev, out_fp32=False, split=args.split, seed_offset=seed_off)
        sr.capture()
        for _ in range(Ws):
            sr.step()
        sr.sync()
        cs1 = sr.kv.layout()[0]
        _barrier_sync()
        el_s = _max_over_ranks(timed(lambda: sr.step(manage=False), sr.main, Ks))
        t1_bytes = L * B * Hkv * cs1[1] * 4 * d
        link_peak = host_link_peak_gbs()
        link_gbs = t1_bytes / (el_s / Ks) / 1e9
        stream_leg = {"steps_per_s": world * Ks / el_s, "ms_per_step": 1e3 * el_s / Ks,
                      "host_link_gbs": link_gbs, "host_link_peak_gbs": link_peak,
                      "host_link_frac": link_gbs / link_peak if link_peak else None,
                      "host_link_nominal_gbs": 63.0, "host_link_frac_of_nominal": link_gbs / 63.0,
                      "t1_bytes_per_step": int(t1_bytes),
                      "prefetch_overhead_pct_vs_control": 100.0 * (1 - tc / (el_s / Ks)),
                      "note": "strict DDR residency: every T1 row re-read from pinned host memory per step "
                              "(zero-copy gather, layer-ahead on a side stream, per-layer kernels); host-link bound"}
        sr.close()
        del sr
        torch.cuda.empty_cache()

        # ---- N1: T1 attended on the host cores where it lives
        Kh, Wh = 4, 1
        hr = H.HostT1Decode(dict(w, staging=0), device=dev, split=args.split, seed_offset=seed_off)
        for _ in range(Wh):
            hr.step()
        hr.sync()
        _barrier_sync()
        el_h = _max_over_ranks(timed(hr.step, hr.run.main, Kh))
        hq = w["Hq"]
        link_b = L * B * (hq * d * 2 + hq * (d + 2) * 4 + hq * 2 * 4 + Hkv * cs1[1] * 4)
        host_t1_leg = {"steps_per_s": world * Kh / el_h, "ms_per_step": 1e3 * el_h / Kh,
                       "link_bytes_per_step": int(link_b), "t1_row_bytes_avoided": int(t1_bytes),
                       "vs_stream_mode": (Kh / el_h) / (Ks / el_s), "host_threads": os.cpu_count()}
        hr.close()
        del hr
        torch.cuda.empty_cache()

        # ---- N4 (partial): the same attention inside a decoder of the model's shape (random bf16
        # weights, torch/cuBLAS for the non-attention layers), per-layer ABI with PDL
        if args.config in MODEL_DIMS:
            hidden, inter = MODEL_DIMS[args.config]
            Km, Wm = 64, 3                      # one Delta: exactly one classify/migrate event (t = 64)
            model_leg = {"hidden": hidden, "intermediate": inter,
                         "note": "random bf16 weights, RMSNorm + GEMMs + SiLU in torch/cuBLAS, no RoPE / LM head; "
                                 "each decoder step is ONE CUDA graph (torch.cuda.graph around the library's "
                                 "kv_tier_capture_begin/_end, kv_tier_graph_advance per replay) except "
                                 "hierarchy_eager; the Delta-step window holds one classify/migrate event; the "
                                 "prefix K/V come from the decoder's own causal prefill over N-1 random prompt "
                                 "embeddings (Alg. 1 line 1), the first decode input is the prompt's last output"}
            for name, extra, graph in (("all_hbm_no_eviction", dict(hbm_bp=10000, evict_bp=0), True),
                                       ("hierarchy", {}, True), ("hierarchy_eager", {}, False),
                                       ("hierarchy_stream_mode", dict(staging=0), True)):
                md = H.ModelDecode(dict(w, **extra), hidden=hidden, inter=inter, device=dev,
                                   split=args.split, seed_offset=seed_off, prefill=True)
                for _ in range(Wm):
                    md.step()
                if graph:
                    md.capture()
                    md.step()
                md.sync()
                _barrier_sync()
                el_m = _max_over_ranks(timed(md.step, md.run.main, Km))
                model_leg[name] = {"tokens_per_s": world * B * Km / el_m, "ms_per_step": 1e3 * el_m / Km}
                md.close()
                del md
                torch.cuda.empty_cache()
            b0 = model_leg["all_hbm_no_eviction"]["ms_per_step"]
            for name in ("hierarchy", "hierarchy_eager", "hierarchy_stream_mode"):
                model_leg[name]["overhead_pct_vs_all_hbm"] = 100.0 * (model_leg[name]["ms_per_step"] / b0 - 1.0)

    # ---- configs[3] strong scaling (N > 1): the 32B-shaped batch (B = 32) split over the ranks, so the
    # whole-job work is fixed as N grows; the driver's SCALE lines stay request-sharded weak scaling
    strong_leg = None
    if world > 1 and not args.no_extras:
        w32 = H.workload("32b", steps=W + K + 66)
        if w32["B"] % world == 0:
            w32 = dict(w32, B=w32["B"] // world)
            sr32 = H.TieredDecode(w32, device=dev, out_fp32=False, split=args.split, seed_offset=seed_off,
                                  step_kernel=STEP_KERNELS[args.step_kernel])
            sr32.capture()
            m32 = measure_tiered(sr32, W, K, w32, local, with_clocks=False)
            sr32.close()
            del sr32
            torch.cuda.empty_cache()
            t32 = _max_over_ranks(m32["t_amortized"])
            strong_leg = {"workload": "32b-shaped (BASELINE.json configs[3]): global B=32 split over the ranks, "
                                      f"B={w32['B']}/GPU L={w32['L']} N={w32['N']}",
                          "scaling": "strong", "steps_per_s": 1.0 / t32, "ms_per_step": 1e3 * t32,
                          "tokens_per_s": 32.0 / t32,
                          "note": "one decode step of the whole 32-request batch = every rank's step; time = max over ranks"}
        else:
            strong_leg = {"skipped": f"B=32 does not split over {world} ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        cpu = cpu_oracle_sample(w, args.cpu_seconds)
        cpu["cpu_model"] = _cpu_model()
        cpu["single_thread"] = cpu_oracle_sample(w, args.cpu_seconds / 2, threads=1)["value"]

    achieved = step_bytes / m["t_step"] / 1e9           # the whole-step kernel: one launch per step
    if rank == 0:
        out = {
            "metric": METRIC,
            "value": sps, "unit": "steps/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * t_amort, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.config}-shaped (BASELINE.json configs[{CONFIG_INDEX.get(args.config, '?')}]): "
                                   f"B={B}/GPU L={L} Hq/Hkv={w['Hq']}/{Hkv} d={d} N={w['N']} beta={args.hbm}bp "
                                   f"r={args.evict}bp Delta={itv} differential staging"
                                   + ("" if pol == 0 else f" policy={args.policy}"
                                      + (f" budget={args.budget}" if pol in (2, 3) else ""))
                                   + ("" if args.scorer == "attention" else f" scorer={args.scorer}")
                                   + ("" if not args.positions else
                                      f" (N overridden: {args.positions} positions per request"
                                      + (", one rank's share of the 8-way sequence split; the per-layer "
                                         "exchange is not in this number" if args.config == "70b" else "") + ")"),
                       "global_batch": B * world, "parallelism": f"request-sharded x{world}",
                       "l2": "no flush: per-step K/V traffic > 126 MB L2",
                       "step_kernel": {"ctas": shape[0], "ctas_per_kv_head": shape[1], "kv_heads_per_cta": shape[2],
                                       "consumer": {8: "mma.sync x 8 warps", 4: "mma.sync x 4 warps",
                                                    5: "tcgen05/TMEM (4 softmax warps + issuer)"}
                                       .get(shape[3], shape[3])}},
            "value_note": "1 / (t_step + t_event / Delta): t_step = the timed window's event-free step time, "
                          "t_event = mean classify + migrate time, both CUDA-event measured in this run",
            "window": {"value_raw": world * K / el_max, "ms_per_step_raw": 1e3 * el_max / K,
                       "events_in_window": m["n_events"], "t_step_us": 1e6 * m["t_step"],
                       "t_event_us": 1e6 * m["t_event"], "event_share_pct": 100.0 * m["t_event"] / itv / t_amort},
            "hbm_gbs": step_bytes / t_amort / 1e9 * world, "hbm_frac_of_measured_peak": step_bytes / t_amort / 1e9 / peaks["hbm_gbs"],
            "bytes_per_step": int(step_bytes), "bytes_note": "a3 + a4 algorithmic bytes at each step's own visible "
                                                             "set (mean over the window); event traffic excluded",
            "census_b0": counts, "n_visible_end": n_vis,
            # differential staging (paper §3.4): no T1 byte crosses the host link between events, so the
            # per-step prefetch cost is the event's offload/migrate share
            "prefetch_overhead_pct": 100.0 * m["t_event"] / itv / t_amort,
            "prefetch_overhead_note": "differential staging: T1 rows cross the link only at manage events; "
                                      "= classify + migrate (incl. D2H offload) amortised over Delta / step time",
            "control": control,
            "hbm_resident": resident,
            "roofline": {"bound": "hbm", "kernel": "k_decode_step", "achieved": achieved, "peak": peaks["hbm_gbs"],
                         "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None,
                         "launch_us": 1e6 * m["t_step"],
                         "launch_us_src": "event-free step time of the timed window (the step graph: begin_step, "
                                          "k_decode_step, end_step), CUDA events on the launching stream",
                         "algorithmic_bytes_per_launch": int(step_bytes), "peak_src": peaks["src"]},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": K * 3 + m["n_events"] * EVENT_LAUNCHES,
            "clocks": m["clocks"],
            "stream_mode": stream_leg, "host_t1": host_t1_leg, "model_decode": model_leg, "strong_32b": strong_leg,
            "context": "paper: 5-7% transfer overhead on RTX 5080 PCIe Gen5, unpinned, 7B int8, batch 1 (P:642)",
        }
        tp = os.path.join(ROOT, "profiles", "attn_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            if tj.get("kernel") == "k_decode_step" and tj.get("config") == args.config and \
                    tj.get("hbm") == args.hbm and tj.get("evict") == args.evict:
                out["roofline"]["traffic"] = tj.get("dram_bytes_per_launch")
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sequence_sharded(args, w, world, rank, local, dev, peaks):
    """--shard sequence: the ranks share ONE batch, each owning the 64-position blocks
    k % world == rank.  The library owns the NCCL communicator (kv_tier_init with an
    nccl_unique_id): per layer decode_attention_lse -> ncclAllGather of (o, m, l) -> the
    rank-order LSE combine -> score_update_lse, the whole step captured as one CUDA graph;
    events all-gather S_part inside kv_tier_classify.  Strong scaling."""
    from paper_2605_09490_b200 import harness as H
    from paper_2605_09490_b200 import kvtier as kt
    W, K = args.warmup, args.steps
    nid = [kt.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        import torch.distributed as dist
        dist.broadcast_object_list(nid, src=0)
    run = H.TieredDecode(w, device=dev, out_fp32=True, shard=kt.SHARD_SEQUENCE, rank=rank, world=world,
                         nccl_id=nid[0])
    run.capture()
    for _ in range(W):
        run.step()
    _barrier_sync()
    with ClockSampler(local) as clk:
        el = timed(run.step, run.main, K)
    _barrier_sync()
    el_max = _max_over_ranks(el)
    run.sync()

    class _Sr:                     # the census / close interface the report below uses
        pass
    sr = _Sr()
    sr.run, sr.close = run, run.close
    counts, _ = sr.run.kv.census()
    own = [int(x) for x in counts[0]]
    n_vis_own = own[0] + own[1] + own[2]
    L = w["L"]
    step_bytes = _sum_over_ranks(L * attn_bytes(w, own, n_vis_own))
    sps = K / el_max
    sr.close()
    del sr, run
    import torch
    torch.cuda.empty_cache()
    # the same batch request-sharded on one GPU, the same events: per-layer kernels (step_kernel = 3,
    # the kernels the sequence step runs plus the exchange) and the whole-step kernel
    ref_rates = None
    if world == 1 and not args.no_extras:
        ref_rates = {}
        for name, sk in (("request_per_layer_kernels", 3), ("request_whole_step_kernel", 0)):
            rr = H.TieredDecode(w, device=dev, out_fp32=True, step_kernel=sk)
            rr.capture()
            for _ in range(W):
                rr.step()
            rr.sync()
            el_r = timed(rr.step, rr.main, K)
            rr.close()
            del rr
            torch.cuda.empty_cache()
            ref_rates[name] = {"steps_per_s": K / el_r, "sequence_over_this": sps / (K / el_r)}
    if rank == 0:
        hbm = step_bytes * sps / 1e9
        print(json.dumps({
            "metric": METRIC, "value": sps, "unit": "steps/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 / sps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.config}-shaped (BASELINE.json configs[{CONFIG_INDEX.get(args.config, '?')}]): "
                                   f"B={w['B']} (whole batch) L={L} Hq/Hkv={w['Hq']}/{w['Hkv']} d={w['d']} N={w['N']} "
                                   f"beta={args.hbm}bp r={args.evict}bp, sequence-sharded",
                       "global_batch": w["B"], "parallelism": f"sequence-sharded x{world} (64-position blocks, "
                                                            f"per-layer NCCL all-gather + LSE combine in the "
                                                            f"step graph)"},
            "hbm_gbs": hbm, "hbm_frac_of_measured_peak": hbm / (peaks["hbm_gbs"] * world),
            "bytes_per_step": int(step_bytes), "census_rank0_b0": own,
            "clocks": clk.summary(), "gpu_launches": K * (4 * L + 2), "request_sharded_n1": ref_rates,
            "note": "one CUDA graph per step: per layer decode + merge + NCCL all-gather + LSE combine + "
                    "score rescale on the library's communicator; events (classify all-gathers S_part) "
                    "inside the window",
        }), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
