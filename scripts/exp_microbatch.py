"""Micro-batch overlap experiment: the 7B batch of 8 requests as M independent ctxs of 8/M
requests, each with its own stream and step graph, launched concurrently every step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_09490_b200 import harness as H

def run(M, K=128, W=64):
    w = H.workload("7b", B=8 // M, steps=W + K + 1)
    runs = [H.TieredDecode(w, out_fp32=False, seed_offset=17 * i) for i in range(M)]
    for r in runs:
        r.capture()
    for _ in range(W):
        for r in runs:
            r.step()
    torch.cuda.synchronize()
    s0 = runs[0].main
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    done = [torch.cuda.Event() for _ in runs]
    a.record(s0)
    for r in runs[1:]:
        r.main.wait_event(a)
    for _ in range(K):
        for r in runs:
            r.step()
    for r, e in zip(runs[1:], done[1:]):
        e.record(r.main)
        s0.wait_event(e)
    b.record(s0)
    b.synchronize()
    ms = a.elapsed_time(b) / K
    for r in runs:
        r.close()
    return ms

for M in (1, 2, 4):
    ms = run(M)
    print(f"M={M}: {ms:.4f} ms/step  {1e3 / ms:.0f} steps/s  {ms * 1e3 / 28:.2f} us/layer-equivalent")
