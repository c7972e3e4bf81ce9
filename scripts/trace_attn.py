"""Timeline of one decode_attention launch per layer (KVTIER_TRACE=1): per-CTA phase durations.

    KVTIER_TRACE=1 python scripts/trace_attn.py --split 4 --variant 3
"""
import argparse
import json
import os
import sys

os.environ.setdefault("KVTIER_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_09490_b200 import harness as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7b")
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--policy", type=int, default=0, help="kv_tier_policy (1 = streaming: tiny layers, the chain's latency floor)")
ap.add_argument("--budget", type=int, default=0)
a = ap.parse_args()
w = H.workload(a.config, steps=70 if a.policy else 4, policy=a.policy, budget=a.budget)
run = H.TieredDecode(w, out_fp32=False, split=a.split, variant=a.variant)
if a.graph:
    run.capture()
for _ in range(w["steps"] - 1):
    run.step()
run.sync()
tr = run.kv.debug_trace().astype(np.int64)        # [L][CTAs][8], last step
names = ["start", "pdl_wait", "first_tile", "loop_done", "partial_written", "merge_released", "merge_resident", "merge_end"]
t0 = tr[0, :, 0].min()
rel = (tr - t0) / 1e3
out = {"config": a.config, "split": a.split, "variant": a.variant, "ctas": int(tr.shape[1])}
for l in (0, 1, 2, tr.shape[0] // 2, tr.shape[0] - 1):
    d = {}
    for i, n in enumerate(names):
        col = rel[l, :, i]
        col = col[tr[l, :, i] > 0]          # merge checkpoints exist only on the last CTA of a unit
        d[n] = [round(float(col.min()), 2), round(float(np.median(col)), 2), round(float(col.max()), 2)] if col.size else None
    out[f"L{l}"] = d
    for i, n in ((8, "cons_wait_us"), (9, "cons_busy_us"), (10, "stages"), (11, "prod_empty_wait_us"), (13, "first_stage_busy_us")):
        col = tr[l, :, i].astype(np.float64) / (1.0 if i == 10 else 1e3)
        d[n] = [round(float(col.min()), 2), round(float(np.median(col)), 2), round(float(col.max()), 2)]
    d["prod_done"] = [round(float(x), 2) for x in np.percentile(rel[l, :, 12], [0, 50, 100])]
ends = [float(rel[l, :, 7].max()) for l in range(tr.shape[0])]
out["layer_end_deltas_us"] = [round(ends[l] - ends[l - 1], 2) for l in range(1, len(ends))]
mt = tr[:, :, :].astype(np.int64)
sel = mt[:, :, 16] > 0
if sel.any():
    l = tr.shape[0] // 2
    x = mt[l]
    x = x[x[:, 16] > 0]
    out["merge_loads_us"] = [round(float(v), 2) for v in np.percentile((x[:, 16] - x[:, 5]) / 1e3, [0, 50, 100])]
    out["merge_factors_us"] = [round(float(v), 2) for v in np.percentile((x[:, 17] - x[:, 16]) / 1e3, [0, 50, 100])]
    out["merge_tail_us"] = [round(float(v), 2) for v in np.percentile((x[:, 7] - x[:, 17]) / 1e3, [0, 50, 100])]
print(json.dumps(out))
run.close()
