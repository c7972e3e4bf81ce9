"""Timeline of the flat decode kernel (KVTIER_TRACE=1): per-CTA checkpoints of every layer of
the last step, min / median / max over CTAs in microseconds from the first CTA start of layer 0.

    python scripts/trace_flat.py [--config 7b] [--fvar 0]
"""
import argparse
import json
import os
import sys

os.environ.setdefault("KVTIER_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2605_09490_b200 import harness as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7b")
ap.add_argument("--fvar", default="")
ap.add_argument("--graph", type=int, default=1)
a = ap.parse_args()
if a.fvar:
    os.environ["KVTIER_FVAR"] = a.fvar
w = H.workload(a.config, steps=4)
run = H.TieredDecode(w, out_fp32=False)
if a.graph:
    run.capture()
for _ in range(3):
    run.step()
run.sync()
tr = run.kv.debug_trace().astype(np.int64)        # [L][CTAs][16], last step
names = {0: "start", 1: "pdl_wait", 2: "first_stage", 3: "loop_done", 4: "side_new_done",
         5: "side_score_done", 6: "last_release", 7: "last_unit_done"}
live = tr[0, :, 0] > 0
t0 = tr[0, live, 0].min()
out = {"config": a.config, "ctas": int(live.sum())}
ends = []
for l in range(tr.shape[0]):
    x = tr[l, live]
    end = np.maximum(np.maximum(x[:, 3], x[:, 5]), x[:, 7])
    ends.append(float((end.max() - t0) / 1e3))
    if l not in (0, 1, 2, tr.shape[0] // 2, tr.shape[0] - 1):
        continue
    d = {}
    for i, n in names.items():
        col = x[:, i]
        col = col[col > 0]
        if col.size:
            r = (col - t0) / 1e3
            d[n] = [round(float(r.min()), 2), round(float(np.median(r)), 2), round(float(r.max()), 2)]
    d["merges"] = int(x[:, 8].sum())
    d["epilogue_us_per_cta"] = [round(float(v), 2) for v in np.percentile(x[:, 9] / 1e3, [0, 50, 100])]
    d["units_per_cta"] = [int(v) for v in np.percentile(x[:, 10], [0, 50, 100])]
    d["cons_wait_us"] = [round(float(v), 2) for v in np.percentile(x[:, 21] / 1e3, [0, 50, 100])]
    d["cons_busy_us"] = [round(float(v), 2) for v in np.percentile(x[:, 22] / 1e3, [0, 50, 100])]
    d["prod_empty_wait_us"] = [round(float(v), 2) for v in np.percentile(x[:, 16] / 1e3, [0, 50, 100])]
    d["prod_done"] = [round(float(v), 2) for v in np.percentile((x[:, 23] - t0) / 1e3, [0, 50, 100])]
    d["warp_skew_us"] = [round(float(v), 2) for v in np.percentile((x[:, 17:17 + 4].max(1) - x[:, 17:17 + 4].min(1)) / 1e3, [0, 50, 100])]
    for i, n in ((14, "epi_shfl_newbar_us"), (15, "epi_first_bar_us"),                  (11, "epi_to_cta_o_us"), (12, "epi_to_release_us"), (13, "atomic_us")):
        d[n] = [round(float(v), 2) for v in np.percentile(x[:, i] / 1e3, [0, 50, 100])]
    out[f"L{l}"] = d
out["layer_end_deltas_us"] = [round(ends[l] - ends[l - 1], 2) for l in range(1, len(ends))]
print(json.dumps(out))
run.close()
