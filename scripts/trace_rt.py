"""Round-trip latency probe from the flat kernel's trace: side-warp new-token time (one global
round trip per owned new token) and layer time, for the current env settings."""
import os, sys, json
os.environ.setdefault("KVTIER_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2605_09490_b200 import harness as H
w = H.workload(sys.argv[1] if len(sys.argv) > 1 else "7b", steps=4)
run = H.TieredDecode(w, out_fp32=False)
run.capture()
for _ in range(3):
    run.step()
run.sync()
tr = run.kv.debug_trace().astype(np.int64)
out = {}
ends = []
newt, loops, scores, probes, nt_load, nt_comp, nt_pub = [], [], [], [], [], [], []
for l in range(tr.shape[0]):
    x = tr[l]
    live = x[:, 0] > 0
    x = x[live]
    pw = x[:, 1].min()
    ends.append(max(x[:, 3].max(), x[:, 5].max()))
    if l >= 4:
        nt = (x[:, 4] - x[:, 1]) / 1e3
        newt += list(nt[nt > 0.3])
        loops.append(float(np.max((x[:, 3] - pw) / 1e3)))
        scores.append(float(np.median((x[:, 5] - x[:, 4]) / 1e3)))
        probes.append(float(np.median(x[:, 11] / 1e3)))
        sel = x[:, 12] > 0
        if sel.any():
            nt_load.append(float(np.median(x[sel, 12] / 1e3))); nt_comp.append(float(np.median(x[sel, 13] / 1e3))); nt_pub.append(float(np.median(x[sel, 14] / 1e3)))
d = np.diff(np.array(ends)) / 1e3
out["layer_us"] = round(float(np.mean(d[4:])), 2)
out["new_token_us_median"] = round(float(np.median(newt)), 2) if newt else None
out["slowest_cta_us"] = round(float(np.mean(loops)), 2)
out["score_pass_us_median"] = round(float(np.median(scores)), 2)
out["probe_rt_us"] = round(float(np.median(probes)), 2)
if nt_load:
    out["nt_load_us"] = round(float(np.median(nt_load)), 2); out["nt_compute_us"] = round(float(np.median(nt_comp)), 2); out["nt_publish_us"] = round(float(np.median(nt_pub)), 2)
print(os.environ.get("TAG", ""), json.dumps(out))
run.close()
