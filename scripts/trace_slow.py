"""Per-CTA breakdown of the slowest CTAs of a mid-step layer (flat kernel, KVT_FLAT_TRACE build)."""
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
l = 14
x = tr[l]
live = x[:, 0] > 0
pw = x[live, 1].min()
rows = []
for c in np.nonzero(live)[0]:
    r = x[c]
    rows.append(dict(c=int(c), loop_end=round((r[3] - pw) / 1e3, 2), first=round((r[2] - pw) / 1e3, 2),
                     side_new=round((r[4] - pw) / 1e3, 2), score=round((r[5] - pw) / 1e3, 2),
                     epi=round(r[9] / 1e3, 2), units=int(r[10]), cwait=round(r[21] / 1e3, 2), cbusy=round(r[22] / 1e3, 2),
                     prod_done=round((r[23] - pw) / 1e3, 2), pwait=round(r[16] / 1e3, 2)))
rows.sort(key=lambda d: -d["loop_end"])
for d in rows[:12]:
    print(json.dumps(d))
print("median", json.dumps(rows[len(rows) // 2]))
print("fastest", json.dumps(rows[-1]))
run.close()
