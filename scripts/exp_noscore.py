"""Upper bound of the 7B step rate without the fused score update (fuse_score_update = 0):
how much the score pass beside the chain costs.  Experiment only (not a bench number)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2605_09490_b200 import harness as H
w = H.workload("7b", steps=400)
for fuse in (1, 0):
    r = H.TieredDecode(w, out_fp32=False)
    with torch.cuda.stream(r.main):
        r.kv.step_graph_capture(r.qbuf, r.kbuf, r.vbuf, r.O, fuse, stream=r.main, side=r.side)
    r.graph = True
    for _ in range(64):
        r.step()
    r.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(r.main)
    for _ in range(192):
        r.step()
    b.record(r.main)
    b.synchronize()
    print(f"fuse={fuse}: {192 / (a.elapsed_time(b) / 1e3):.1f} steps/s")
    r.close()
