"""Where a decode step's time goes: graph replay alone vs with per-step input copies, and
per-launch device times of one step (CUDA events around individual ABI calls).

    python scripts/step_breakdown.py --split 8 --variant 4
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_09490_b200 import harness as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7b")
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--steps", type=int, default=32)
a = ap.parse_args()
w = H.workload(a.config, steps=2 + 2 * a.steps + 2)
run = H.TieredDecode(w, out_fp32=False, split=a.split, variant=a.variant)
run.capture()
run.step()
run.step()
run.sync()
st = run.main
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
res = {"config": a.config, "split": a.split, "variant": a.variant}
# (a) graph replay only (inputs of step 2 reused; state still advances)
e0, e1 = ev(), ev()
with torch.cuda.stream(st):
    e0.record(st)
    for _ in range(a.steps):
        run.kv.step_graph_launch(stream=st)
        run.t += 1
    e1.record(st)
e1.synchronize()
res["graph_only_ms"] = e0.elapsed_time(e1) / a.steps
# (b) with per-step input copies (what bench.py times)
e0, e1 = ev(), ev()
e0.record(st)
for _ in range(a.steps):
    with torch.cuda.stream(st):
        run.qbuf.copy_(run.Q[run.t], non_blocking=True)
        run.kbuf.copy_(run.Kn[run.t], non_blocking=True)
        run.vbuf.copy_(run.Vn[run.t], non_blocking=True)
        run.kv.step_graph_launch(stream=st)
    run.t += 1
e1.record(st)
e1.synchronize()
res["with_copies_ms"] = e0.elapsed_time(e1) / a.steps
# (c) per-call device times of one step through the layer API
L = w["L"]
evs = []
with torch.cuda.stream(st):
    t = run.t
    x = [ev(), ev()]
    x[0].record(st)
    run.kv.begin_step(stream=st)
    x[1].record(st)
    evs.append(("begin_step", x))
    for l in range(L):
        x = [ev(), ev()]
        x[0].record(st)
        run.kv.decode_attention(l, run.Q[t, l], run.O[l], 1, stream=st, k_new=run.Kn[t, l], v_new=run.Vn[t, l])
        x[1].record(st)
        evs.append((f"attn{l}", x))
    x = [ev(), ev()]
    x[0].record(st)
    run.kv.end_step(stream=st)
    x[1].record(st)
    evs.append(("end_step(+flush)", x))
    run.t += 1
st.synchronize()
d = {n: round(x[0].elapsed_time(x[1]) * 1e3, 2) for n, x in evs}
res["begin_us"] = d["begin_step"]
res["end_flush_us"] = d["end_step(+flush)"]
att = [d[f"attn{l}"] for l in range(L)]
res["attn_us_min_med_max"] = [min(att), sorted(att)[L // 2], max(att)]
print(json.dumps(res))
run.close()
