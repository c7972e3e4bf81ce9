"""Sweep decode-attention launch shapes (cluster split x kernel variant) on a workload.

    python scripts/sweep_attn.py --config 7b --steps 64
Prints one line per (split, variant): ms/step of the captured step graph (no events in
the timed window) and the isolated kernel time of one layer.
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
ap.add_argument("--steps", type=int, default=48)
ap.add_argument("--splits", default="1,2,3,4,6,8")
ap.add_argument("--variants", default="0,1,2,3,4,5")
ap.add_argument("--env", default="", help="KEY=VAL,... set before each ctx (e.g. KVTIER_PDL_PRE=1)")
a = ap.parse_args()
res = []
for kv_ in [x for x in a.env.split(",") if x]:
    k_, v_ = kv_.split("=")
    os.environ[k_] = v_
for split in [int(x) for x in a.splits.split(",")]:
    for var in [int(x) for x in a.variants.split(",")]:
        w = H.workload(a.config, steps=2 + a.steps)
        try:
            run = H.TieredDecode(w, out_fp32=False, split=split, variant=var)
        except Exception as e:      # e.g. smem too large for this variant
            print(json.dumps({"split": split, "variant": var, "error": str(e)[:120]}), flush=True)
            continue
        run.capture()
        run.step()
        run.step()          # t = 0 event done, t = 1 plain
        run.sync()
        st = run.main
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def plain():
            with torch.cuda.stream(st):
                run.qbuf.copy_(run.Q[run.t], non_blocking=True)
                run.kbuf.copy_(run.Kn[run.t], non_blocking=True)
                run.vbuf.copy_(run.Vn[run.t], non_blocking=True)
                run.kv.step_graph_launch(stream=st)
            run.t += 1
        e0.record(st)
        for _ in range(a.steps):
            plain()
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
        r = {"split": split, "variant": var, "ms_per_step": round(ms, 4), "us_per_layer": round(1e3 * ms / w["L"], 2)}
        res.append(r)
        print(json.dumps(r), flush=True)
        run.close()
        del run
        torch.cuda.empty_cache()
best = min(res, key=lambda r: r["ms_per_step"])
print("BEST", json.dumps(best))
