"""Probe of the whole-step kernel (k_decode_step): steps/s with and without a4, and (with
KVTIER_TRACE=1) the per-layer timeline of the last step from the kernel's %globaltimer trace.

    python scripts/step_probe.py [--config 7b] [--steps 32] [--trace]
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="7b")
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--positions", type=int, default=0, help="override N (positions per request)")
    ap.add_argument("--t2", type=int, default=0)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--step-kernel", type=int, default=0, help="kv_tier_config::step_kernel (2 = tcgen05)")
    a = ap.parse_args()
    if a.trace:
        os.environ["KVTIER_TRACE"] = "1"
    import torch
    from paper_2605_09490_b200 import harness as H
    over = {"B": a.batch} if a.batch else {}
    if a.positions:
        over["N"] = a.positions
    for fuse in (1, 0):
        w = H.workload(a.config, steps=a.steps + 10, t2_bp=a.t2, **over)
        run = H.TieredDecode(w, out_fp32=False, step_kernel=a.step_kernel)
        with torch.cuda.stream(run.main):
            run.kv.step_graph_capture(run.qbuf, run.kbuf, run.vbuf, run.O, fuse, stream=run.main, side=run.side)
        run.graph = True
        for _ in range(2):
            run.step()
        run.sync()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(run.main)
        for _ in range(a.steps):
            run.step(manage=False)
        ev1.record(run.main)
        ev1.synchronize()
        ms = ev0.elapsed_time(ev1) / a.steps
        print(f"fuse_score_update={fuse}: {ms * 1e3:.1f} us/step, {1e3 / ms:.0f} steps/s")
        if a.trace and fuse == 1:
            raw = run.kv.debug_trace().reshape(-1)
            grid = int(raw[23])
            print("grid", grid)
            tr = raw[: w["L"] * grid * 24].reshape(w["L"], grid, 24).astype(np.int64)
            tr[0, 0, 23] = 0
            os.makedirs("gpurun_out", exist_ok=True)
            np.save("gpurun_out/step_trace.npy", tr)
            L = tr.shape[0]
            t = tr[:, :, :6]
            base = t[0, :, 0][t[0, :, 0] > 0].min()
            print("layer  prod_first  cons_start(min/max)  part_end(max)  merged(max)  done(max)  scored")
            for l in range(L):
                def col(k, f):
                    x = t[l, :, k]
                    x = x[x > 0]
                    return (f(x) - base) / 1e3 if x.size else float("nan")
                print(f"{l:5d}  {col(0, np.min):9.2f}  {col(1, np.min):8.2f}/{col(1, np.max):8.2f}  "
                      f"{col(2, np.max):9.2f}  {col(3, np.max):9.2f}  {col(4, np.max):9.2f}  {col(5, np.max):8.2f}")
        run.close()


if __name__ == "__main__":
    main()
