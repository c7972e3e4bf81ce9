"""Whole-step kernel shape sweep at the 7B shape: for each fixed split s (CTAs per kv head,
kv_tier_config::split), the shape step_plan picks (CTAs, s, m, consumer warps) and the event-free
steps/s through the step graph.

    python scripts/split_sweep.py [--config 7b] [--steps 64] [--splits 2,3,4,5,6,7,8,9]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="7b")
    ap.add_argument("--steps", type=int, default=56)
    ap.add_argument("--splits", default="0,2,3,4,5,6,7,8,9,10,12")
    ap.add_argument("--positions", type=int, default=0, help="override N (positions per request)")
    a = ap.parse_args()
    import torch
    from paper_2605_09490_b200 import harness as H
    for s in (int(x) for x in a.splits.split(",")):
        w = H.workload(a.config, steps=a.steps + 12, **({"N": a.positions} if a.positions else {}))
        try:
            run = H.TieredDecode(w, out_fp32=False, split=s)
        except Exception as e:      # noqa: BLE001 - report the shape as not placeable
            print(f"split={s}: {e}", flush=True)
            continue
        shape = run.kv.layout()[1]
        if shape[0] == 0:
            print(f"split={s}: no whole-step shape", flush=True)
            run.close()
            continue
        run.capture()
        for _ in range(4):
            run.step()                      # t = 0: the event that sets the tiered layout
        run.sync()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(run.main)
        for _ in range(a.steps):
            run.step(manage=False)
        ev1.record(run.main)
        ev1.synchronize()
        us = ev0.elapsed_time(ev1) / a.steps * 1e3
        print(f"split={s}: shape (ctas, s, m, warps) = {shape}: {us:.1f} us/step, {1e6 / us:.0f} steps/s", flush=True)
        run.close()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
