"""Run a few captured decode steps of a workload (for ncu): python scripts/prof_step.py --split 8 --variant 2"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_09490_b200 import harness as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="7b")
ap.add_argument("--split", type=int, default=0)
ap.add_argument("--variant", type=int, default=0)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--staging", type=int, default=-1, help="0 = stream mode (T1 re-read from pinned host memory)")
ap.add_argument("--step-kernel", type=int, default=0)
a = ap.parse_args()
over = {} if a.staging < 0 else {"staging": a.staging}
run = H.TieredDecode(H.workload(a.config, steps=a.steps, **over), out_fp32=False, split=a.split, variant=a.variant,
                     step_kernel=a.step_kernel)
run.capture()
for _ in range(a.steps):
    run.step()
run.close()
