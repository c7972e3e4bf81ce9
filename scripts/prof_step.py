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
a = ap.parse_args()
run = H.TieredDecode(H.workload(a.config, steps=a.steps), out_fp32=False, split=a.split, variant=a.variant)
run.capture()
for _ in range(a.steps):
    run.step()
run.close()
