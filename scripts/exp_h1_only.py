"""Host-T1 (N1) step rate alone on the 7B shape (stream mode): python scripts/exp_h1_only.py"""
import sys, time, torch
sys.path.insert(0, ".")
from paper_2605_09490_b200 import harness as H
import os
w = H.workload("7b", steps=12, staging=0, hbm_bp=int(os.environ.get("HBM", "5000")))
h = H.HostT1Decode(w)
for _ in range(2):
    h.step()
h.sync()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(h.run.main)
for _ in range(8):
    h.step()
b.record(h.run.main)
b.synchronize()
print(round(8 / (a.elapsed_time(b) / 1e3), 1))
h.close()
