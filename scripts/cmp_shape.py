import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2605_09490_b200 import harness as H
from tests.oracle_runner import OracleRun, o_close
w = H.workload("tiny", L=2, interval=8, steps=18, hbm_bp=5000, evict_bp=500, t2_bp=0, B=24, Hq=8, Hkv=4, d=64, N=120, P=16)
for flat in ("0", "1"):
    os.environ["KVTIER_FLAT"] = flat
    run = H.TieredDecode(w); run.capture(); orc = OracleRun(w, reqs=list(range(24)))
    errs = []
    for t in range(w["steps"]):
        run.step(); o = run.output(); ref = orc.step()
        d = np.abs(o - ref); bound = 2e-3 + 1e-2 * np.abs(ref)
        i = np.unravel_index(np.argmax(d - bound), d.shape)
        errs.append((t, float(d.max()), float((d - bound).max()), tuple(int(x) for x in i)))
    run.close()
    print("flat", flat, [e for e in errs if e[2] > -1e-3])
