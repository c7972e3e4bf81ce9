import sys, numpy as np
sys.path.insert(0, '.')
from paper_2605_09490_b200 import harness as H
from tests.oracle_runner import OracleRun, o_close, s_close
from paper_2605_09490_b200 import kvtier as kt
w = H.workload("tiny", B=1, L=2, Hq=14, Hkv=2, d=128, N=500, P=64, interval=8, steps=10, hbm_bp=4000, evict_bp=800, t2_bp=0)
run = H.TieredDecode(w, split=2, step_kernel=2)
print("layout", run.kv.layout(), flush=True)
run.capture()
orc = OracleRun(w)
for t in range(w["steps"]):
    run.step()
    o = run.output()
    ref = orc.step()
    ok, mabs, _ = o_close(o, ref)
    print(t, ok, mabs, flush=True)
run.sync()
ok, mrel = s_close(run.kv.export(kt.X_SCORES), orc.st.S_part[:, :, :orc.st.n])
print("scores", ok, mrel)
