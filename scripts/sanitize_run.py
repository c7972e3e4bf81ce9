"""Small workload for compute-sanitizer: the tiny config through the step graph
(whole-step kernel), the per-layer ABI, stream mode and T2, with events, checked against the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_09490_b200 import harness as H  # noqa: E402
from tests.oracle_runner import OracleRun, o_close  # noqa: E402

for name, kw, layers in (("step graph, T2", dict(t2_bp=3000, B=2, L=2), False),
                         ("per-layer ABI", dict(B=2, L=2), True),
                         ("stream mode", dict(staging=0, L=2), True)):
    w = H.workload("tiny", interval=4, steps=9, **kw)
    run = H.TieredDecode(w)
    if not layers:
        run.capture()
    orc = OracleRun(w)
    for t in range(w["steps"]):
        run.step_layers() if layers else run.step()
        ok, mabs, _ = o_close(run.output(), orc.step())
        assert ok, (name, t, mabs)
    run.sync()
    run.close()
    print("ok", name, flush=True)
