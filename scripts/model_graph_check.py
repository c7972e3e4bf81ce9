"""ModelDecode: the decoder step replayed as one CUDA graph vs eager (per-step max |diff| of the hidden states)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2605_09490_b200 import harness as H
base = dict(B=2, L=3, Hq=8, Hkv=2, d=64, N=400, P=16, interval=4, steps=14, evict_bp=800, hbm_bp=5000)
def run(mode):
    m = H.ModelDecode(H.workload("tiny", **base), hidden=256, inter=512)
    seq = []
    for t in range(base["steps"]):
        if mode == "graph" and t == 2:
            m.capture()
        if mode == "body" and t >= 2:
            r = m.run
            with torch.cuda.stream(r.main):
                x = m._body(m.x)
                if r.is_event(r.t):
                    r.classify(); r.kv.migrate(stream=r.main, side=r.side)
                m.x = x
            r.t += 1
            seq.append(m.x.float().cpu().numpy())
            continue
        seq.append(m.step().float().cpu().numpy())
    m.sync(); m.close()
    return np.stack(seq)
e = run("eager"); b = run("body"); g = run("graph")
print("body vs eager per-step max diff", [float(np.abs(b[t]-e[t]).max()) for t in range(len(e))])
print("graph vs eager per-step max diff", [float(np.abs(g[t]-e[t]).max()) for t in range(len(e))])
