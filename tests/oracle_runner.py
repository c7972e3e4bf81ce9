"""Runs the CPU oracle on the same seeded workload as the GPU harness (tests only)."""
import numpy as np

from oracle import kvtier_oracle as O
from paper_2605_09490_b200.synth import synth as S


class OracleRun:
    """Oracle for requests `reqs` of workload `w` (dict as harness.workload returns)."""

    def __init__(self, w, reqs=None, seed_offset=0):
        self.w = w
        B, L, Hq, Hkv, d, N, P, T = (w[k] for k in ("B", "L", "Hq", "Hkv", "d", "N", "P", "steps"))
        self.reqs = list(range(B)) if reqs is None else list(reqs)
        seed = w["seed"] + seed_offset
        n0 = N - 1
        self.K = S.gen_kv(seed, "k", L, B, Hkv, d, 0, n0 + T, P, S.SINK_SIZE, reqs=self.reqs)
        self.V = S.gen_kv(seed, "v", L, B, Hkv, d, 0, n0 + T, P, S.SINK_SIZE, reqs=self.reqs)
        self.Q = S.gen_q(seed, 0, T, L, B, Hq, Hkv, d, reqs=self.reqs)
        self.cfg = O.OracleConfig(B=len(self.reqs), L=L, Hq=Hq, Hkv=Hkv, d=d, prompt_len=P,
                                  manage_interval=w["interval"], hbm_bp=w["hbm_bp"], evict_bp=w["evict_bp"],
                                  t2_bp=w.get("t2_bp", 0), evict_mode=w.get("evict_mode", 0),
                                  policy=w.get("policy", 0), budget=w.get("budget", 0),
                                  policy_seed=w.get("policy_seed", 0), req_ids=self.reqs,
                                  scorer=w.get("scorer", 0))
        self.st = O.init_state(self.cfg, self.K, self.V, n0)

    def step(self):
        return O.decode_step(self.st, self.Q[self.st.t])


def o_close(g, o):
    """north-star tolerance: |g - o| <= 2e-3 + 1e-2 |o| elementwise (AMB-17)."""
    g = np.asarray(g, dtype=np.float64)
    err = np.abs(g - o)
    ok = err <= 2e-3 + 1e-2 * np.abs(o)
    return bool(ok.all()), float(err.max()), float((err / np.maximum(np.abs(o), 1e-12)).max())


def s_close(g, s):
    """scores: |g - s| <= 1e-5 |s|."""
    g = np.asarray(g, dtype=np.float64)
    s = np.asarray(s, dtype=np.float64)
    err = np.abs(g - s)
    ok = err <= 1e-5 * np.abs(s) + 1e-30
    return bool(ok.all()), float((err / np.maximum(np.abs(s), 1e-30)).max())
