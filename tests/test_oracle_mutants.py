"""Mutation check of the oracle's pins (-m "not gpu").

Each mutant is a plausible mistake in one oracle behaviour that the GPU parity tests alone
could not arbitrate (they only compare kernel and oracle).  The pins in test_oracle_pins.py
must fail on every mutant: the mutated oracle is written to a scratch tree and the pin file
runs against it.  The repo's own oracle is never modified.
"""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, the exact original text, its mutated replacement, the passage the pin follows)
MUTANTS = [
    ("decode loop attends T3 tokens",                                         # Eq. 3
     "        vis = np.nonzero(st.tier[b, :st.n] != T3)[0]\n        if vis.size == 0:",
     "        vis = np.arange(st.n)\n        if vis.size == 0:"),
    ("T2 rows attended at full precision",                                    # P:151, AMB-12
     "    t2 = st.tier[b, vis] == T2\n    if t2.any():",
     "    t2 = st.tier[b, vis] == T2\n    if False:"),
    ("external score update sums one head per group",
     "        for h in range(g * G, (g + 1) * G):\n            inc += np.asarray(probs_b[h]",
     "        for h in range(g * G, g * G + 1):\n            inc += np.asarray(probs_b[h]"),
    ("a row leaving T2 keeps its original bytes",                             # AMB-12
     "        for p in np.nonzero(from_t2)[0]:\n            st.rowK",
     "        for p in np.nonzero(from_t2)[0][:0]:\n            st.rowK"),
    ("protected window one token short",                                      # AMB-6
     "    m[max(0, n - window_size):n] = True",
     "    m[max(0, n - window_size + 1):n] = True"),
    ("eviction floor on the survivors instead of U_all",                      # AMB-9
     "        n_tot = (evict_bp * (n_live + n_t3)) // 10000",
     "        n_tot = (evict_bp * n_live) // 10000"),
    ("softmax without the 1/sqrt(d) scale",                                   # Eq. 2
     "                z = (K @ q[b, h]) * inv_sqrt_d",
     "                z = (K @ q[b, h])"),
    ("T2 takes the highest-scored survivors",                                 # AMB-11
     "    new[surv[:n_t2]] = T2\n    new[surv[n_t2:len(surv) - n_hbm]] = T1",
     "    new[surv[len(surv) - n_hbm - n_t2:len(surv) - n_hbm]] = T2\n"
     "    new[surv[:len(surv) - n_hbm - n_t2]] = T1"),
    ("observation window one step short",                                     # P:137, AMB-32
     "    return (t + w - 1) % cfg.manage_interval == 0",
     "    return (t + w - 2) % cfg.manage_interval == 0"),
    ("max-pool over every position (T3 included)",                            # P:976, AMB-32
     "    vis = np.nonzero(np.asarray(tier_b[:n]) != T3)[0]\n    return max_pool_visible(W, vis)",
     "    vis = np.arange(n)\n    return max_pool_visible(W, vis)"),
    ("R-KV weights swapped",
     "        return ((RKV_LAMBDA * I).astype(np.float32) - (RKV_ONE_MINUS_LAMBDA * rho)",
     "        return ((RKV_ONE_MINUS_LAMBDA * I).astype(np.float32) - (RKV_LAMBDA * rho)"),
]


@pytest.mark.parametrize("name,orig,mut", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_pins_kill_mutant(name, orig, mut, tmp_path):
    src = open(os.path.join(ROOT, "oracle", "kvtier_oracle.py")).read()
    assert src.count(orig) == 1, f"mutation site not found: {name}"
    os.makedirs(tmp_path / "oracle")
    (tmp_path / "oracle" / "__init__.py").write_text("")
    (tmp_path / "oracle" / "kvtier_oracle.py").write_text(src.replace(orig, mut))
    shutil.copytree(os.path.join(ROOT, "tests"), tmp_path / "tests",
                    ignore=shutil.ignore_patterns("__pycache__"))
    os.symlink(os.path.join(ROOT, "paper_2605_09490_b200"), tmp_path / "paper_2605_09490_b200")
    shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp_path / "pytest.ini")
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_oracle_pins.py", "-x", "-q"],
                       cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0, f"mutant survived every pin: {name}\n{r.stdout[-2000:]}"
    assert "failed" in r.stdout, r.stdout[-2000:]
