"""Mean SM-clock cycles of the step kernel's per-layer segments (KVTIER_TRACE clock64 slots)."""
import sys
import numpy as np
tr = np.load(sys.argv[1]).astype(np.int64)
L, n, _ = tr.shape
names = [(12, 13, "wait request"), (13, 14, "q load"), (14, 15, "stage loop"), (15, 16, "combine"),
         (16, 17, "push + new token"), (17, 18, "rx wait"), (18, 19, "merge + o store"), (19, 20, "signal")]
tot = 0
for a, b, nm in names:
    d = (tr[1:L - 1, :, b] - tr[1:L - 1, :, a]).astype(np.float64)
    d = d[(tr[1:L - 1, :, a] > 0) & (tr[1:L - 1, :, b] > 0)]
    print(f"{nm:18s} mean {d.mean():8.0f} cyc  median {np.median(d):8.0f}")
    tot += d.mean()
cyc = (tr[2:L - 1, :, 12] - tr[1:L - 2, :, 12]).astype(np.float64)
print(f"{'layer (12->12)':18s} mean {cyc.mean():8.0f} cyc; sum of segments {tot:.0f}")

if tr.shape[2] > 21:
    wf = tr[1:L - 1, :, 21].astype(np.float64)
    wf = wf[wf > 0]
    if wf.size:
        print(f"{'stage data waits':18s} mean {wf.mean():8.0f} cyc per layer (warp 0, inside the stage loop)")
