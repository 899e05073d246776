"""Summarise a bench --timeline .npy: per-frame K1/K4a/K4b/wait times and K4 latency."""
import sys
import numpy as np

tl = np.load(sys.argv[1])
kinds = {0: "K1", 1: "K4a", 2: "K4b", 3: "wait"}
rec = {}
for f, k, s, e in tl:
    rec.setdefault(int(f), {})[int(k)] = (s, e)
fr = sorted(rec)
print("frame   K1[s,e]            K4a[s,e] dur       K4b[s,e] dur       wait  lat(K1 end->K4b end)")
for f in fr[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    r = rec[f]
    k1 = r.get(0, (np.nan, np.nan)); a = r.get(1, (np.nan, np.nan)); b = r.get(2, (np.nan, np.nan))
    w = r.get(3, (0, 0))
    print(f"{f:5d} {k1[0]:8.2f} {k1[1]:8.2f}  {a[0]:8.2f} {a[1]-a[0]:6.2f}  {b[0]:8.2f} {b[1]-b[0]:6.2f}  {w[1]-w[0]:5.2f}  {b[1]-k1[1]:6.2f}")
for k, nm in kinds.items():
    d = np.array([e - s for f, kk, s, e in tl if kk == k])
    if d.size:
        print(f"{nm}: n={d.size} mean {d.mean():.3f} med {np.median(d):.3f} max {d.max():.3f}")
