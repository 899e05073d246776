"""Debug: build-up DMD λ vs oracle per frame (A/B with SDMD_ATILDE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from oracle import sdmd_oracle as O
from paper_1612_07875_b200 import StreamingDMD
pm = synth.planted_c1()
m, T = 16, int(os.environ.get("DBG_T", "12"))
X = pm.frames(0, T)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
eng = StreamingDMD(pm.n, m, dtype="f64", workers=2, buildup=True)
ref = O.StreamingDMD(m, background=False, buildup=True)
for t in range(T):
    eng.push(Xd[t]); out = ref.push(X[:, t])
    if t == 0: continue
    eng.sync(); d = eng.frame_diag()
    try:
        sp = eng.spectrum()
        lam = np.sort_complex(sp["lam"])[:3]
    except Exception as e:
        lam = str(e)[:60]
    print(os.environ.get("SDMD_ATILDE", "tiled"), t, d["status"], d["r"], lam, np.sort_complex(out["lam"])[:3], flush=True)
