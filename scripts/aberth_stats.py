"""Per-frame eig(Ã) diagnostics on a C4-shaped stream (m = 200): Aberth iterations (−1 = did not
certify → QR fallback), evaluations and eigenvalue-phase cycles.  Usage:
python scripts/aberth_stats.py [frames] [workers]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1612_07875_b200 import StreamingDMD  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 120
W = int(sys.argv[2]) if len(sys.argv) > 2 else 6
m = 200
vs = synth.video_config("C4s")
frames = torch.stack([vs.frame(t, "cuda:0") for t in range(m + 1 + T)])
eng = StreamingDMD(vs.n, m, dtype="f32", workers=W, background=True)
eng.init_window(frames[: m + 1])
its, fails, ev, cyc = [], 0, [], []
for t in range(m + 1, m + 1 + T):
    eng.push(frames[t])
    eng.sync()
    d = eng.frame_diag()
    its.append(d["aberth_its"])
    fails += d["aberth_its"] < 0
    ev.append(d["aberth_evals"])
    cyc.append(d["cycles"]["qr"])
import collections  # noqa: E402
reasons = dict(collections.Counter(i for i in its if i < 0))
print(json.dumps({"reasons": {str(k): v for k, v in reasons.items()}, "lib": os.environ.get("SDMD_LIB", "default"), "workers": W, "frames": T,
                  "fails": fails, "its": its, "evals_mean": sum(ev) / len(ev),
                  "qr_cycles_mean": sum(cyc) / len(cyc), "qr_cycles_max": max(cyc)}))
