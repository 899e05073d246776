"""K4 phase breakdown (SM cycles) for several window widths on video-like data (K4 cost does not
depend on n).  Usage: python scripts/diag_k4.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1612_07875_b200 import StreamingDMD  # noqa: E402

vs = synth.video_config("C4s")
for m in [int(a) for a in (sys.argv[1:] or ["16", "100", "150", "200"])]:
    frames = torch.stack([vs.frame(t, "cuda:0") for t in range(m + 9)])
    eng = StreamingDMD(vs.n, m, dtype="f32", workers=1, background=True)
    eng.set_timing(True)
    for t in range(m + 9):
        eng.push(frames[t])
    eng.sync()
    st = eng.stats(reset=True)
    d = eng.frame_diag()
    d["m"] = m
    d["k4_ms_avg"] = st["k4_ms"] / max(1, st["k4_launches"])
    d["k1_ms_avg"] = st["k1_ms"] / max(1, st["k1_launches"])
    print(json.dumps(d), flush=True)
    eng.close()
