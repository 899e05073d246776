"""NEXT-4 scoring (Table 2's methodology: foreground = |x - l| > .2 against the
ground truth; recall, precision, F-measure, PSNR pooled over the scored frames) of the streamed
background of a full-size synthetic video config, on the device through the C ABI.

    python scripts/score_stream.py [--config C3|C4] [--frames T] [--out profiles/x.json]

Every frame pushed after the first full window + lag yields the background of frame t - lag
(sdmd_get_background, DEVICE); its mask is scored against synth's ground truth (the moving
squares) with sdmd_score_background (device counters, no host read-back of the masks)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1612_07875_b200 import StreamingDMD  # noqa: E402

CFG = {"C3": (100, 16), "C4": (200, 6)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3", choices=sorted(CFG))
    ap.add_argument("--frames", type=int, default=400)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    m, W = CFG[a.config]
    vs = synth.video_config(a.config)
    eng = StreamingDMD(vs.n, m, dtype="f32", background=True, workers=W)
    lag = eng.info()["lag"]
    mask = torch.empty(vs.n, dtype=torch.uint8, device="cuda")
    scored = []
    t0 = time.perf_counter()
    for t in range(a.frames):
        eng.push(vs.frame(t, device="cuda"))
        fb = t - lag
        if fb < m:
            continue
        f = eng.background_device(mask=mask)
        assert f == fb, (f, fb)
        gt = torch.from_numpy(vs.truth_mask(f).astype(np.uint8)).cuda()
        eng.score(f, gt)
        scored.append(f)
    eng.sync()
    sc = eng.scores()
    out = {"config": a.config, "n": vs.n, "m": m, "lag": lag, "frames_pushed": a.frames,
           "frames_scored": len(scored), "first_scored": scored[0] if scored else None,
           "threshold": 0.2, "wall_s": round(time.perf_counter() - t0, 2),
           **{k: (float(v) if isinstance(v, (float, np.floating)) else v) for k, v in sc.items()},
           "data": "synthetic: static textured background + 3 moving squares (ground truth), "
                   "noise sigma 0.01 (synth.video_config)"}
    eng.close()
    s = json.dumps(out)
    print(s)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(s + "\n")


if __name__ == "__main__":
    main()
