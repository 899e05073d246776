"""K1 in isolation at full C4 size (n = 24,883,200, m = 200, fp32): K1 variants with and without
the fused background (SDMD_BG_NODMD=1 runs the background pass with zero coefficients and no
DMD, so no eigen workers compete).  Frame content does not affect the timing.
Usage: python scripts/k1_micro.py [frames]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1612_07875_b200 import StreamingDMD  # noqa: E402

n, m = 3840 * 2160 * 3, 200
T = int(sys.argv[1]) if len(sys.argv) > 1 else 30
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["v2", "v1"]
src = torch.rand(n, device="cuda:0")
os.environ["SDMD_BG_NODMD"] = "1"
for mode in modes:
    os.environ["SDMD_K1"] = mode
    for bg in (False, True):
        eng = StreamingDMD(n, m, dtype="f32", dmd=False, background=bg, workers=4)
        for t in range(m + 8):
            eng.push(src)
        eng.sync()
        eng.stats(reset=True)
        eng.set_timing(True)
        for t in range(T):
            eng.push(src)
        eng.sync()
        st = eng.stats(reset=True)
        ms = st["k1_ms"] / st["k1_launches"]
        gbs = ((m + 1) * n * 4 + (9 * n if bg else 0)) / (ms / 1e3) / 1e9
        print(json.dumps({"mode": mode, "bg": bg, "k1_ms": round(ms, 4), "GB/s": round(gbs, 1),
                          "frac_of_6537": round(gbs / 6537.3, 3)}), flush=True)
        eng.close()
