"""C3 Gram-pass probe: the full pipeline vs the Gram pass alone (no eigen work, every SM) with and
without the fused background pass (SDMD_BG_NODMD=1: background pass with zero coefficients), and
background lags.  Usage: python scripts/c3_probe.py"""
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import bench_configs as B  # noqa: E402

vs = synth.video_config("C3")
pool = torch.empty((400, vs.n), dtype=torch.float32, device="cuda")
for t in range(400):
    pool[t].copy_(vs.frame(t, device="cuda"))
runs = [("pipeline", {}, dict(background=True)),
        ("pipeline lag 44", {}, dict(background=True, lag=44)),
        ("K1 + background, no DMD, lag 28", {"SDMD_BG_NODMD": "1"}, dict(background=True, dmd=False, lag=28)),
        ("K1 + background, no DMD, lag 12", {"SDMD_BG_NODMD": "1"}, dict(background=True, dmd=False, lag=12)),
        ("K1 only, no DMD", {}, dict(background=False, dmd=False))]
for name, env, kw in runs:
    os.environ.update(env)
    try:
        r = B.dense_run("C3 " + name, pool, vs.n, 100, "f32", 400, 16, **kw)
    finally:
        for k in env:
            os.environ.pop(k, None)
    print(json.dumps(r), flush=True)
