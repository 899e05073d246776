"""Eigen-worker split sweep on the K4-bound configs (C3, C5) and C4: snapshots/s for several
(workers, cluster streams SDMD_WA, single-CTA streams SDMD_WB).  Usage: python scripts/worker_sweep.py"""
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import bench_configs as B  # noqa: E402


def with_env(wa, wb, f):
    for k, v in (("SDMD_WA", wa), ("SDMD_WB", wb)):
        if v:
            os.environ[k] = str(v)
        else:
            os.environ.pop(k, None)
    try:
        return f()
    finally:
        os.environ.pop("SDMD_WA", None)
        os.environ.pop("SDMD_WB", None)


vs = synth.video_config("C3")
pool = torch.empty((400, vs.n), dtype=torch.float32, device="cuda")
for t in range(400):
    pool[t].copy_(vs.frame(t, device="cuda"))
for W, wa, wb in [(20, 0, 0), (16, 8, 4), (12, 8, 4), (12, 10, 3), (16, 10, 6), (10, 8, 2), (14, 12, 4)]:
    r = with_env(wa, wb, lambda: B.dense_run("C3", pool, vs.n, 100, "f32", 400, W, background=True))
    r.update(wa=wa, wb=wb)
    print(json.dumps(r), flush=True)
del pool
torch.cuda.empty_cache()
for W, wa, wb in [(20, 0, 0), (16, 8, 4), (12, 10, 3), (14, 12, 4)]:
    r = with_env(wa, wb, lambda: B.sparse_run(400, W))
    r.update(wa=wa, wb=wb)
    print(json.dumps(r), flush=True)
