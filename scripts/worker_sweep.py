"""Eigen-worker split sweep on the K4-bound configs: snapshots/s for several (workers W, K4a streams
SDMD_WA, K4b streams SDMD_WB) and extra environment knobs (e.g. SDMD_K4_CL=4, SDMD_JACQ=0).
Usage: python scripts/worker_sweep.py [C2|C3|C5 ...] [--tl DIR]  (--tl: save each run's device
timeline as DIR/<config>_<W>_<wa>_<wb>_<tag>.npy for scripts/tl_view.py)"""
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import bench_configs as B  # noqa: E402

KNOBS = ("SDMD_WA", "SDMD_WB", "SDMD_K4_CL", "SDMD_K1_WAVES")


def with_env(env, f):
    for k in KNOBS:
        os.environ.pop(k, None)
    for k, v in env.items():
        if v:
            os.environ[k] = str(v)
    try:
        return f()
    finally:
        for k in KNOBS:
            os.environ.pop(k, None)
        os.environ.pop("SDMD_TL_OUT", None)


args = sys.argv[1:]
tl_dir = ""
if "--tl" in args:
    i = args.index("--tl")
    tl_dir = args[i + 1]
    del args[i:i + 2]
    os.makedirs(tl_dir, exist_ok=True)
which = args or ["C2", "C3", "C5"]
K = 400
# (W, SDMD_WA, SDMD_WB, extra env)
RUNS = {   # (W, SDMD_WA, SDMD_WB, env, background lag (C3; 0 = library default))
    "C5": [(16, 0, 0, {}, 0)],
    "C3": [(16, 0, 0, {}, 0), (16, 16, 3, {}, 0), (16, 18, 3, {}, 0), (16, 17, 2, {}, 0), (16, 14, 3, {}, 0)],
    "C2": [(14, 0, 0, {}, 0), (14, 18, 3, {}, 0), (14, 22, 3, {}, 0)],
}


def run(cfg, W, wa, wb, extra, f):
    env = {"SDMD_WA": wa, "SDMD_WB": wb, **{k: v for k, v in extra.items() if k.startswith("SDMD")}}
    if tl_dir:
        tag = "_".join(f"{k[5:]}{v}" for k, v in extra.items()) or "def"
        env["SDMD_TL_OUT"] = os.path.join(tl_dir, f"{cfg}_{W}_{wa}_{wb}_{tag}.npy")
    r = with_env(env, f)
    r.update(wa=wa, wb=wb, env=extra)
    print(json.dumps(r), flush=True)


if "C5" in which:
    for W, wa, wb, ex, _ in RUNS["C5"]:
        run("C5", W, wa, wb, ex, lambda: B.sparse_run(K, W))
if "C2" in which:
    cw = synth.cylinder_wake()
    X = torch.from_numpy(cw.frames(0, 300).T.copy()).cuda()
    for W, wa, wb, ex, _ in RUNS["C2"]:
        run("C2", W, wa, wb, ex, lambda: B.dense_run("C2", X, cw.n, 150, "f64", K, W, r_max=21))
    del X
if "C3" in which:
    vs = synth.video_config("C3")
    pool = torch.empty((400, vs.n), dtype=torch.float32, device="cuda")
    for t in range(400):
        pool[t].copy_(vs.frame(t, device="cuda"))
    for W, wa, wb, ex, lag in RUNS["C3"]:
        run("C3", W, wa, wb, dict(ex, lag=lag),
            lambda: B.dense_run("C3", pool, vs.n, 100, "f32", K, W, background=True, lag=lag))
