"""Batched streaming (K1b): snapshots/s of k-frame pushes vs single pushes.

    python scripts/bench_batch.py [--frames K] [--k 8] [--workers W]

Configs without a background (push_batch needs cfg.background == 0): C4 (3840x2160x3 fp32,
m = 200), C3-shaped (1920x1080 fp32, m = 100) and C2 (cylinder wake fp64, m = 150, r = 21).
Modes: 'single' = push_dense per frame (K1, DMD per frame); 'batch' = push_batch of k frames with
the DMD of every window; 'catchup' = push_batch with the DMD of the newest window only.  K1b
algorithmic bytes per launch = (m + k)·n·s; device-resident frames; CUDA events on the ctx stream
with a device-side join of the eigen workers inside the timed region."""
from __future__ import annotations

import argparse
import json
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1612_07875_b200 import StreamingDMD  # noqa: E402


def measure(name, pool, n, m, dtype, K, k, mode, workers, r_max=0):
    P = pool.shape[0]
    eng = StreamingDMD(n, m, dtype=dtype, workers=workers, r_max=r_max, batch_max=k)
    eng.init_window(pool[: m + 1])
    t = m + 1

    def step():
        nonlocal t
        if mode == "single":
            eng.push(pool[t % P])
            t += 1
        else:
            if t % P + k > P:
                t += P - t % P
            eng.push_batch(pool[t % P: t % P + k], dmd_every=(mode == "batch"))
            t += k
    for _ in range(max(2, (2 * (m + 1)) // (1 if mode == "single" else k))):
        step()
    eng.sync()
    eng.stats(reset=True)
    eng.set_timing(True)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t_start = t
    e0.record(s)
    steps = K if mode == "single" else K // k
    for _ in range(steps):
        step()
    eng.join()
    e1.record(s)
    e1.synchronize()
    eng.sync()
    ms = e0.elapsed_time(e1)
    st = eng.stats(reset=True)
    frames = t - t_start
    es = 4 if dtype == "f32" else 8
    kk = 1 if mode == "single" else k
    k1 = st["k1_ms"] / max(1, st["k1_launches"])
    alg = (m + kk) * n * es
    out = {"config": name, "mode": mode, "k": kk, "n": n, "m": m, "dtype": dtype,
           "frames": frames, "snapshots_per_s": round(frames / (ms / 1e3), 1),
           "gram_pass_ms": round(k1, 4), "gram_pass_GBps": round(alg / (k1 / 1e3) / 1e9, 1),
           "gram_pass_share": round(st["k1_ms"] / ms, 3),
           "k4_launches": int(st["k4_launches"]), "workers": workers}
    eng.close()
    print(json.dumps(out), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=400)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--only", default="")
    ap.add_argument("--modes", default="single,batch,catchup")
    a = ap.parse_args()
    modes = tuple(a.modes.split(","))
    res = []
    if not a.only or a.only == "C4":
        vs = synth.video_config("C4")
        Pn = 200 + 1 + 3 * a.k + 16
        pool = torch.empty((Pn, vs.n), dtype=torch.float32, device="cuda")
        for t in range(Pn):
            pool[t].copy_(vs.frame(t, device="cuda"))
        for mode in modes:
            res.append(measure("C4", pool, vs.n, 200, "f32", a.frames, a.k, mode, a.workers))
        del pool
        torch.cuda.empty_cache()
    if not a.only or a.only == "C3":
        vs = synth.video_config("C3")
        pool = torch.empty((300, vs.n), dtype=torch.float32, device="cuda")
        for t in range(300):
            pool[t].copy_(vs.frame(t, device="cuda"))
        for mode in modes:
            res.append(measure("C3 (no background)", pool, vs.n, 100, "f32", a.frames, a.k, mode, 16))
        del pool
    if not a.only or a.only == "C1":
        pm = synth.planted_c1()
        X = pm.frames(0, 17 + 400)
        pool = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
        for mode in modes:
            res.append(measure("C1", pool, pm.n, 16, "f64", a.frames, a.k, mode, 4))
        del pool
    if not a.only or a.only == "C2":
        cw = synth.cylinder_wake()
        Xc = cw.frames(0, 300)
        pool = torch.from_numpy(np.ascontiguousarray(Xc.T)).cuda()
        for mode in modes:
            res.append(measure("C2", pool, cw.n, 150, "f64", a.frames, a.k, mode, 16, r_max=21))


if __name__ == "__main__":
    main()
