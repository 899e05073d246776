"""K2 (DMMA) timing: a0 init Gram and a12 modes on the C4 and C2 shapes, one GPU.

    python scripts/k2_bench.py [--skip-c4]

Wall time of sdmd_init_window (D2D copy of the window into the ring + Gram) and of
sdmd_get_modes (T = Y W, Φ = X'T), synchronised on both sides; kernel-only times come from the
ncu launch list of the same command (profiles/).  Algorithmic flops: init n·k(k+1) (upper
triangle incl. diagonal, k = m+1), modes 4·n·m·nc (real n x m by complex m x nc)."""
from __future__ import annotations

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


def wall(f, reps=1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def run(name, Zd, n, m, dtype, nc, r_max=0):
    eng = StreamingDMD(n, m, dtype=dtype, workers=1, r_max=r_max)
    eng.init_window(Zd)                                  # warm-up (module load, allocation)
    eng.sync()
    t_init = wall(lambda: (eng.init_window(Zd), eng.sync()), reps=3)
    sp = eng.spectrum()
    nc = min(nc, sp["r"])
    out = torch.empty((nc, n), dtype=torch.complex128, device="cuda:0")
    eng.modes(list(range(nc)), out=out)
    t_modes = wall(lambda: eng.modes(list(range(nc)), out=out), reps=3)
    k = m + 1
    res = {"config": name, "n": n, "m": m, "dtype": dtype, "r": sp["r"], "nc": nc,
           "init_ms_wall": round(t_init * 1e3, 3),
           "init_gram_flops": n * k * (k + 1),
           "modes_ms_wall": round(t_modes * 1e3, 3),
           "modes_flops": 4 * n * m * nc,
           }
    eng.close()
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-c4", action="store_true")
    a = ap.parse_args()
    cw = synth.cylinder_wake()
    X = cw.frames(0, 151)
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
    run("C2", Xd, cw.n, 150, "f64", 21, r_max=21)
    del Xd
    if not a.skip_c4:
        vs = synth.video_config("C4")
        m = 200
        Zd = torch.empty((m + 1, vs.n), dtype=torch.float32, device="cuda:0")
        for t in range(m + 1):
            Zd[t] = vs.frame(t, device="cuda:0")
        run("C4", Zd, vs.n, m, "f32", 64)


if __name__ == "__main__":
    main()
