"""Host cost of a push: wall time of K enqueued pushes (no sync inside) vs the device time of the
same region, for C1 (n = 4096, m = 16, fp64: a push is tiny on the device) and C4s.
Usage: python scripts/host_cost.py"""
import json
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1612_07875_b200 import StreamingDMD  # noqa: E402

pm = synth.planted_c1()
m, K = 16, 2000
X = pm.frames(0, 64)
Xd = torch.from_numpy(np.ascontiguousarray(X.T)).cuda()
for dmd in (True, False):
    eng = StreamingDMD(pm.n, m, dtype="f64", workers=4, dmd=dmd)
    for t in range(m + 40):
        eng.push(Xd[t % 64])
    eng.sync()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(s)
    for t in range(K):
        eng.push(Xd[t % 64])
    w1 = time.perf_counter()
    eng.join()
    e1.record(s)
    e1.synchronize()
    w2 = time.perf_counter()
    eng.sync()
    print(json.dumps({"config": "C1", "dmd": dmd, "pushes": K,
                      "host_enqueue_us_per_push": round((w1 - w0) / K * 1e6, 2),
                      "wall_us_per_push": round((w2 - w0) / K * 1e6, 2),
                      "device_us_per_push": round(e0.elapsed_time(e1) / K * 1e3, 2)}), flush=True)
    eng.close()

# timeline of 40 C1 frames with DMD (K1 / K4a / K4b device intervals, ms relative to the first)
eng = StreamingDMD(pm.n, m, dtype="f64", workers=4)
for t in range(m + 40):
    eng.push(Xd[t % 64])
eng.sync()
eng.stats(reset=True)
eng.set_timing(True)
for t in range(40):
    eng.push(Xd[t % 64])
eng.sync()
tl = eng.timeline()
info = eng.info()
print(json.dumps({"info": info}))
for f, k, a, b in tl[:120]:
    print(f"{int(f):4d} {['K1','K4a','K4b','wait'][int(k)]:4s} {a:8.3f} {b:8.3f} {b-a:7.3f}")
eng.close()
