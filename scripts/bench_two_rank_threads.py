"""The multi-rank pipeline under load on ONE GPU: C4 split over 2 ranks (row halves) driven by two
host threads, collectives through the in-process test group (SDMD_LOCAL_GROUP=1), eigen sharding
on.  Both ranks share the GPU, so the aggregate should match one rank's rate; the point is that
the sharded pipeline (per-frame allreduce, broadcast of c_t, per-rank K4 of every other frame)
streams at full speed without stalls.  Prints snapshots/s (wall clock around the device work)."""
import os
import sys
import threading
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
os.environ["SDMD_LOCAL_GROUP"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1612_07875_b200 import StreamingDMD, row_partition  # noqa: E402


def main(steps=200, ranks=2, workers=3):
    vs = synth.video_config("C4")
    m = 200
    uid = bytes((17 * i + 1) % 256 for i in range(128))
    pools, engs = {}, {}
    P = m + 1 + 60
    for r in range(ranks):
        b, e = row_partition(vs.n, ranks, r)
        pool = torch.empty((P, e - b), dtype=torch.float32, device="cuda")
        for t in range(P):
            pool[t].copy_(vs.frame(t, device="cuda", row_slice=(b, e)))
        pools[r] = pool
    out = {}

    def run(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            b, e = row_partition(vs.n, ranks, r)
            eng = StreamingDMD(e - b, m, dtype="f32", background=True, workers=workers, rank=r,
                               nranks=ranks, row_begin=b, n_global=vs.n, nccl_uid=uid)
            eng.init_window(pools[r][: m + 1])
            t = m + 1
            for _ in range(40):                                   # fill + warm-up
                eng.push(pools[r][t % P]); t += 1
            eng.sync()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(steps):
                eng.push(pools[r][t % P]); t += 1
            eng.join()
            eng.sync()
            torch.cuda.synchronize()
            out[r] = (time.perf_counter() - t0, eng.info()["lag"], eng.spectrum()["frame"])
            eng.close()
    th = [threading.Thread(target=run, args=(r,)) for r in range(ranks)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    wall = max(v[0] for v in out.values())
    print(f"{ranks} ranks on one GPU: {steps / wall:.1f} snapshots/s (wall), lag {out[0][1]}, "
          f"newest frames solved per rank {[out[r][2] for r in sorted(out)]}")


if __name__ == "__main__":
    main()
