"""Two NCCL ranks sharing one GPU (diagnostic: NCCL normally refuses duplicate devices).
Each rank holds half the rows of a planted C1 stream with a background; eigen sharding on.
Prints the max normwise Gram error and the spectrum/background agreement with one rank."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    from paper_1612_07875_b200 import StreamingDMD, nccl_unique_id, row_partition
    torch.cuda.set_device(0)
    vs = synth.VideoStream(108, 192, 1, seed=31, side=24)
    m, T = 24, 60
    b, e = row_partition(vs.n, world, rank)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    try:
        eng = StreamingDMD(e - b, m, dtype="f32", background=True, workers=2, rank=rank,
                           nranks=world, row_begin=b, n_global=vs.n, nccl_uid=obj[0])
    except Exception as ex:                                  # NCCL refuses a shared device
        q.put((rank, "create failed: " + str(ex)[:200]))
        dist.destroy_process_group()
        return
    for t in range(T):
        eng.push(vs.frame(t, "cuda:0", (b, e)))
    eng.sync()
    G = eng.gram()
    low, sp, mask, fb = eng.background()
    spec = eng.spectrum()
    q.put((rank, G, low, fb, spec["frame"], spec["lam"]))
    eng.close()
    dist.destroy_process_group()


def main():
    import socket
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=600) for _ in range(2)], key=lambda x: x[0])
    for p in ps:
        p.join(timeout=120)
    if isinstance(res[0][1], str):
        print(res[0][1]); print(res[1][1]); return
    import synth
    from paper_1612_07875_b200 import StreamingDMD
    vs = synth.VideoStream(108, 192, 1, seed=31, side=24)
    m, T = 24, 60
    one = StreamingDMD(vs.n, m, dtype="f32", background=True, workers=2)
    for t in range(T):
        one.push(vs.frame(t, "cuda:0"))
    one.sync()
    G1 = one.gram()
    low1, _, _, fb1 = one.background()
    d = np.sqrt(np.diag(G1))
    print("gram normwise err rank0/rank1:",
          float(np.max(np.abs(res[0][1] - G1) / np.outer(d, d))),
          float(np.max(np.abs(res[1][1] - G1) / np.outer(d, d))))
    print("bitwise equal Gram across ranks:", np.array_equal(res[0][1], res[1][1]))
    low = np.concatenate([res[0][2], res[1][2]])
    print("background frames:", res[0][3], res[1][3], fb1,
          "max rel diff:", float(np.max(np.abs(low - low1)) / np.max(np.abs(low1))))
    print("spectrum frames (rank 0, rank 1):", res[0][4], res[1][4])


if __name__ == "__main__":
    main()
