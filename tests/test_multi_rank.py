"""world_size-2 gloo tests (CPU) of the row-sharding host logic used when nranks > 1:
row partition, 128-byte NCCL-uid broadcast, and the sum of per-rank partial Gram columns
(the only collective of the path) == the unsharded Gram column."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import synth
        from oracle import sdmd_oracle as O
        from paper_1612_07875_b200.sdmd import row_partition
        # uid broadcast (same path bench.py uses for the NCCL unique id)
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        vs = synth.VideoStream(54, 96, 3, seed=77, side=12)
        m = 12
        b, e = row_partition(vs.n, world, rank)
        eng = O.StreamingGram(m)
        for t in range(m + 4):
            eng.push(vs.frame(t, "cpu", (b, e)).numpy())
        g = torch.from_numpy(eng.G[:, -1].copy())
        Gp = torch.from_numpy(eng.G.copy())
        dist.all_reduce(g)
        dist.all_reduce(Gp)
        if rank == 0:
            full = O.StreamingGram(m)
            for t in range(m + 4):
                full.push(vs.frame(t, "cpu").numpy())
            d = np.sqrt(np.diag(full.G))
            err = float(np.max(np.abs(Gp.numpy() - full.G) / np.outer(d, d)))
            err_g = float(np.max(np.abs(g.numpy() - full.G[:, -1]) / (d * d[-1])))
            q.put((rank, err, err_g, (b, e)))
        else:
            q.put((rank, 0.0, 0.0, (b, e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_partial_gram_sum_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0 = [r for r in res if r[0] == 0][0]
    assert r0[1] < 1e-14 and r0[2] < 1e-14
    spans = sorted(r[3] for r in res)
    assert spans[0][0] == 0 and spans[0][1] == spans[1][0] and spans[1][1] == 54 * 96 * 3


def _shard_worker(rank, world, port, q):
    """Eigen sharding (cfg.eigen_shard): frame t's eigenproblems are solved only on
    rank t mod P from the allreduced Gram, its m background coefficients c_t = b_idx λ_idx^m Y w_idx
    are broadcast from that rank, and every rank forms l = X'_rows c_t for its own rows."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        import synth
        from oracle import sdmd_oracle as O
        from paper_1612_07875_b200.sdmd import row_partition
        vs = synth.VideoStream(54, 96, 3, seed=78, side=12)
        m, T = 12, 12 + 1 + 7
        b, e = row_partition(vs.n, world, rank)
        frames = [vs.frame(t, "cpu").numpy().astype(np.float64) for t in range(T)]
        part = O.StreamingGram(m)
        lows = {}
        solved = []
        for t in range(T):
            part.push(frames[t][b:e])
            if not part.full:
                continue
            G = torch.from_numpy(part.G.copy())
            dist.all_reduce(G)                               # every rank: the full-window Gram
            c = torch.zeros(2 * m, dtype=torch.float64)
            if t % world == rank:                            # this rank owns frame t's eigenwork
                d = O.dmd_from_gram(G.numpy())
                bb, _ = O.amplitudes(d)
                idx = O.background_index(d["lam"])
                cc = bb[idx] * d["lam"][idx] ** m * (d["vsi"] @ d["W"][:, idx])
                c = torch.from_numpy(np.ascontiguousarray(cc).view(np.float64).copy())
                solved.append(t)
            dist.broadcast(c, src=t % world)
            cc = c.numpy().view(np.complex128)
            Xp = np.stack([frames[k][b:e] for k in range(t - m + 1, t + 1)], axis=1)
            lows[t] = np.abs(Xp @ cc)
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, lows, solved))
        if rank == 0:
            full = O.StreamingDMD(m, background=True)
            err = 0.0
            for t in range(T):
                out = full.push(frames[t])
                if out is None:
                    continue
                low = np.concatenate([g[1][t] for g in sorted(gathered, key=lambda g: g[0])])
                err = max(err, float(np.max(np.abs(low - out["lowrank"])) / np.max(out["lowrank"])))
            owners = sorted((t, g[0]) for g in gathered for t in g[2])
            q.put((err, owners))
    finally:
        dist.destroy_process_group()


def test_two_rank_eigen_sharding_background_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, owners = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12
    assert [t for t, _ in owners] == list(range(12, 20))
    assert all(r == t % 2 for t, r in owners)
