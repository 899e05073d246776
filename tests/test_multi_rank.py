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
    """Eigen sharding (cfg.eigen_shard) with ONE collective per frame: frame t's
    eigenproblems are solved only on rank t mod P from the allreduced Gram history; its m background
    coefficients c_t = b_idx λ_idx^m Y w_idx ride the allreduce of the Gram column of frame
    t + L - 1 (the owner's values, zeros on the other ranks, so the sum is exact), and every rank
    forms l = X'_rows c_t for its own rows in the Gram pass of frame t + L.  The same protocol as
    libsdmd's enqueue_frame/stage_c/commit_kernel, at the oracle level (no GPU here)."""
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
        m, L = 12, 3
        T = m + 1 + 9
        b, e = row_partition(vs.n, world, rank)
        frames = [vs.frame(t, "cpu").numpy().astype(np.float64) for t in range(T)]
        cols = []                       # this rank's rows of the window
        G = np.zeros((0, 0))            # allreduced full-window Gram (identical on every rank)
        own_c, recv_c, lows, solved = {}, {}, {}, []
        n_coll = 0
        for t in range(T):
            # Gram pass of frame t: partial column + the background of frame t - L (c received)
            cols = (cols + [frames[t][b:e]])[-(m + 1):]
            g = O.gram_column(cols, cols[-1])
            fb = t - L
            if fb >= m:
                cc = recv_c[fb]
                Xp = np.stack([frames[k][b:e] for k in range(fb - m + 1, fb + 1)], axis=1)
                lows[fb] = np.abs(Xp @ cc)
            # the one collective: g_t, with c_{t+1-L} appended when the next pass needs it
            fb1 = t + 1 - L
            fold = m <= fb1 <= t - 1
            vec = g
            if fold:
                c = own_c[fb1] if fb1 % world == rank else np.zeros(m, dtype=np.complex128)
                vec = np.concatenate([g, np.ascontiguousarray(c).view(np.float64)])
            v = torch.from_numpy(vec.copy())
            dist.all_reduce(v)
            n_coll += 1
            v = v.numpy()
            gs = v[:len(g)]
            if fold:
                recv_c[fb1] = v[len(g):].copy().view(np.complex128)
            # commit: slide the Gram and append the reduced column (Alg 1)
            k = len(gs) - 1
            Gn = np.zeros((k + 1, k + 1))
            Gn[:k, :k] = G[1:, 1:] if G.shape[0] == k + 1 else G
            Gn[:, k] = gs
            Gn[k, :] = gs
            G = Gn
            if t >= m and t % world == rank:                # this rank owns frame t's eigenwork
                d = O.dmd_from_gram(G)
                bb, _ = O.amplitudes(d)
                idx = O.background_index(d["lam"])
                own_c[t] = bb[idx] * d["lam"][idx] ** m * (d["vsi"] @ d["W"][:, idx])
                solved.append(t)
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, lows, solved, n_coll))
        if rank == 0:
            full = O.StreamingDMD(m, background=True)
            err, checked = 0.0, 0
            for t in range(T):
                out = full.push(frames[t])
                if out is None or t not in gathered[0][1]:
                    continue
                low = np.concatenate([g[1][t] for g in sorted(gathered, key=lambda g: g[0])])
                err = max(err, float(np.max(np.abs(low - out["lowrank"])) / np.max(out["lowrank"])))
                checked += 1
            owners = sorted((t, g[0]) for g in gathered for t in g[2])
            q.put((err, owners, checked, [g[3] for g in gathered]))
    finally:
        dist.destroy_process_group()


def test_two_rank_eigen_sharding_background_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err, owners, checked, n_coll = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12 and checked == 22 - 3 - 12
    assert [t for t, _ in owners] == list(range(12, 22))
    assert all(r == t % 2 for t, r in owners)
    assert n_coll == [22, 22]                       # one collective per frame on every rank
