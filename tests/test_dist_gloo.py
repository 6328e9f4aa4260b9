"""World-size-2 gloo tests of the multi-GPU plumbing (CPU): shard slicing, the
parameter broadcast, the unique-id broadcast and the top-k all-gather, driving
the oracle as the per-rank engine, against the oracle's single-process sharded
semantics."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_16007_b200 import dist as rdist


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(77)
    mu = rng.standard_normal((12, 24)) * 2
    X = (mu[rng.integers(0, 12, 3001)] + rng.standard_normal((3001, 24))).astype(np.float32)
    Q = (mu[rng.integers(0, 12, 9)] + rng.standard_normal((9, 24))).astype(np.float32)
    return X, Q


def _worker(rank, world, port, out_path):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X, Q = _data()
    N, D = X.shape
    nlist, k, nprobe, M = 12, 8, 4, 30
    # rank 0 trains P and the centroids; the others receive them
    P = torch.zeros(D, D)
    C = torch.zeros(nlist, D)
    if rank == 0:
        idx = oracle.OracleIndex(X, nlist, seed=5, max_iter=8)
        P.copy_(torch.from_numpy(idx.P))
        C.copy_(torch.from_numpy(idx.Cr))
    rdist.broadcast_params(P, C)
    uid = rdist.share_unique_id(b"u" * 128 if rank == 0 else None)
    assert uid == b"u" * 128
    lo, hi = rdist.shard_range(N, rank, world)
    Pn, Cn = P.numpy(), C.numpy()
    Cd = Cn.astype(np.float64) @ Pn.astype(np.float64).T  # c = P c'
    a = oracle.assign(X[lo:hi], Cd)
    order = np.argsort(a, kind="stable")
    off = np.concatenate([[0], np.cumsum(np.bincount(a, minlength=nlist))]).astype(np.int64)
    codes, n_o, rho = oracle.encode(X[lo:hi], Pn, Cn, a)
    ids, d = oracle.search(Q, Pn, Cn, off, (order + lo).astype(np.int64), codes[order], n_o[order], rho[order],
                           X[lo:hi], k, nprobe, M, 5, id_offset=lo)
    gi, gd = rdist.allgather_topk(torch.from_numpy(ids), torch.from_numpy(d))
    mi, md = oracle.merge_topk(gi.numpy(), gd.numpy())
    if rank == 0:
        np.savez(out_path, ids=mi, d=md, P=Pn, C=Cn)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_plumbing_matches_oracle_semantics(tmp_path, orc, world):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _port(), out), nprocs=world, join=True)
    r = np.load(out)
    X, Q = _data()
    N, D = X.shape
    P, C = r["P"], r["C"]
    Cd = C.astype(np.float64) @ P.astype(np.float64).T
    # single-process reference of the sharded semantics (O-SH) over the same shards
    outs_i, outs_d = [], []
    for g in range(world):
        lo, hi = rdist.shard_range(N, g, world)
        a = orc.assign(X[lo:hi], Cd)
        order = np.argsort(a, kind="stable")
        off = np.concatenate([[0], np.cumsum(np.bincount(a, minlength=12))]).astype(np.int64)
        codes, n_o, rho = orc.encode(X[lo:hi], P, C, a)
        i, d = orc.search(Q, P, C, off, (order + lo).astype(np.int64), codes[order], n_o[order], rho[order],
                          X[lo:hi], 8, 4, 30, 5, id_offset=lo)
        outs_i.append(i)
        outs_d.append(d)
    ri, rd = orc.merge_topk(np.stack(outs_i), np.stack(outs_d))
    assert np.array_equal(r["ids"], ri) and np.array_equal(r["d"], rd)
    # ids are global and every returned id belongs to some shard
    assert r["ids"].min() >= 0 and r["ids"].max() < N


def test_shard_range_partitions():
    for N in (1, 7, 1000, 10**9):
        for G in (1, 2, 3, 8):
            rs = [rdist.shard_range(N, g, G) for g in range(G)]
            assert rs[0][0] == 0 and rs[-1][1] == N
            assert all(rs[g][1] == rs[g + 1][0] for g in range(G - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
