"""The sharded path on one GPU (-m gpu): SURVEY 8(e), P:L397-407 [sec 3.4].

Every rank of a G-GPU job holds a contiguous id slice of the corpus (so 1/G
of every list), built with rank 0's rotation and centroids; it scans
and re-ranks its shard for all queries and the per-rank top-k are merged by
(dist, id) after one all-gather.  With one GPU in this run:

  * G logical shards are built and searched on the same device and merged
    with rabitq_merge_topk -- each shard's stages checked against the oracle
    on that shard (GPU q' / probes injected: L5 top-M tie band, L6 = the
    oracle's re-rank of the GPU's top-M), the merged result = the oracle's
    merge of the GPU's per-shard results (bit-exact) and = the oracle's
    sharded search (O-SH) up to the L1/L5/L6 tie sets;
  * rabitq_search_sharded over a 1-rank NCCL communicator (the real
    all-gather code path) equals rabitq_search bit for bit, with and without
    query-split probing;
  * query-split probing composed from G probe slices (rabitq_probe on each
    slice, then probes_in) equals the default search bit for bit.
"""
import numpy as np
import pytest
import torch

import synth
import parity_util as pu

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_16007_b200 as rq  # noqa: E402

SEED = 42


@pytest.fixture(scope="module")
def orc():
    import oracle

    oracle.build()
    return oracle


def make_data(D, N, ncent, nq, seed=11):
    s = synth.spec(1, D=D, N=N, ncent=ncent, nlist=ncent, nq=nq, kind="iso", data_seed=seed)
    cen = synth.centres(s, "cpu")
    return synth.base_rows(s, 0, N, "cpu", cen=cen), synth.queries(s, "cpu", cen=cen)


def shard_range(N, g, G):
    return (N * g) // G, (N * (g + 1)) // G


def build_shards(X, nlist, G):
    """rank 0 trains P and the centroids on its own slice (as bench.py's
    G-GPU job does); every rank builds its slice with them and id_offset."""
    N = X.shape[0]
    lo, hi = shard_range(N, 0, G)
    r0 = rq.Index(X[lo:hi].cuda(), nlist=nlist, seed=SEED, id_offset=lo)
    ex0 = r0.export()
    shards = [r0]
    for g in range(1, G):
        lo, hi = shard_range(N, g, G)
        shards.append(rq.Index(X[lo:hi].cuda(), nlist=nlist, seed=SEED, id_offset=lo, rotation=ex0["rotation"],
                               centroids_rot=ex0["centroids"]))
    return shards, ex0


@pytest.mark.parametrize("G", [2, 4])
def test_logical_shards_vs_oracle(orc, G):
    D, N, nlist, nq, k, nprobe, M = 96, 24000, 32, 24, 10, 6, 80
    X, Q = make_data(D, N, nlist, nq)
    shards, ex0 = build_shards(X, nlist, G)
    Xn, Qn = X.numpy(), Q.numpy()
    per_i, per_d, orc_i, orc_d = [], [], [], []
    for g, sh in enumerate(shards):
        lo, hi = shard_range(N, g, G)
        ex = sh.export()
        assert np.array_equal(ex["rotation"], ex0["rotation"]) and np.array_equal(ex["centroids"], ex0["centroids"])
        assert ex["ids"].min() >= lo and ex["ids"].max() < hi  # global ids of the slice
        dbg = dict(qrot=torch.empty(nq, D, device="cuda"),
                   probes=torch.empty(nq, nprobe, dtype=torch.int32, device="cuda"),
                   topm_ids=torch.empty(nq, M, dtype=torch.int64, device="cuda"),
                   topm_est=torch.empty(nq, M, device="cuda"))
        ids, d = sh.search(Q.cuda(), k, nprobe, M, debug=dbg)
        torch.cuda.synchronize()
        ids, d = ids.cpu().numpy(), d.cpu().numpy()
        qr, probes = dbg["qrot"].cpu().numpy(), dbg["probes"].cpu().numpy()
        gt, gest = dbg["topm_ids"].cpu().numpy(), dbg["topm_est"].cpu().numpy()
        pu.check_probe_lists(probes, qr, ex["centroids"], nprobe)
        # L5: the oracle on this shard with the GPU's q' and probes injected
        oi, od, _, tids, test = orc.search(Qn, ex["rotation"], ex["centroids"], ex["list_off"], ex["ids"],
                                           ex["codes"], ex["n_o"], ex["rho"], Xn[lo:hi], k, nprobe, M, SEED,
                                           id_offset=lo, qr_in=qr, probes_in=probes, debug=True)
        for q in range(nq):
            a, b = set(gt[q][gt[q] >= 0].tolist()), set(tids[q][tids[q] >= 0].tolist())
            if a == b:
                continue
            mth = float(test[q][np.isfinite(test[q])].max())
            nq2 = float((((qr[q][None] - ex["centroids"][probes[q]]) ** 2).sum(1)).max())
            band = 2 * pu.est_tol(float(ex["n_o"].max()), nq2)
            ge = dict(zip(gt[q].tolist(), gest[q].tolist()))
            oe = dict(zip(tids[q].tolist(), test[q].tolist()))
            for x in a - b:
                assert abs(ge[x] - mth) <= band, (g, q, x)
            for x in b - a:
                assert abs(oe[x] - mth) <= band, (g, q, x)
        # L6: the oracle's exact re-rank of the GPU's top-M (global ids -> slice rows)
        loc = np.where(gt >= 0, gt - lo, -1)
        ri, rd = orc.rerank(Qn, Xn[lo:hi], loc, k)
        ri = np.where(ri >= 0, ri + lo, -1)
        pu.check_final(ids, d, ri, rd, k)
        per_i.append(ids)
        per_d.append(d)
        orc_i.append(oi)
        orc_d.append(od)
    # merge: the GPU kernel vs the oracle's merge of the same inputs, bit-exact
    mi, md = rq.merge_topk(torch.from_numpy(np.stack(per_i)).cuda(), torch.from_numpy(np.stack(per_d)).cuda())
    ri, rd = orc.merge_topk(np.stack(per_i), np.stack(per_d))
    assert np.array_equal(mi.cpu().numpy(), ri) and np.array_equal(md.cpu().numpy(), rd)
    # vs the oracle's own sharded search (O-SH) on the exported shards: ties only
    oi, od = orc.merge_topk(np.stack(orc_i), np.stack(orc_d))
    pu.check_final(mi.cpu().numpy(), md.cpu().numpy(), oi, od, k)


def test_logical_shards_exhaustive_exact(orc):
    """nprobe = nlist and M >= N on every shard: the merged result is the exact
    kNN whatever G."""
    D, N, nlist, nq, k = 64, 6000, 12, 10, 10
    X, Q = make_data(D, N, nlist, nq, seed=5)
    gi, gd = orc.bruteforce(X.numpy(), Q.numpy(), k)
    for G in (1, 3):
        shards, _ = build_shards(X, nlist, G)
        outs = [sh.search(Q.cuda(), k, nlist, N) for sh in shards]
        mi, md = rq.merge_topk(torch.stack([o[0] for o in outs]), torch.stack([o[1] for o in outs]))
        pu.check_final(mi.cpu().numpy(), md.cpu().numpy(), gi, gd.astype(np.float32), k)


@pytest.mark.parametrize("D,N,nlist,nq,nprobe", [(128, 30000, 64, 300, 8), (96, 20000, 4096, 100, 64)])
def test_query_split_probe_composition(D, N, nlist, nq, nprobe):
    """Query-split probing: each of G ranks probes its slice of the queries
    (rabitq_probe), the slices are concatenated (the all-gather), and the
    search over probes_in equals the default search bit for bit; the probe
    lists equal the search's own S2-S3 output."""
    X, Q = make_data(D, N, min(nlist, 256), nq)
    idx = rq.Index(X.cuda(), nlist=nlist, seed=SEED)
    Qd = Q.cuda()
    base_i, base_d = idx.search(Qd, 10, nprobe, 100)
    own = torch.empty(nq, nprobe, dtype=torch.int32, device="cuda")
    idx.search(Qd, 10, nprobe, 100, debug=dict(probes=own))
    for G in (2, 4):
        c = (nq + G - 1) // G
        parts = [idx.probe(Qd[g * c:min(nq, (g + 1) * c)], nprobe) for g in range(G)]
        P = torch.cat(parts)
        assert torch.equal(P, own)
        si, sd = idx.search(Qd, 10, nprobe, 100, probes=P)
        assert torch.equal(si, base_i) and torch.equal(sd, base_d)
    # host probe lists are staged too; an out-of-range list id is rejected
    hi, hd = idx.search(Qd, 10, nprobe, 100, probes=own.cpu().numpy())
    assert torch.equal(hi, base_i) and torch.equal(hd, base_d)
    bad = own.clone()
    bad[3, 0] = nlist
    with pytest.raises(rq.RabitqError) as e:
        idx.search(Qd, 10, nprobe, 100, probes=bad)
    assert e.value.status == rq.ERR_INVALID_ARGUMENT


@pytest.mark.parametrize("query_split", [0, 1])
def test_nccl_one_rank_equals_single(query_split):
    """rabitq_search_sharded over a 1-rank NCCL communicator runs the real
    exchange code (ncclAllGather of the top-k, merge kernel; with query_split
    the probe all-gather too) and equals rabitq_search bit for bit."""
    X, Q = make_data(128, 20000, 48, 64)
    idx = rq.Index(X.cuda(), nlist=48, seed=SEED)
    comm = rq.Comm(rq.Comm.unique_id(), 0, 1, 0)
    try:
        a_i, a_d = idx.search(Q.cuda(), 10, 8, 100)
        b_i, b_d = comm.search_sharded(idx, Q.cuda(), 10, 8, 100, query_split=query_split)
        torch.cuda.synchronize()
        assert torch.equal(a_i, b_i) and torch.equal(a_d, b_d)
        h_i, h_d = comm.search_sharded(idx, Q, 10, 8, 100, query_split=query_split)  # host buffers
        assert torch.equal(h_i.cpu(), a_i.cpu()) and torch.equal(h_d.cpu(), a_d.cpu())
    finally:
        comm.free()
