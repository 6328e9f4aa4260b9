"""GPU (librabitq via the C ABI) vs the oracle, stage by stage (-m gpu).

Layered parity: L0 build, L1 probe, L2 quantizer (bit-exact under
injection of the GPU's q'), L3 integer inner products (bit-exact), L4
estimator (1e-4 n_q n_o + 2^-20 (n_o^2 + n_q^2)), L5 coarse top-M (set equal
except the tie band), L6 final top-k (oracle re-rank of the GPU's top-M:
identical except exact-distance ties), end to end, and invariances.
"""
import math

import numpy as np
import pytest
import torch

import synth
import parity_util as pu

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # the whole module needs a B200
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_16007_b200 as rq  # noqa: E402

SEED = 42


@pytest.fixture(scope="module")
def orc():
    import oracle

    oracle.build()
    return oracle


def make_data(D, N, ncent, nq, kind="iso", seed=7):
    s = synth.spec(1, D=D, N=N, ncent=ncent, nlist=ncent, nq=nq, kind=kind, data_seed=seed)
    cen = synth.centres(s, "cpu")
    X = synth.base_rows(s, 0, N, "cpu", cen=cen)
    Q = synth.queries(s, "cpu", cen=cen)
    return X, Q


def build(X, nlist, **kw):
    return rq.Index(X.cuda(), nlist=nlist, seed=SEED, **kw)


def debug_search(idx, Q, k, nprobe, M, dump=True, **kw):
    nq, D = Q.shape
    dev = "cuda"
    info = idx.info()
    dbg = dict(
        qrot=torch.empty(nq, D, device=dev), probes=torch.empty(nq, nprobe, dtype=torch.int32, device=dev),
        qbar=torch.empty(nq, nprobe, D, dtype=torch.uint8, device=dev),
        qscal=torch.empty(nq, nprobe, 4, device=dev), topm_ids=torch.empty(nq, M, dtype=torch.int64, device=dev),
        topm_est=torch.empty(nq, M, device=dev), topm_bound=torch.empty(nq, M, device=dev),
        tau=torch.empty(nq, device=dev), survivors=torch.empty(nq, dtype=torch.int32, device=dev),
        retries=torch.zeros(1, dtype=torch.int32, device=dev),
    )
    if dump:
        cap = nq * nprobe * ((info["max_list"] + 31) // 32) * 32
        dbg["scan_ip"] = torch.full((cap,), -1, dtype=torch.int32, device=dev)
        dbg["scan_est"] = torch.zeros(cap, device=dev)  # pad slots are never written
        dbg["scan_dump_cap"] = cap
    ids, d = idx.search(Q.cuda(), k, nprobe, M, debug=dbg, **kw)
    torch.cuda.synchronize()
    out = {k_: (v.cpu().numpy() if torch.is_tensor(v) else v) for k_, v in dbg.items()}
    return ids.cpu().numpy(), d.cpu().numpy(), out


# ----------------------------------------------------------------------------
@pytest.mark.parametrize("D,N,nlist", [(128, 20000, 64), (96, 12000, 40), (33, 5000, 16)])
def test_build_parity(orc, D, N, nlist):
    """L0: the exported lists partition the ids (ascending within a list), every
    vector sits in its nearest list (fp64, tie band), and the codes/factors
    equal the oracle's encode of the exported P and centroids."""
    X, _ = make_data(D, N, nlist, 4)
    idx = build(X, nlist)
    ex = idx.export()
    Xn = X.numpy()
    P, Cr, off, ids = ex["rotation"], ex["centroids"], ex["list_off"], ex["ids"]
    assert np.abs(P.astype(np.float64).T @ P.astype(np.float64) - np.eye(D)).max() <= 1e-5  # NS: P^T P = I
    assert off[0] == 0 and off[-1] == N
    assert np.array_equal(np.sort(ids), np.arange(N))
    assign = np.empty(N, np.int32)
    for j in range(nlist):
        seg = ids[off[j]:off[j + 1]]
        assert np.all(np.diff(seg) > 0)
        assign[seg] = j
    # nearest list (rotated space, fp64) up to fp32 near-ties
    Xr = orc.rotate(Xn, P)
    d = ((Xr[:, None, :] - Cr.astype(np.float64)[None]) ** 2).sum(-1) if N * nlist * D < 2e8 else None
    if d is not None:
        best = d.min(1)
        mine = d[np.arange(N), assign]
        assert np.all(mine <= best + 1e-4 * np.maximum(best, 1.0))
    codes, n_o, rho = orc.encode(Xn[ids], P, Cr, assign[ids])
    # The GPU forms r_o = x' - c' from an fp32 GEMM x' (P:L324 restructuring);
    # its rounding is ~ sqrt(D) eps32 ||x||, so a bit may differ only where the
    # fp64 residual is within that scale of 0.
    xs = np.linalg.norm(Xn[ids].astype(np.float64), axis=1)
    scale = 8 * math.sqrt(D) * 2.0 ** -24 * (xs + np.linalg.norm(Cr[assign[ids]].astype(np.float64), axis=1))
    diff = codes ^ ex["codes"]
    nflip = 0
    if diff.any():
        r = Xr[ids] - Cr[assign[ids]].astype(np.float64)
        rows, words = np.nonzero(diff)
        for v, w in zip(rows, words):
            bits = int(diff[v, w])
            for b in range(32):
                if bits >> b & 1:
                    i = 32 * w + b
                    assert abs(r[v, i]) <= scale[v], (v, i, r[v, i], scale[v])
                    nflip += 1
    assert nflip <= 1e-4 * N * D
    assert np.all(np.abs(ex["n_o"] - n_o) <= 1e-5 * n_o + math.sqrt(D) * scale)
    ok = n_o > 1e3 * scale  # rho of a residual at rounding-noise scale is itself noise (R#27)
    assert np.allclose(ex["rho"][ok], rho[ok], rtol=1e-5, atol=1e-6)


def _stage_checks(orc, idx, X, Q, k, nprobe, M, rank_key=0, scan_path=0):
    ex = idx.export()
    P, Cr, off, lids, codes = ex["rotation"], ex["centroids"], ex["list_off"], ex["ids"], ex["codes"]
    n_o, rho = ex["n_o"], ex["rho"]
    Qn, Xn = Q.numpy(), X.numpy()
    nq, D = Qn.shape
    ids, d, dbg = debug_search(idx, Q, k, nprobe, M, rank_key=rank_key, scan_path=scan_path)
    qr, probes, qbar, qscal = dbg["qrot"], dbg["probes"], dbg["qbar"], dbg["qscal"]
    # S1 rotation: q' = P^T q within fp32 GEMM rounding
    ref_qr = orc.rotate(Qn, P)
    assert np.abs(qr - ref_qr).max() <= 1e-5 * np.abs(ref_qr).max() + 1e-6
    # L1 probes (GPU q' injected)
    pu.check_probe_lists(probes, qr, Cr, nprobe)
    # L2 quantizer: bit-exact under injection
    nq2 = np.empty((nq, nprobe))
    for q in range(nq):
        for p in range(nprobe):
            j = int(probes[q, p])
            qb, vl, dl, sq, n2 = orc.quantize(qr[q], Cr[j], SEED, j, q)
            assert np.array_equal(qb, qbar[q, p]), (q, p)
            assert np.float32(vl) == qscal[q, p, 0] and np.float32(dl) == qscal[q, p, 1]
            assert sq == int(qscal[q, p, 3])
            assert abs(qscal[q, p, 2] - n2) <= 1e-5 * n2 + 1e-12
            nq2[q, p] = n2
    # L3 ip bit-exact + L4 est tolerance, every scanned (pair, slot)
    pair, lst, pos, valid, nitems = pu.list_pos_of_items(probes.reshape(-1), off)
    sip, sest = dbg["scan_ip"][: nitems * 32], dbg["scan_est"][: nitems * 32]
    assert np.all(sip[~valid] == -1)
    e = np.nonzero(valid)[0]
    row = off[lst[e]] + pos[e]
    qb_flat = qbar.reshape(nq * nprobe, D)
    W = codes.shape[1]
    checked = 0
    for t in range(e.size):
        p_ = pair[e[t]]
        ipv, pcv = orc.ip(codes[row[t]], qb_flat[p_], D)
        assert ipv == int(sip[e[t]]), (t, ipv, sip[e[t]])
        q_, pp = divmod(int(p_), nprobe)
        est, bd = orc.estimate(ipv, pcv, D, float(n_o[row[t]]), float(rho[row[t]]), float(qscal[q_, pp, 0]),
                               float(qscal[q_, pp, 1]), int(qscal[q_, pp, 3]), nq2[q_, pp])
        tol = pu.est_tol(float(n_o[row[t]]), nq2[q_, pp])
        assert abs(float(sest[e[t]]) - est) <= tol, (t, sest[e[t]], est, tol)
        checked += 1
    assert checked == e.size and checked > 0
    # L5 coarse top-M vs the oracle with the GPU's q' and probes injected
    oi, od, _, tids, test = orc.search(Qn, P, Cr, off, lids, codes, n_o, rho, Xn, k, nprobe, M, SEED,
                                       rank_key=rank_key, qr_in=qr, probes_in=probes, debug=True)
    gt = dbg["topm_ids"]
    row_of = {int(x): i for i, x in enumerate(lids)}

    def pair_est(q, x):  # oracle (est, bound, tolerance) of candidate id x for query q
        r = row_of[int(x)]
        j = int(np.searchsorted(off, r, side="right") - 1)
        p = int(np.nonzero(probes[q] == j)[0][0])
        ipv, pcv = orc.ip(codes[r], qbar[q, p], D)
        est, bd = orc.estimate(ipv, pcv, D, float(n_o[r]), float(rho[r]), float(qscal[q, p, 0]),
                               float(qscal[q, p, 1]), int(qscal[q, p, 3]), nq2[q, p])
        return est, bd, pu.est_tol(float(n_o[r]), nq2[q, p])

    for q in range(nq):
        # the GPU's fused error bound of every top-M candidate vs the oracle's (fp32 vs fp64)
        for i in np.nonzero(gt[q] >= 0)[0]:
            _, bd, _ = pair_est(q, gt[q][i])
            assert abs(float(dbg["topm_bound"][q][i]) - bd) <= 1e-5 * bd + 1e-6, (q, i, dbg["topm_bound"][q][i], bd)
        a, b = set(gt[q][gt[q] >= 0].tolist()), set(tids[q][tids[q] >= 0].tolist())
        if a == b:
            continue
        # L5 (R#18): a swapped id ties with the oracle's M-th key within the two pairs' own
        # estimator tolerances (each estimate is within its tolerance, L4)
        fin = np.isfinite(test[q])
        im = int(np.argmax(np.where(fin, test[q], -np.inf)))
        mth = float(test[q][im])
        tol_m = pair_est(q, tids[q][im])[2] * (2 if rank_key == 1 else 1)
        for x in a ^ b:
            est, bd, tol = pair_est(q, x)
            key = est - bd if rank_key == 1 else est
            band = tol * (2 if rank_key == 1 else 1) + tol_m
            assert abs(key - mth) <= band, (q, x, key, mth, band)
    # L6 final: the oracle's re-rank of the GPU's own top-M
    ri, rd = orc.rerank(Qn, Xn, gt, k)
    pu.check_final(ids, d, ri, rd, k)
    # end to end vs the injected oracle: identical except tie-explained slots
    return ids, d, oi, od, dbg


@pytest.mark.parametrize("scan_path", [rq.SCAN_POPC, rq.SCAN_IMMA])
@pytest.mark.parametrize("D,N,nlist,nq,nprobe,k,M", [
    (128, 20000, 64, 12, 8, 10, 100),     # CFG1 shape (W = 4)
    (96, 15000, 48, 10, 6, 10, 200),      # CFG3/CFG5 dim (W = 3)
    (960, 6000, 16, 4, 4, 100, 1000),     # CFG2 dim (W = 30), M > list sizes
    (33, 4000, 10, 8, 3, 5, 40),          # ragged W = 2 (generic path)
    (128, 30000, 8, 300, 5, 10, 100),     # many queries per list: multi-group, multi-tile
])
def test_stage_parity(orc, D, N, nlist, nq, nprobe, k, M, scan_path):
    X, Q = make_data(D, N, nlist, nq)
    idx = build(X, nlist)
    _stage_checks(orc, idx, X, Q, k, nprobe, M, scan_path=scan_path)


@pytest.mark.parametrize("nlist,nprobe,nq", [(2048, 300, 40), (4096, 64, 300), (16384, 128, 64)])
def test_probe_select_large_nlist(nlist, nprobe, nq):
    """Probe lists at large nlist (sampled-threshold select, search.cu
    probe_select_big_kernel): the oracle's ranking of the GPU's own q' (L1),
    and bit-identical to the radix select over the whole row."""
    X, Q = make_data(32, 4 * nlist, nlist, nq)
    idx = build(X, nlist)
    _, _, a = debug_search(idx, Q, 10, nprobe, 50, dump=False)
    pu.check_probe_lists(a["probes"], a["qrot"], idx.export()["centroids"], nprobe)
    _, _, b = debug_search(idx, Q, 10, nprobe, 50, dump=False, variant=rq.VARIANT_RADIX_PROBE)
    assert np.array_equal(a["probes"], b["probes"])


@pytest.mark.parametrize("scan_path", [rq.SCAN_POPC, rq.SCAN_IMMA])
def test_stage_parity_lower_bound_key(orc, scan_path):
    X, Q = make_data(128, 12000, 32, 8)
    idx = build(X, 32)
    _stage_checks(orc, idx, X, Q, 10, 6, 80, rank_key=1, scan_path=scan_path)


@pytest.mark.parametrize("D", [96, 128, 960])
def test_scan_paths_identical(D):
    """The bit-plane popc scan and the tcgen05 int8 scan give bit-identical
    results (exact integer ip, one estimator function): S:L352 invariance."""
    X, Q = make_data(D, 40000 if D < 900 else 8000, 32, 256)
    idx = build(X, 32)
    a_i, a_d = idx.search(Q.cuda(), 10, 8, 200, scan_path=rq.SCAN_POPC)
    b_i, b_d = idx.search(Q.cuda(), 10, 8, 200, scan_path=rq.SCAN_IMMA)
    assert torch.equal(a_i, b_i) and torch.equal(a_d, b_d)


@pytest.mark.parametrize("D", [96, 960])
def test_scan_code_operand_paths_identical(D):
    """The grouped scan's A operand from the expanded codes in HBM (TMA) and
    from the in-kernel expansion into TMEM (index built without the expanded
    copy) give bit-identical results, including the debug dump of every ip and
    estimate."""
    X, Q = make_data(D, 40000 if D < 900 else 8000, 32, 256)
    a = build(X, 32)
    assert a.info()["bytes_codes8"] > 0
    ai, ad, adbg = debug_search(a, Q[:64], 10, 8, 200, scan_path=rq.SCAN_IMMA)
    si, sd = a.search(Q.cuda(), 10, 8, 200, scan_path=rq.SCAN_IMMA)
    # the same index, codes expanded in the kernel
    bi, bd, bdbg = debug_search(a, Q[:64], 10, 8, 200, scan_path=rq.SCAN_IMMA, variant=rq.VARIANT_EXPAND_IN_KERNEL)
    ti, td = a.search(Q.cuda(), 10, 8, 200, scan_path=rq.SCAN_IMMA, variant=rq.VARIANT_EXPAND_IN_KERNEL)
    assert np.array_equal(ai, bi) and np.array_equal(ad, bd)
    assert np.array_equal(adbg["scan_ip"], bdbg["scan_ip"]) and np.array_equal(adbg["scan_est"], bdbg["scan_est"])
    assert torch.equal(si, ti) and torch.equal(sd, td)


@pytest.mark.parametrize("D,M", [(128, 100), (960, 400)])
def test_adaptive_rerank_parity(orc, D, M):
    """NEXT-4 (rerank = RERANK_BOUND): the GPU keeps exactly the top-M candidates
    with est - bound <= the k-th smallest est + bound, computed here in fp32
    from the GPU's own top-M capture (est, bound), and returns the oracle's
    re-rank of that set; the profile counts the kept candidates.  Against the
    oracle's independent adaptive search (fp64 decisions) the results agree
    except where a decision sits on the fp32/fp64 boundary."""
    X, Q = make_data(D, 20000 if D < 900 else 6000, 24, 32)
    idx = build(X, 24)
    k, nprobe = 10, 6
    _, _, dbg = debug_search(idx, Q, k, nprobe, M, dump=False)
    prof = rq.Profile()
    ai, ad = idx.search(Q.cuda(), k, nprobe, M, rerank=rq.RERANK_BOUND, profile=prof)
    ai, ad = ai.cpu().numpy(), ad.cpu().numpy()
    tids, test, tb = dbg["topm_ids"], dbg["topm_est"], dbg["topm_bound"]
    kept = np.full((Q.shape[0], M), -1, np.int64)
    total = 0
    for q in range(Q.shape[0]):
        v = tids[q] >= 0
        est, bnd = test[q][v].astype(np.float32), tb[q][v].astype(np.float32)
        ub, lb = est + bnd, est - bnd
        if v.sum() > k:
            tau = np.sort(ub)[k - 1]
            keep = lb <= tau
        else:
            keep = np.ones(v.sum(), bool)
        s = tids[q][v][keep]
        kept[q, :s.size] = s
        total += s.size
    assert prof.reranked == total
    ri, rd = orc.rerank(Q.numpy(), X.numpy(), kept, k)
    pu.check_final(ai, ad, ri, rd, k)
    ex = idx.export()
    oi, _ = orc.search(Q.numpy(), ex["rotation"], ex["centroids"], ex["list_off"], ex["ids"], ex["codes"],
                       ex["n_o"], ex["rho"], X.numpy(), k, nprobe, M, SEED, rerank_mode=1)
    agree = np.mean([len(set(a.tolist()) & set(b.tolist())) / k for a, b in zip(ai, oi)])
    assert agree >= 0.98, agree


@pytest.mark.parametrize("D,N,nlist,nq,nprobe,k,M", [
    (128, 20000, 64, 12, 8, 10, 100),
    (96, 15000, 48, 10, 6, 10, 200),
    (960, 6000, 16, 4, 4, 100, 1000),
    (33, 4000, 10, 8, 3, 5, 40),
])
def test_fullq_parity(orc, D, N, nlist, nq, nprobe, k, M):
    """NEXT-1 (query_bits = 32): every scanned estimate within the estimator
    tolerance of the oracle's exact-residual estimator (estimate_fullq, fp64,
    on the GPU's own q' and probes), the top-M equal to the oracle's qmode-1
    search except inside the tie band, and the final top-k = the oracle's
    re-rank of the GPU's top-M."""
    X, Q = make_data(D, N, nlist, nq)
    idx = build(X, nlist)
    ids, d, dbg = debug_search(idx, Q, k, nprobe, M, query_bits=32)
    ex = idx.export()
    Cr, off, lids, codes, n_o, rho = ex["centroids"], ex["list_off"], ex["ids"], ex["codes"], ex["n_o"], ex["rho"]
    qr, probes = dbg["qrot"], dbg["probes"]
    pu.check_probe_lists(probes, qr, Cr, nprobe)
    pair, lst, pos, valid, nitems = pu.list_pos_of_items(probes.reshape(-1), off)
    sest = dbg["scan_est"][: nitems * 32]
    e = np.nonzero(valid)[0]
    row = off[lst[e]] + pos[e]
    rng = np.random.default_rng(0)
    pick = e.size if e.size <= 20000 else 20000
    sel = rng.choice(e.size, size=pick, replace=False)
    for t_ in sel:
        p_ = int(pair[e[t_]])
        q_, pp = divmod(p_, nprobe)
        rq = qr[q_].astype(np.float64) - Cr[int(probes[q_, pp])].astype(np.float64)
        est, _ = orc.estimate_fullq(codes[row[t_]], rq, D, float(n_o[row[t_]]), float(rho[row[t_]]))
        tol = pu.est_tol(float(n_o[row[t_]]), float((rq * rq).sum()))
        assert abs(float(sest[e[t_]]) - est) <= tol, (t_, sest[e[t_]], est, tol)
    oi, od, _, tids, test = orc.search(Q.numpy(), ex["rotation"], Cr, off, lids, codes, n_o, rho, X.numpy(), k,
                                       nprobe, M, SEED, qr_in=qr, probes_in=probes, debug=True, qmode=1)
    gt = dbg["topm_ids"]
    for q in range(nq):
        a, b = set(gt[q][gt[q] >= 0].tolist()), set(tids[q][tids[q] >= 0].tolist())
        if a == b:
            continue
        mth = test[q][np.isfinite(test[q])].max()
        band = 2 * pu.EST_REL * float(np.sqrt(((qr[q][None] - Cr[probes[q]]) ** 2).sum(1)).max()) * float(n_o.max())
        for x in a ^ b:
            r_ = int(np.nonzero(lids == x)[0][0])
            j = int(np.searchsorted(off, r_, side="right") - 1)
            rq = qr[q].astype(np.float64) - Cr[j].astype(np.float64)
            est, _ = orc.estimate_fullq(codes[r_], rq, D, float(n_o[r_]), float(rho[r_]))
            assert abs(est - mth) <= band + 1e-6 * abs(mth), (q, x, est, mth, band)
    ri, rd = orc.rerank(Q.numpy(), X.numpy(), gt, k)
    pu.check_final(ids, d, ri, rd, k)


def _near_tau(idx, dbg, M, s_max=8192, nnear=32):
    """The near-list seed's tau where it is exact: the touched lists (nearest
    probes until >= M vectors) taken whole (<= s_max vectors) -> the M-th
    smallest dumped est over them; NaN where the seed samples or does not prune."""
    lo = idx.export()["list_off"]
    sizes = np.diff(lo)
    probes = dbg["probes"]
    ip, est = dbg["scan_ip"], dbg["scan_est"]
    out = np.full(probes.shape[0], np.nan)
    off = 0
    for q in range(probes.shape[0]):
        blk = [int((sizes[j] + 31) // 32) * 32 for j in probes[q]]
        cov, npr = 0, 0
        while npr < min(nnear, len(blk)) and cov < M:
            cov += int(sizes[probes[q][npr]])
            npr += 1
        P = int(sum(sizes[j] for j in probes[q]))
        if cov >= M and cov <= s_max and P > 2 * M:
            n = sum(blk[:npr])
            m = ip[off:off + n] >= 0
            out[q] = np.sort(est[off:off + n][m])[M - 1]
        off += sum(blk)
    return out


def _dump_counts(idx, dbg, nprobe, tau):
    """Per query: the scanned pairs with est <= tau, from the scan dump (pairs in
    query-major order, ceil(L / 32) 32-slot blocks each, ip = -1 on pad slots)."""
    lo = idx.export()["list_off"]
    sizes = np.diff(lo)
    probes = dbg["probes"]
    ip, est = dbg["scan_ip"], dbg["scan_est"]
    out = np.zeros(probes.shape[0], dtype=np.int64)
    off = 0
    for q in range(probes.shape[0]):
        n = int(sum((sizes[j] + 31) // 32 for j in probes[q])) * 32
        m = ip[off:off + n] >= 0
        out[q] = int(np.count_nonzero(est[off:off + n][m] <= tau[q]))
        off += n
    return out


@pytest.mark.parametrize("D,N,nlist,nq", [(128, 40000, 32, 300), (96, 60000, 24, 700), (33, 20000, 16, 200)])
def test_small_scan_identical(D, N, nlist, nq):
    """d <= 128: the folded small-K scan (survivor test on the tensor cores),
    the small-K scan with the CUDA-core test (VARIANT_NO_FOLD) and the generic
    grouped scan give bit-identical stage outputs: threshold, top-M ids and
    estimates, final ids and distances, with several query groups per list
    (nq * nprobe / nlist > 256) and ragged Dp (33 -> 64).  The two CUDA-core
    tests flag the same pairs (equal survivor counts); the folded test is
    conservative: it keeps every pair with est <= tau (counted from the scan
    dump) and few others.  The uniform-prefix threshold seed
    (VARIANT_UNIFORM_SEED) changes tau but not the results."""
    X, Q = make_data(D, N, nlist, nq)
    idx = build(X, nlist)
    nprobe = 12 if nlist >= 24 else 8
    a = debug_search(idx, Q, 10, nprobe, 200, scan_path=rq.SCAN_IMMA, dump=False)
    n = debug_search(idx, Q, 10, nprobe, 200, scan_path=rq.SCAN_IMMA, dump=False, variant=rq.VARIANT_NO_FOLD)
    b = debug_search(idx, Q, 10, nprobe, 200, scan_path=rq.SCAN_IMMA, dump=False, variant=rq.VARIANT_GENERIC_SCAN)
    for x in (n, b):
        assert np.array_equal(a[0], x[0]) and np.array_equal(a[1], x[1])
        for key in ("tau", "topm_ids", "topm_est"):
            assert np.array_equal(a[2][key], x[2][key]), key
    assert np.array_equal(n[2]["survivors"], b[2]["survivors"])
    # the dump runs the CUDA-core test; count the pairs the folded test must keep
    dmp = debug_search(idx, Q, 10, nprobe, 200, scan_path=rq.SCAN_IMMA)
    assert np.array_equal(dmp[2]["tau"], a[2]["tau"])
    # the near-list seed's keys are the scan's: where it takes the touched lists whole,
    # tau is exactly their M-th smallest est
    nt = _near_tau(idx, dmp[2], 200)
    ok = ~np.isnan(nt)
    assert ok.sum() > 0 and np.array_equal(a[2]["tau"][ok], nt[ok].astype(np.float32))
    need = _dump_counts(idx, dmp[2], nprobe, a[2]["tau"])
    assert np.all(a[2]["survivors"] >= need), "folded test dropped a pair with est <= tau"
    assert a[2]["survivors"].sum() <= need.sum() * 1.01 + 16 * nq
    # the folded scan defers its flagged pairs to a tail phase; with a 2-record region
    # nearly all of them take the region-full path instead: same keys, same counts
    fi = debug_search(idx, Q, 10, nprobe, 200, scan_path=rq.SCAN_IMMA, dump=False, variant=rq.VARIANT_FOLD_INPLACE)
    assert np.array_equal(a[0], fi[0]) and np.array_equal(a[1], fi[1])
    for key in ("tau", "topm_ids", "topm_est", "survivors"):
        assert np.array_equal(a[2][key], fi[2][key]), key
    u = debug_search(idx, Q, 10, nprobe, 200, scan_path=rq.SCAN_IMMA, dump=False, variant=rq.VARIANT_UNIFORM_SEED)
    assert np.array_equal(a[0], u[0]) and np.array_equal(a[1], u[1])
    assert np.array_equal(a[2]["topm_ids"], u[2]["topm_ids"])
    # without the dump and with the lower-bound key
    for kw in (dict(), dict(rank_key=rq.RANK_LOWER_BOUND)):
        si, sd = idx.search(Q.cuda(), 10, nprobe, 200, scan_path=rq.SCAN_IMMA, **kw)
        gi, gd = idx.search(Q.cuda(), 10, nprobe, 200, scan_path=rq.SCAN_IMMA, variant=rq.VARIANT_GENERIC_SCAN, **kw)
        assert torch.equal(si, gi) and torch.equal(sd, gd)


def test_scan_paths_identical_multigroup_d960():
    """D = 960 with > 160 queries per list: several query groups per list (the
    TMA-A kernel's 160-column groups) and several 8-tile items per group; the
    tensor-core scan must still equal the popc scan bit for bit."""
    X, Q = make_data(960, 24000, 8, 400)
    idx = build(X, 8)
    a_i, a_d = idx.search(Q.cuda(), 10, 4, 300, scan_path=rq.SCAN_POPC)
    b_i, b_d = idx.search(Q.cuda(), 10, 4, 300, scan_path=rq.SCAN_IMMA)
    assert torch.equal(a_i, b_i) and torch.equal(a_d, b_d)


def test_cfg1_end_to_end(orc):
    """CFG1 at full size (N = 1e5, D = 128, nlist 256, 100 queries, nprobe 16,
    k 10, M 100): GPU vs the oracle running the whole path independently (its
    own fp64 rotation and probing) on the exported index; recall vs exact kNN."""
    s = synth.spec(1)
    cen = synth.centres(s, "cpu")
    X = synth.base_rows(s, 0, s.N, "cpu", cen=cen)
    Q = synth.queries(s, "cpu", cen=cen)
    idx = build(X, s.nlist)
    ex = idx.export()
    ids, d = idx.search(Q.cuda(), s.k, s.nprobe, s.M)
    ids, d = ids.cpu().numpy(), d.cpu().numpy()
    oi, od = orc.search(Q.numpy(), ex["rotation"], ex["centroids"], ex["list_off"], ex["ids"], ex["codes"],
                        ex["n_o"], ex["rho"], X.numpy(), s.k, s.nprobe, s.M, SEED)
    same = np.mean([np.array_equal(a, b) for a, b in zip(ids, oi)])
    assert same >= 0.95, same
    gt, _ = orc.bruteforce(X.numpy(), Q.numpy(), s.k)
    rg, ro = pu.recall(ids, gt, s.k), pu.recall(oi, gt, s.k)
    assert abs(rg - ro) <= 0.01, (rg, ro)
    assert rg >= 0.85, rg
    # host-buffer (end-to-end) call path returns the same answer
    hi, hd = idx.search(Q, s.k, s.nprobe, s.M)
    assert np.array_equal(hi.numpy(), ids) and np.array_equal(hd.numpy(), d)


def test_exhaustive_is_exact_knn(orc):
    """nprobe = nlist and M >= N -> exact kNN."""
    X, Q = make_data(64, 3000, 12, 10)
    idx = build(X, 12)
    ids, d = idx.search(Q.cuda(), 10, 12, 3000)
    gi, gd = orc.bruteforce(X.numpy(), Q.numpy(), 10)
    pu.check_final(ids.cpu().numpy(), d.cpu().numpy(), gi, gd.astype(np.float32), 10)


def test_invariances(orc):
    """Results do not depend on batch split (query_id_base), survivor buffer
    size (forced overflow re-scans), threshold seeding size."""
    X, Q = make_data(128, 20000, 64, 40)
    idx = build(X, 64)
    Qd = Q.cuda()
    base_i, base_d = idx.search(Qd, 10, 8, 100)
    a_i, a_d = idx.search(Qd[:17], 10, 8, 100)
    b_i, b_d = idx.search(Qd[17:], 10, 8, 100, query_id_base=17)
    assert torch.equal(torch.cat([a_i, b_i]), base_i) and torch.equal(torch.cat([a_d, b_d]), base_d)
    retries = torch.zeros(1, dtype=torch.int32, device="cuda")
    c_i, c_d = idx.search(Qd, 10, 8, 100, cap=200, seed_max=100, debug=dict(retries=retries))
    assert torch.equal(c_i, base_i) and torch.equal(c_d, base_d)
    assert int(retries.item()) >= 1  # the overflow path ran
    s_i, s_d = idx.search(Qd, 10, 8, 100, seed_max=100)
    assert torch.equal(s_i, base_i) and torch.equal(s_d, base_d)
    # the tensor-core scan and its regrouped overflow re-scan give the same answer
    r2 = torch.zeros(1, dtype=torch.int32, device="cuda")
    t_i, t_d = idx.search(Qd, 10, 8, 100, cap=200, seed_max=100, scan_path=rq.SCAN_IMMA, debug=dict(retries=r2))
    assert torch.equal(t_i, base_i) and torch.equal(t_d, base_d)
    assert int(r2.item()) >= 1


def test_edge_cases():
    X, Q = make_data(32, 500, 50, 6)
    idx = build(X, 50)
    # nq = 0
    i0, d0 = idx.search(Q[:0].cuda(), 5, 3, 10)
    assert i0.shape == (0, 5)
    # fewer candidates than k -> (-1, +inf) padding
    ids, d = idx.search(Q.cuda(), 64, 1, 64)
    ids, d = ids.cpu().numpy(), d.cpu().numpy()
    for q in range(6):
        n = int((ids[q] >= 0).sum())
        assert np.all(ids[q, n:] == -1) and np.all(np.isinf(d[q, n:])) and np.all(np.isfinite(d[q, :n]))
    # errors
    with pytest.raises(rq.RabitqError) as e:
        idx.search(Q.cuda(), 0, 3, 10)
    assert e.value.status == rq.ERR_INVALID_ARGUMENT
    with pytest.raises(rq.RabitqError):
        idx.search(Q.cuda(), 10, 3, 5)  # n_rerank < k
    with pytest.raises(rq.RabitqError):
        idx.search(Q.cuda(), 10, 51, 20)  # nprobe > nlist
    bad = Q.clone()
    bad[2, 3] = float("nan")
    with pytest.raises(rq.RabitqError) as e:
        idx.search(bad.cuda(), 5, 3, 10)
    assert e.value.status == rq.ERR_INVALID_DATA
    # >= 256 queries: the side-stream dense re-rank block is in flight when the
    # error is raised; the workspace it reads must outlive it (no corruption of
    # the next searches)
    _, Qbig = make_data(32, 500, 50, 400)
    ref_i, ref_d = idx.search(Qbig.cuda(), 5, 3, 10)
    badbig = Qbig.clone()
    badbig[300, 1] = float("inf")
    for _ in range(3):
        with pytest.raises(rq.RabitqError) as e:
            idx.search(badbig.cuda(), 5, 3, 10)
        assert e.value.status == rq.ERR_INVALID_DATA
        again_i, again_d = idx.search(Qbig.cuda(), 5, 3, 10)
        assert torch.equal(again_i, ref_i) and torch.equal(again_d, ref_d)
    Xb = X.clone()
    Xb[0, 0] = float("inf")
    with pytest.raises(rq.RabitqError) as e:
        rq.Index(Xb.cuda(), nlist=10)
    assert e.value.status == rq.ERR_INVALID_DATA
    with pytest.raises(rq.RabitqError):
        rq.Index(X[:5].cuda(), nlist=10)  # n < nlist


@pytest.mark.parametrize("scan_path", [rq.SCAN_POPC, rq.SCAN_IMMA])
def test_degenerate_inputs(orc, scan_path):
    """Degenerate cases of the method on the GPU vs the oracle (ledger R#9,
    R#10, R#17, R#22): a far outlier forms a singleton list, so its vector
    equals its centroid (n_o = 0, rho := 1); a query placed on that centroid has
    a constant (zero) residual (Delta = 0, every qbar = 0); exact duplicates give
    exact distance ties, broken by ascending id; every stage checked."""
    X, Q = make_data(64, 6000, 16, 6, seed=3)
    X = X.clone()
    X[100] = 400.0                      # outlier: its own list
    X[2000:2010] = X[50]                # 11 identical vectors (ids 50, 2000..2009)
    Q = Q.clone()
    Q[0] = X[100]                       # on the singleton centroid
    Q[1] = X[50] + 0.01                 # next to the duplicates
    # k-means seeded with the outlier as its own centroid, every row in training:
    # its cluster stays a singleton (centroid = the point itself)
    C0 = torch.cat([X[torch.arange(16) * 300 + 7], X[100:101]])
    idx = build(X, 17, init_centroids=C0, train_size=6000)
    ex = idx.export()
    r = int(np.nonzero(ex["ids"] == 100)[0][0])
    assert ex["n_o"][r] == 0.0 and ex["rho"][r] == 1.0
    ids, d, _, _, dbg = _stage_checks(orc, idx, X, Q, 10, 4, 40, scan_path=scan_path)
    if dbg["qscal"][0, 0, 1] == 0.0:  # the rotated residual is exactly 0 (both GEMMs agree)
        assert np.all(dbg["qbar"][0, 0] == 0)
    assert ids[0, 0] == 100 and d[0, 0] == 0.0
    dup = [50] + list(range(2000, 2010))
    assert ids[1].tolist() == dup[:10]  # equal distances, ascending ids
    assert np.all(d[1] == d[1, 0])


def test_one_dimension(orc):
    """D = 1 (W = 1, Dp = 32): the estimator is exact (SURVEY pins), so the
    search equals exact kNN over the probed lists; every stage vs the oracle."""
    X, Q = make_data(1, 3000, 8, 10, seed=9)
    idx = build(X, 8)
    _stage_checks(orc, idx, X, Q, 5, 3, 20)


@pytest.mark.parametrize("D,N,nlist,nq,scan_path", [(128, 20000, 64, 64, rq.SCAN_IMMA), (960, 8000, 32, 64, rq.SCAN_AUTO),
                                                   (128, 20000, 64, 100, rq.SCAN_POPC)])
def test_graph_latency_mode(D, N, nlist, nq, scan_path):
    """NEXT-2 latency mode (graph = 1): the batch captured once as a CUDA graph
    (no host synchronisation inside, sizes from host-side bounds) and replayed
    gives bit-identical results to the normal path, on repeated calls (graph
    reuse), with host buffers, and when survivor buffers overflow (the batch is
    re-run on the normal path); non-finite queries still raise."""
    X, Q = make_data(D, N, nlist, nq)
    idx = build(X, nlist)
    Qd = Q.cuda()
    base_i, base_d = idx.search(Qd, 10, 8, 100, scan_path=scan_path)
    for _ in range(3):
        g_i, g_d = idx.search(Qd, 10, 8, 100, scan_path=scan_path, graph=1)
        assert torch.equal(g_i, base_i) and torch.equal(g_d, base_d)
    h_i, h_d = idx.search(Q, 10, 8, 100, scan_path=scan_path, graph=1)
    assert torch.equal(h_i, base_i.cpu()) and torch.equal(h_d, base_d.cpu())
    # other queries through the same graph (same shape)
    Q2 = Qd.flip(0).contiguous()
    r_i, r_d = idx.search(Q2, 10, 8, 100, scan_path=scan_path)
    g_i, g_d = idx.search(Q2, 10, 8, 100, scan_path=scan_path, graph=1)
    assert torch.equal(g_i, r_i) and torch.equal(g_d, r_d)
    # overflowing survivor buffers: the graph flags the batch, the normal path re-runs it
    o_i, o_d = idx.search(Qd, 10, 8, 100, scan_path=scan_path, cap=200, seed_max=100, graph=1)
    assert torch.equal(o_i, base_i) and torch.equal(o_d, base_d)
    bad = Q.clone()
    bad[5, 0] = float("nan")
    with pytest.raises(rq.RabitqError) as e:
        idx.search(bad.cuda(), 10, 8, 100, scan_path=scan_path, graph=1)
    assert e.value.status == rq.ERR_INVALID_DATA


def test_merge_topk_kernel(orc):
    rng = np.random.default_rng(3)
    G, nq, k = 4, 9, 10
    ids = rng.permutation(100000)[: G * nq * k].reshape(G, nq, k).astype(np.int64)
    d = np.sort(rng.integers(0, 30, (G, nq, k)).astype(np.float32), -1)
    oi, od = rq.merge_topk(torch.from_numpy(ids).cuda(), torch.from_numpy(d).cuda())
    ri, rd = orc.merge_topk(ids, d)
    assert np.array_equal(oi.cpu().numpy(), ri) and np.array_equal(od.cpu().numpy(), rd)


def test_borrow_and_shard_offsets(orc):
    """A shard built over a contiguous id slice (id_offset, shared P and
    centroids) returns global ids; borrowed vectors re-rank identically."""
    X, Q = make_data(64, 8000, 20, 6)
    full = build(X, 20)
    ex = full.export()
    Xd = X.cuda()
    lo, hi = 3000, 8000
    shard = rq.Index(Xd[lo:hi], nlist=20, seed=SEED, id_offset=lo, rotation=ex["rotation"],
                     centroids_rot=ex["centroids"], borrow=True)
    ids, d = shard.search(Q.cuda(), 10, 20, 5000)
    ids = ids.cpu().numpy()
    assert ids.min() >= lo and ids.max() < hi
    gi, gd = orc.bruteforce(X.numpy()[lo:hi], Q.numpy(), 10)
    pu.check_final(ids, d.cpu().numpy(), gi + lo, gd.astype(np.float32), 10)


def test_selftest_reciprocal_division():
    """The quantizer divides with a per-pair reciprocal (Markstein correction);
    R#11 pins t = fl((r - v_l) / Delta) to the IEEE quotient, so the two must be
    bit-identical on the quantizer's domain and on arbitrary normal operands."""
    assert rq.selftest(1, 1 << 28, seed=7) == 0
    assert rq.selftest(1, 1 << 26, seed=12345) == 0
    with pytest.raises(rq.RabitqError):
        rq.selftest(99, 1)
