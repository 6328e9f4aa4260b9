"""CPU oracle of the IVF-RaBitQ search hot path (arxiv 2605.16007).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2605_16007_b200``) never imports it and
shares no code with it.  The arithmetic lives in ``oracle.c`` (plain C, fp64,
OpenMP); this module only marshals numpy arrays through ctypes.

Parity status: every function is pinned by ``tests/test_oracle_*.py`` except the
exact centroids of ``kmeans`` ("parity unpinned": float summation order; only
its invariants are checked).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

EPS0 = 1.9  # DESIGN.md R#14


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (plain gcc, fp-contract off)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        cmd = [
            "gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp",
            "-ffp-contract=off", "-fno-fast-math", "-o", _SO, src, "-lm",
        ]
        subprocess.check_call(cmd, cwd=_HERE)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_SO)
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def philox(key, ctr):
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    o = (ctypes.c_uint32 * 4)()
    lib().oracle_philox4x32_10(k, c, o)
    return [int(x) for x in o]


def haar_rotation(D: int, seed: int):
    P64 = np.empty((D, D), np.float64)
    P32 = np.empty((D, D), np.float32)
    rc = lib().oracle_haar_rotation(ctypes.c_int(D), ctypes.c_uint64(seed), _p(P64), _p(P32))
    if rc != 0:
        raise ValueError("haar_rotation failed")
    return P64, P32


def rotate(X, P):
    X = _c(X, np.float32)
    P = _c(P, np.float32)
    n, D = X.shape
    out = np.empty((n, D), np.float64)
    lib().oracle_rotate(_p(X), ctypes.c_int64(n), ctypes.c_int(D), _p(P), _p(out))
    return out


def kmeans(T, nlist, init_rows=None, init_centroids=None, max_iter=25):
    T = _c(T, np.float32)
    nt, D = T.shape
    C = np.empty((nlist, D), np.float64)
    trace = np.full(max_iter, np.nan)
    ir = None if init_rows is None else _c(init_rows, np.int64)
    ic = None if init_centroids is None else _c(init_centroids, np.float32)
    it = lib().oracle_kmeans(_p(T), ctypes.c_int64(nt), ctypes.c_int(D), ctypes.c_int(nlist),
                             _p(ir), _p(ic), ctypes.c_int(max_iter), _p(C), _p(trace))
    if it < 0:
        raise ValueError("kmeans: bad arguments")
    return C, it, trace[:it]


def assign(X, C):
    X = _c(X, np.float32)
    C = _c(C, np.float64)
    n, D = X.shape
    a = np.empty(n, np.int32)
    lib().oracle_assign(_p(X), ctypes.c_int64(n), ctypes.c_int(D), _p(C), ctypes.c_int(C.shape[0]), _p(a))
    return a


def encode(X, P, Cr, assign_):
    X = _c(X, np.float32)
    P = _c(P, np.float32)
    Cr = _c(Cr, np.float32)
    a = _c(assign_, np.int32)
    n, D = X.shape
    W = (D + 31) // 32
    codes = np.empty((n, W), np.uint32)
    n_o = np.empty(n, np.float32)
    rho = np.empty(n, np.float32)
    lib().oracle_encode(_p(X), ctypes.c_int64(n), ctypes.c_int(D), _p(P), _p(Cr), _p(a), _p(codes),
                        _p(n_o), _p(rho))
    return codes, n_o, rho


def probe(qr, Cr, nprobe):
    qr = _c(qr, np.float32)
    Cr = _c(Cr, np.float32)
    out = np.empty(nprobe, np.int32)
    lib().oracle_probe(_p(qr), ctypes.c_int(qr.shape[0]), _p(Cr), ctypes.c_int(Cr.shape[0]),
                       ctypes.c_int(nprobe), _p(out))
    return out


def quantize(qr, cr, seed, list_id, qglobal):
    """Returns (qbar uint8[D], v_l, delta, S_q, nq2)."""
    qr = _c(qr, np.float32)
    cr = _c(cr, np.float32)
    D = qr.shape[0]
    qbar = np.empty(D, np.uint8)
    vl = ctypes.c_float()
    dl = ctypes.c_float()
    sq = ctypes.c_int32()
    nq2 = ctypes.c_double()
    lib().oracle_quantize(_p(qr), _p(cr), ctypes.c_int(D), ctypes.c_uint64(seed), ctypes.c_int32(list_id),
                          ctypes.c_int64(qglobal), _p(qbar), ctypes.byref(vl), ctypes.byref(dl),
                          ctypes.byref(sq), ctypes.byref(nq2))
    return qbar, vl.value, dl.value, sq.value, nq2.value


def ip(code, qbar, D):
    code = _c(code, np.uint32)
    qbar = _c(qbar, np.uint8)
    pc = ctypes.c_int64()
    v = lib().oracle_ip  # returns int64
    v.restype = ctypes.c_int64
    r = v(_p(code), _p(qbar), ctypes.c_int(D), ctypes.byref(pc))
    return int(r), int(pc.value)


def estimate(ip_, pc, D, n_o, rho, v_l, delta, S_q, nq2, eps0=EPS0):
    est = ctypes.c_double()
    bd = ctypes.c_double()
    lib().oracle_estimate(ctypes.c_int64(ip_), ctypes.c_int64(pc), ctypes.c_int(D), ctypes.c_double(n_o),
                          ctypes.c_double(rho), ctypes.c_double(v_l), ctypes.c_double(delta),
                          ctypes.c_int64(S_q), ctypes.c_double(nq2), ctypes.c_double(eps0),
                          ctypes.byref(est), ctypes.byref(bd))
    return est.value, bd.value


def estimate_fullq(code, rq, D, n_o, rho, eps0=EPS0):
    code = _c(code, np.uint32)
    rq = _c(rq, np.float64)
    est = ctypes.c_double()
    bd = ctypes.c_double()
    lib().oracle_estimate_fullq(_p(code), _p(rq), ctypes.c_int(D), ctypes.c_double(n_o),
                                ctypes.c_double(rho), ctypes.c_double(eps0), ctypes.byref(est),
                                ctypes.byref(bd))
    return est.value, bd.value


def search(Q, P, Cr, list_off, list_ids, codes, n_o, rho, X, k, nprobe, M, seed, qid_base=0,
           id_offset=0, rank_key=0, eps0=EPS0, qr_in=None, probes_in=None, num_threads=0,
           debug=False, rerank_mode=0, n_reranked=None, qmode=0):
    """Full oracle search (O-S1..O-S6; qmode 1: the unquantized query, NEXT-1;
    rerank_mode 1 adds O-S5b, the
    bound-driven re-rank set of SURVEY 8(f) NEXT-4).  Returns (ids, dists) or,
    with debug, (ids, dists, probes, topm_ids, topm_est).  n_reranked: optional
    int64 [nq] array receiving the number of candidates re-ranked per query."""
    Q = _c(Q, np.float32)
    nq, D = Q.shape
    nlist = Cr.shape[0]
    ids = np.empty((nq, k), np.int64)
    dists = np.empty((nq, k), np.float32)
    probes = np.empty((nq, nprobe), np.int32) if debug else None
    tids = np.empty((nq, M), np.int64) if debug else None
    test = np.empty((nq, M), np.float64) if debug else None
    args = [
        _p(Q), ctypes.c_int64(nq), ctypes.c_int(D), _p(_c(P, np.float32)), _p(_c(Cr, np.float32)),
        ctypes.c_int(nlist), _p(_c(list_off, np.int64)), _p(_c(list_ids, np.int64)),
        _p(_c(codes, np.uint32)), _p(_c(n_o, np.float32)), _p(_c(rho, np.float32)),
        _p(_c(X, np.float32)), ctypes.c_int64(id_offset), ctypes.c_int(k), ctypes.c_int(nprobe),
        ctypes.c_int(M), ctypes.c_uint64(seed), ctypes.c_int64(qid_base), ctypes.c_int(rank_key),
        ctypes.c_double(eps0),
        _p(None if qr_in is None else _c(qr_in, np.float32)),
        _p(None if probes_in is None else _c(probes_in, np.int32)),
        ctypes.c_int(num_threads), _p(ids), _p(dists), _p(probes), _p(tids), _p(test),
        ctypes.c_int(rerank_mode), _p(n_reranked), ctypes.c_int(qmode),
    ]
    # keep temporaries alive for the duration of the call
    keep = [a for a in args]
    rc = lib().oracle_search(*keep)
    if rc != 0:
        raise ValueError("oracle_search: bad arguments")
    if debug:
        return ids, dists, probes, tids, test
    return ids, dists


def rerank(Q, X, cand, k, id_offset=0):
    Q = _c(Q, np.float32)
    X = _c(X, np.float32)
    cand = _c(cand, np.int64)
    nq, D = Q.shape
    M = cand.shape[1]
    ids = np.empty((nq, k), np.int64)
    d = np.empty((nq, k), np.float32)
    lib().oracle_rerank(_p(Q), ctypes.c_int64(nq), ctypes.c_int(D), _p(X), ctypes.c_int64(id_offset), _p(cand),
                        ctypes.c_int(M), ctypes.c_int(k), _p(ids), _p(d))
    return ids, d


def merge_topk(in_ids, in_d):
    in_ids = _c(in_ids, np.int64)
    in_d = _c(in_d, np.float32)
    G, nq, k = in_ids.shape
    oi = np.empty((nq, k), np.int64)
    od = np.empty((nq, k), np.float32)
    lib().oracle_merge_topk(_p(in_ids), _p(in_d), ctypes.c_int(G), ctypes.c_int64(nq), ctypes.c_int(k),
                            _p(oi), _p(od))
    return oi, od


def bruteforce(X, Q, k, num_threads=0):
    X = _c(X, np.float32)
    Q = _c(Q, np.float32)
    n, D = X.shape
    nq = Q.shape[0]
    ids = np.empty((nq, k), np.int64)
    d = np.empty((nq, k), np.float64)
    lib().oracle_bruteforce(_p(X), ctypes.c_int64(n), ctypes.c_int(D), _p(Q), ctypes.c_int64(nq),
                            ctypes.c_int(k), ctypes.c_int(num_threads), _p(ids), _p(d))
    return ids, d


# --------------------------------------------------------------------------
# Index construction in the oracle's own (independent) mode, from raw X.
# --------------------------------------------------------------------------
class OracleIndex:
    """An IVF-RaBitQ index built entirely by the oracle (independent mode)."""

    def __init__(self, X, nlist, seed, max_iter=25, train_rows=None, init_rows=None,
                 init_centroids=None):
        X = _c(X, np.float32)
        n, D = X.shape
        self.D, self.n, self.nlist, self.seed = D, n, nlist, seed
        self.P64, self.P = haar_rotation(D, seed)
        rng = np.random.default_rng(seed)
        if train_rows is None:
            ts = min(n, 256 * nlist)
            train_rows = np.sort(rng.choice(n, size=ts, replace=False)) if ts < n else np.arange(n)
        T = X[train_rows]
        if init_centroids is None and init_rows is None:
            init_rows = rng.choice(T.shape[0], size=nlist, replace=False)
        C, self.iters, self.obj_trace = kmeans(T, nlist, init_rows=init_rows,
                                               init_centroids=init_centroids, max_iter=max_iter)
        self.C = C
        # c' = P^T c, stored in fp32 (the index stores rotated centroids, R#4, R#6)
        self.Cr = (C @ self.P.astype(np.float64)).astype(np.float32)
        self.assign = assign(X, C)
        codes, n_o, rho = encode(X, self.P, self.Cr, self.assign)
        order = np.argsort(self.assign, kind="stable")  # ids ascending within each list
        counts = np.bincount(self.assign, minlength=nlist)
        self.list_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.list_ids = order.astype(np.int64)
        self.codes = codes[order]
        self.n_o = n_o[order]
        self.rho = rho[order]
        self.X = X

    def search(self, Q, k, nprobe, M, seed=None, **kw):
        return search(Q, self.P, self.Cr, self.list_off, self.list_ids, self.codes, self.n_o,
                      self.rho, self.X, k, nprobe, M, self.seed if seed is None else seed, **kw)
