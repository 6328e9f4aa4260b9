"""Pins of the oracle (oracle/) against what the paper and mathematics fix.

Each test names the passage or identity it pins (P:Lnnn = PAPER.md line; NS =
BASELINE.json north_star; R#n = DESIGN.md reading).  None of these re-types the
oracle's own formula: they use worked examples, closed forms, special cases,
identities checked by a different algorithm, library routines and brute force.
"""
import ctypes
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --------------------------------------------------------------------------
# Philox4x32-10 (NS(2) "counter-based (Philox, seeded)")
# --------------------------------------------------------------------------
def test_philox_known_answers(orc):
    """Random123 KAT vectors + libcurand blocks (tests/golden/philox_kat.txt)."""
    n = 0
    for line in open(os.path.join(GOLDEN, "philox_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(t, 16) for t in line.split()]
        ctr, key, out = w[0:4], w[4:6], w[6:10]
        assert orc.philox(key, ctr) == out
        n += 1
    assert n == 5


def _curand():
    for p in ("/usr/local/cuda/lib64/libcurand.so",):
        if os.path.exists(p):
            try:
                return ctypes.CDLL(p)
            except OSError:
                return None
    return None


def test_philox_matches_libcurand(orc):
    """Independent implementation: curand's host Philox4_32_10 generator emits
    Philox(ctr=(0,0,b,0), key=(seed_lo, seed_hi)) for block b."""
    cur = _curand()
    if cur is None:
        pytest.skip("libcurand not present")
    for seed in (0, 1, 0x0123456789ABCDEF, 0xDEADBEEFCAFEF00D):
        gen = ctypes.c_void_p()
        assert cur.curandCreateGeneratorHost(ctypes.byref(gen), 161) == 0
        assert cur.curandSetPseudoRandomGeneratorSeed(gen, ctypes.c_ulonglong(seed)) == 0
        buf = (ctypes.c_uint32 * 64)()
        assert cur.curandGenerate(gen, buf, 64) == 0
        cur.curandDestroyGenerator(gen)
        key = [seed & 0xFFFFFFFF, seed >> 32]
        for b in range(16):
            assert orc.philox(key, [0, 0, b, 0]) == list(buf[4 * b:4 * b + 4])


# --------------------------------------------------------------------------
# Rotation P ("random orthogonal rotation"; NS "P^T P = I to 1e-5")
# --------------------------------------------------------------------------
@pytest.mark.parametrize("D", [1, 2, 31, 96, 128, 960])
def test_rotation_orthogonal(orc, D):
    P64, P32 = orc.haar_rotation(D, 42)
    G = P32.astype(np.float64).T @ P32.astype(np.float64)
    assert np.abs(G - np.eye(D)).max() <= 1e-5
    # deterministic for a fixed seed
    _, P32b = orc.haar_rotation(D, 42)
    assert np.array_equal(P32, P32b)
    if D == 1:
        assert abs(P32[0, 0]) == 1.0


def test_rotation_preserves_norms(orc):
    """P:L324 'rotation does not change vector norms' (oracle_rotate)."""
    D = 128
    _, P = orc.haar_rotation(D, 7)
    X = np.random.default_rng(0).standard_normal((200, D)).astype(np.float32)
    Xr = orc.rotate(X, P)
    rel = np.abs(np.linalg.norm(Xr, axis=1) / np.linalg.norm(X.astype(np.float64), axis=1) - 1)
    assert rel.max() < 1e-5
    # x' = P^T x: rotating by P = I is the identity
    assert np.array_equal(orc.rotate(X, np.eye(D, dtype=np.float32)), X.astype(np.float64))


def test_rotation_is_haar(orc):
    """Haar-distributed orthogonal matrices have E[tr Q] = 0 and E[tr(Q)^2] = 1
    (Diaconis-Shahshahani); a missing diag(R) sign fix biases both."""
    D, S = 12, 600
    tr = np.array([np.trace(orc.haar_rotation(D, 1000 + s)[0]) for s in range(S)])
    assert abs(tr.mean()) < 4 / math.sqrt(S)
    assert abs((tr ** 2).mean() - 1.0) < 0.25
    # each entry has variance 1/D
    e = np.array([orc.haar_rotation(D, 5000 + s)[0][3, 5] for s in range(S)])
    assert abs((e ** 2).mean() * D - 1.0) < 0.2


# --------------------------------------------------------------------------
# k-means (R#6) -- invariants only (parity unpinned)
# --------------------------------------------------------------------------
def test_kmeans_invariants(orc):
    rng = np.random.default_rng(1)
    mu = rng.standard_normal((8, 16)) * 4
    T = (mu[rng.integers(0, 8, 2000)] + rng.standard_normal((2000, 16))).astype(np.float32)
    C, it, trace = orc.kmeans(T, 8, init_rows=rng.choice(2000, 8, replace=False), max_iter=25)
    assert it >= 1
    assert np.all(np.diff(trace) <= 1e-9 * trace[0])  # objective non-increasing
    # assignment optimality: each point's centroid is its nearest (numpy, direct subtraction)
    a = orc.assign(T, C)
    d = ((T[:, None, :].astype(np.float64) - C[None]) ** 2).sum(-1)
    assert np.array_equal(a, d.argmin(1))


def test_kmeans_fixed_point(orc):
    """k distinct points with nlist = k converge to those points."""
    T = np.array([[0, 0], [10, 0], [0, 10], [10, 10]], np.float32)
    C, it, _ = orc.kmeans(T, 4, init_rows=np.array([2, 0, 3, 1]), max_iter=25)
    assert it <= 2
    assert sorted(map(tuple, C.tolist())) == sorted(map(tuple, T.astype(np.float64).tolist()))


def test_kmeans_two_blobs(orc):
    rng = np.random.default_rng(3)
    A = rng.standard_normal((100, 2)) * 0.3 + np.array([-5.0, 0.0])
    B = rng.standard_normal((100, 2)) * 0.3 + np.array([5.0, 1.0])
    T = np.concatenate([A, B]).astype(np.float32)
    C, _, _ = orc.kmeans(T, 2, init_rows=np.array([0, 1]), max_iter=25)
    means = sorted([tuple(T[:100].astype(np.float64).mean(0)), tuple(T[100:].astype(np.float64).mean(0))])
    got = sorted(map(tuple, C.tolist()))
    assert np.allclose(got, means, atol=1e-9)


def test_kmeans_empty_cluster_reseed(orc):
    """An empty cluster is re-seeded from the farthest point (R#6)."""
    T = np.array([[0, 0], [0.1, 0], [0, 0.1], [50, 50]], np.float32)
    init = np.array([[0, 0], [1000, 1000]], np.float32)  # cluster 1 starts empty
    C, _, _ = orc.kmeans(T, 2, init_centroids=init, max_iter=10)
    assert np.allclose(sorted(map(tuple, C.tolist()))[1], (50, 50))


# --------------------------------------------------------------------------
# Encode (Eq. 1; NS factors ||o_r - c||, <obar, o>)
# --------------------------------------------------------------------------
def test_encode_worked_example(orc):
    rows = [l.split() for l in open(os.path.join(GOLDEN, "encode_example.txt")) if not l.startswith("#")]
    rows = [r for r in rows if r]
    X = np.array([[float(r[0]), float(r[1])] for r in rows], np.float32)
    codes, n_o, rho = orc.encode(X, np.eye(2, dtype=np.float32), np.zeros((1, 2), np.float32),
                                 np.zeros(len(rows), np.int32))
    for i, r in enumerate(rows):
        assert int(codes[i, 0]) == int(r[2])
        assert n_o[i] == np.float32(float(r[3]))
        assert rho[i] == np.float32(float(r[4]))


def test_encode_properties(orc):
    """Norm invariance gives n_o = ||x - c|| in the original space;
    rho in [1/sqrt(D), 1]; negating the residual flips every bit;
    a vector equal to its centroid has n_o = 0, rho = 1, all bits 1 (R#7, R#9)."""
    D, n = 96, 500
    rng = np.random.default_rng(5)
    _, P = orc.haar_rotation(D, 11)
    c = rng.standard_normal(D)
    Cr = (c @ P.astype(np.float64)).astype(np.float32)  # c' = P^T c
    c_back = P.astype(np.float64) @ Cr.astype(np.float64)  # c = P c'
    X = (c_back + rng.standard_normal((n, D))).astype(np.float32)
    codes, n_o, rho = orc.encode(X, P, Cr[None], np.zeros(n, np.int32))
    ref = np.linalg.norm(X.astype(np.float64) - c_back, axis=1)
    assert np.allclose(n_o, ref, rtol=1e-5)
    assert np.all(rho >= 1 / math.sqrt(D) - 1e-6) and np.all(rho <= 1 + 1e-6)
    # mirrored vectors x2 = 2c - x have residual -r: every bit flips unless r_i == 0
    X2 = (2 * c_back - X.astype(np.float64)).astype(np.float32)
    codes2, n2, _ = orc.encode(X2, P, Cr[None], np.zeros(n, np.int32))
    Xr1 = orc.rotate(X, P) - Cr.astype(np.float64)
    safe = (np.abs(Xr1) > 1e-4).all(1)
    W = (D + 31) // 32
    mask = [(1 << 32) - 1] * (D // 32) + ([(1 << (D % 32)) - 1] if D % 32 else [])
    for v in np.nonzero(safe)[0]:
        for w in range(W):
            assert int(codes[v, w]) ^ int(codes2[v, w]) == mask[w]
    # x == c exactly (P = I so the residual is exactly 0)
    z, nz, rz = orc.encode(np.zeros((1, 4), np.float32), np.eye(4, dtype=np.float32),
                           np.zeros((1, 4), np.float32), np.zeros(1, np.int32))
    assert int(z[0, 0]) == 0b1111 and nz[0] == 0.0 and rz[0] == 1.0


@pytest.mark.parametrize("D,expect", [(96, 0.79997), (128, 0.79944), (960, 0.79809)])
def test_rho_closed_form(orc, D, expect):
    """For isotropic residuals E[rho] = sqrt(D) Gamma(D/2) / (sqrt(pi) Gamma((D+1)/2))."""
    cf = math.exp(0.5 * math.log(D) + math.lgamma(D / 2) - 0.5 * math.log(math.pi) - math.lgamma((D + 1) / 2))
    assert abs(cf - expect) < 1e-5
    n = 20000 if D < 960 else 4000
    X = np.random.default_rng(D).standard_normal((n, D)).astype(np.float32)
    _, _, rho = orc.encode(X, np.eye(D, dtype=np.float32), np.zeros((1, D), np.float32), np.zeros(n, np.int32))
    se = rho.std() / math.sqrt(n)
    assert abs(rho.mean() - cf) < max(4 * se, 1e-4)


# --------------------------------------------------------------------------
# Probe (P:L320-321 fused L2 = GEMM + norms)
# --------------------------------------------------------------------------
def test_probe_matches_gemm_decomposition(orc):
    """The paper's decomposition ||q||^2 + ||c||^2 - 2 q.c (a different formula,
    numpy fp64) ranks the centroids the same way, ties -> lower id."""
    rng = np.random.default_rng(8)
    C = rng.standard_normal((300, 64)).astype(np.float32)
    for t in range(20):
        q = rng.standard_normal(64).astype(np.float32)
        got = orc.probe(q, C, 17)
        q64, C64 = q.astype(np.float64), C.astype(np.float64)
        d = (q64 @ q64) + (C64 * C64).sum(1) - 2 * C64 @ q64
        ref = np.lexsort((np.arange(300), d))[:17]
        assert np.array_equal(got, ref)
    # a query equal to centroid j probes j first; nprobe = nlist is a permutation
    assert orc.probe(C[123], C, 1)[0] == 123
    assert sorted(orc.probe(C[5], C, 300).tolist()) == list(range(300))
    # exact ties -> lower id
    C2 = np.array([[1, 0], [0, 1], [-1, 0], [0, -1]], np.float32)
    assert orc.probe(np.zeros(2, np.float32), C2, 4).tolist() == [0, 1, 2, 3]


# --------------------------------------------------------------------------
# Quantizer (NS(2); R#10-12)
# --------------------------------------------------------------------------
def test_quantizer_unbiased(orc):
    """E_u[Delta qbar + v_l] = r (randomized rounding is unbiased)."""
    rng = np.random.default_rng(9)
    D = 64
    qr = rng.standard_normal(D).astype(np.float32)
    cr = rng.standard_normal(D).astype(np.float32)
    r = (qr - cr).astype(np.float64)  # the fp32 residual the quantizer sees (R#11)
    S = 4000
    acc = np.zeros(D)
    acc2 = np.zeros(D)
    for s in range(S):
        qb, vl, dl, sq, nq2 = orc.quantize(qr, cr, 77, 3, s)
        deq = dl * qb.astype(np.float64) + vl
        acc += deq
        acc2 += deq ** 2
        assert sq == int(qb.astype(np.int64).sum())
        assert abs(nq2 - (r ** 2).sum()) < 1e-9 * (r ** 2).sum() + 1e-6
    mean = acc / S
    sd = np.sqrt(np.maximum(acc2 / S - mean ** 2, 1e-30))
    rng_ = r.max() - r.min()
    det = sd < 1e-9 * rng_  # min / max coordinates are deterministic (qbar = 0 / 15)
    assert np.abs(mean - r)[det].max() <= 1e-6 * rng_
    t = (mean - r)[~det] / (sd[~det] / math.sqrt(S))
    assert np.abs(t).max() < 4.5
    assert np.abs(mean - r).max() < 0.05 * (r.max() - r.min()) / 15


def test_quantizer_special_cases(orc):
    rng = np.random.default_rng(10)
    D = 37
    qr = rng.standard_normal(D).astype(np.float32)
    cr = np.zeros(D, np.float32)
    for s in range(200):
        qb, vl, dl, sq, _ = orc.quantize(qr, cr, 5, 1, s)
        assert qb[np.argmin(qr)] == 0          # the minimum always maps to 0
        assert qb.max() <= 15
        assert vl == qr.min()
    # r on the 16-level grid -> qbar exact for every u
    grid = (np.arange(D) % 16).astype(np.float32) * 0.5 - 2.0  # Delta = 0.5
    for s in range(50):
        qb, vl, dl, _, _ = orc.quantize(grid, cr, 5, 2, s)
        assert dl == 0.5 and vl == -2.0
        assert np.array_equal(qb, (np.arange(D) % 16).astype(np.uint8))
    # Delta = 0 (all residual coordinates equal, incl. q = c): all zero (R#10)
    qb, vl, dl, sq, nq2 = orc.quantize(np.full(D, 3.0, np.float32), np.full(D, 1.0, np.float32), 5, 0, 0)
    assert dl == 0.0 and vl == 2.0 and sq == 0 and not qb.any() and nq2 == 4.0 * D
    # the counter carries the list id and the query id: different pairs draw differently
    a = orc.quantize(qr, cr, 5, 1, 0)[0]
    b = orc.quantize(qr, cr, 5, 2, 0)[0]
    c = orc.quantize(qr, cr, 5, 1, 1)[0]
    assert not np.array_equal(a, b) and not np.array_equal(a, c)


def test_quantizer_uniform_draws(orc):
    """u = (w >> 8) 2^-24 from Philox is uniform on [0,1): the fractional
    rounding probability equals the fractional part."""
    D = 16
    qr = np.zeros(D, np.float32)
    qr[1] = 15.0  # v_l = qr[0] = 0, v_r = 15 -> Delta = 1
    qr[2:] = 7.25  # t = 7.25 -> qbar in {7, 8}, P(8) = 0.25
    cr = np.zeros(D, np.float32)
    ups = 0
    S = 3000
    for s in range(S):
        qb = orc.quantize(qr, cr, 9, 0, s)[0]
        assert qb[0] == 0 and qb[1] == 15
        assert set(qb[2:].tolist()) <= {7, 8}
        ups += int((qb[2:] == 8).sum())
    p = ups / (S * (D - 2))
    assert abs(p - 0.25) < 4 * math.sqrt(0.25 * 0.75 / (S * (D - 2)))


# --------------------------------------------------------------------------
# Inner product (Eq. 3) -- checked by a different algorithm
# --------------------------------------------------------------------------
def test_ip_eq3_hamming_identity_exhaustive(orc):
    """Eq. (3): Ham(Q(q), Q(x)) = (D - Q(q).Q(x))/2 for +-1 codes.  In 0/1 form
    with a 1-bit query, <b, q> = (popc(b) + popc(q) - popc(b XOR q)) / 2 --
    computed here with Python integer popcounts, exhaustively at D = 8."""
    D = 8
    for b in range(256):
        code = np.array([b], np.uint32)
        for q in range(256):
            qbar = np.array([(q >> i) & 1 for i in range(D)], np.uint8)
            ip, pc = orc.ip(code, qbar, D)
            assert pc == bin(b).count("1")
            assert 2 * ip == bin(b).count("1") + bin(q).count("1") - bin(b ^ q).count("1")
            # and the +-1 form of Eq. (3): sum (2b-1)(2q-1) = D - 2 Ham
            pm = 4 * ip - 2 * pc - 2 * bin(q).count("1") + D
            assert pm == D - 2 * bin(b ^ q).count("1")


@pytest.mark.parametrize("D", [1, 31, 32, 33, 96, 128, 960])
def test_ip_bitplane_identity(orc, D):
    """ip = sum_j 2^j popc(code AND plane_j) over the 4 bit-planes of qbar
    (the bit-plane form of Eq. 3), with Python integers."""
    rng = np.random.default_rng(D)
    W = (D + 31) // 32
    for _ in range(20):
        bits = rng.integers(0, 2, D)
        qbar = rng.integers(0, 16, D).astype(np.uint8)
        code = np.zeros(W, np.uint32)
        for i in range(D):
            code[i >> 5] |= np.uint32(int(bits[i]) << (i & 31))
        cint = sum(int(code[w]) << (32 * w) for w in range(W))
        ref = 0
        for j in range(4):
            plane = sum(((int(qbar[i]) >> j) & 1) << i for i in range(D))
            ref += (1 << j) * bin(cint & plane).count("1")
        ip, pc = orc.ip(code, qbar, D)
        assert ip == ref and pc == bin(cint).count("1")


# --------------------------------------------------------------------------
# Estimator (NS(4): unbiasedness, O(1/sqrt(D)) error bound at eps0 = 1.9)
# --------------------------------------------------------------------------
def _pairs(rng, n, D, ip_target=None):
    o = rng.standard_normal((n, D))
    o /= np.linalg.norm(o, axis=1, keepdims=True)
    g = rng.standard_normal((n, D))
    g -= (g * o).sum(1, keepdims=True) * o
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    t = rng.uniform(-0.9, 0.9, n) if ip_target is None else np.full(n, ip_target)
    q = t[:, None] * o + np.sqrt(1 - t ** 2)[:, None] * g
    return o.astype(np.float32), q.astype(np.float32)


def _errors(orc, D, n, seed, fourbit, ip_target=None):
    """<o,q> estimation errors for n random unit pairs (P = I: isotropic pairs
    make the rotation irrelevant), with either the 4-bit query (NS(2)) or the
    exact query residual."""
    rng = np.random.default_rng(seed)
    o, q = _pairs(rng, n, D, ip_target)
    codes, n_o, rho = orc.encode(o, np.eye(D, dtype=np.float32), np.zeros((1, D), np.float32),
                                 np.zeros(n, np.int32))
    z = np.zeros(D, np.float32)
    err = np.empty(n)
    viol = 0
    for v in range(n):
        if fourbit:
            qb, vl, dl, sq, nq2 = orc.quantize(q[v], z, seed, 0, v)
            ip, pc = orc.ip(codes[v], qb, D)
            est, bd = orc.estimate(ip, pc, D, float(n_o[v]), float(rho[v]), vl, dl, sq, nq2)
        else:
            nq2 = float((q[v].astype(np.float64) ** 2).sum())
            est, bd = orc.estimate_fullq(codes[v], q[v].astype(np.float64), D, float(n_o[v]), float(rho[v]))
        no, nq = float(n_o[v]), math.sqrt(nq2)
        oq = float(o[v].astype(np.float64) @ q[v].astype(np.float64))
        exact = no * no + nq2 - 2 * oq  # ||o - q||^2 with c = 0
        err[v] = (no * no + nq2 - est) / (2 * no * nq) - oq / (no * nq)
        if abs(est - exact) > bd:
            viol += 1
    return err, viol / n


def test_estimator_unbiased(orc):
    """NS: mean error ~ 0 over 1e5 random pairs (4-bit query, D = 128)."""
    err, _ = _errors(orc, 128, 100_000, 21, fourbit=True)
    t = err.mean() / (err.std() / math.sqrt(err.size))
    assert abs(t) < 4.0


@pytest.mark.parametrize("D", [64, 256, 960])
def test_estimator_unbiased_other_D(orc, D):
    n = 20000 if D < 960 else 6000
    err, _ = _errors(orc, D, n, 22 + D, fourbit=True)
    assert abs(err.mean() / (err.std() / math.sqrt(n))) < 4.0


def test_estimator_error_scaling_and_bound(orc):
    """O(1/sqrt(D)): sd * sqrt(D-1) ~ E[sqrt(1-rho^2)/rho] sqrt(1-<o,q>^2) ~ 0.75,
    log-log slope ~ -1/2; the bound at eps0 = 1.9 is violated with probability
    <= 2(1 - Phi(1.9)) = 5.74 % (exact query); the 4-bit query costs <= 6 % sd."""
    Ds = [64, 128, 256, 512]
    sds = []
    for D in Ds:
        n = 20000
        err, viol = _errors(orc, D, n, 100 + D, fourbit=False)
        sd = err.std()
        sds.append(sd)
        assert 0.62 <= sd * math.sqrt(D - 1) <= 0.80  # pairs span <o,q> in [-0.9,0.9]
        assert viol <= 0.0574 + 4 * math.sqrt(0.0574 * 0.9426 / n)
        if D == 128:
            err4, viol4 = _errors(orc, D, n, 100 + D, fourbit=True)
            assert err4.std() / sd <= 1.06
            assert viol4 <= 0.08
    slope = np.polyfit(np.log(Ds), np.log(sds), 1)[0]
    assert -0.55 <= slope <= -0.45


@pytest.mark.parametrize("t", [0.0, 0.5])
def test_bound_violation_rate_two_sided(orc, t):
    """Two-sided pin of the error bound (NS(4), eps0 = 1.9, R#14).  At fixed
    <o,q> = t the exact-query estimator's error is
        <obar,q>/<obar,o> - t = sqrt(1-rho^2) sqrt(1-t^2) u / rho,
    u = <e, w> a coordinate of a uniform unit vector in D-1 dimensions,
    independent of rho (obar = rho o + sqrt(1-rho^2) e, q = t o + sqrt(1-t^2) w,
    e, w unit and orthogonal to o).  The bound is eps0 sqrt(1-rho^2)/(rho
    sqrt(D-1)), so P(|err| > bound) = P(|u| > a), a = eps0 / (sqrt(1-t^2)
    sqrt(D-1)), = I_{1-a^2}((D-2)/2, 1/2) exactly (regularized incomplete beta).
    The measured rate must lie within 4 SE of it on both sides: a bound 2x too
    wide (rate ~1e-8) or too narrow (~0.45) fails."""
    from scipy.special import betainc

    D, n = 128, 20000
    _, viol = _errors(orc, D, n, 300 + int(10 * t), fourbit=False, ip_target=t)
    m = D - 1
    a = 1.9 / (math.sqrt(1 - t * t) * math.sqrt(m))
    p = float(betainc((m - 1) / 2, 0.5, 1 - a * a))
    se = math.sqrt(p * (1 - p) / n)
    assert abs(viol - p) <= 4 * se, (viol, p, se)


def test_estimator_special_cases(orc):
    """D = 1 is exact; n_o = 0 gives est = n_q^2; with P = I, all |r_o,i| equal
    (rho = 1) and r_q on the 16-level grid the estimate is the exact distance."""
    # D = 1
    for ro, rq in [(1.5, -0.25), (-2.0, 3.0), (0.5, 0.5)]:
        code, n_o, rho = orc.encode(np.array([[ro]], np.float32), np.eye(1, dtype=np.float32),
                                    np.zeros((1, 1), np.float32), np.zeros(1, np.int32))
        qb, vl, dl, sq, nq2 = orc.quantize(np.array([rq], np.float32), np.zeros(1, np.float32), 1, 0, 0)
        ip, pc = orc.ip(code[0], qb, 1)
        est, bd = orc.estimate(ip, pc, 1, float(n_o[0]), float(rho[0]), vl, dl, sq, nq2)
        assert est == pytest.approx((ro - rq) ** 2, rel=1e-12, abs=1e-12) and bd == 0.0
    # n_o = 0
    est, bd = orc.estimate(37, 20, 64, 0.0, 1.0, -1.0, 0.2, 400, 7.5)
    assert est == 7.5 and bd == 0.0
    # rho = 1 and grid-exact query (D = 64 so n_o = 8a is exact in the stored fp32)
    D = 64
    a = 0.75
    signs = np.where(np.random.default_rng(2).integers(0, 2, D) > 0, 1.0, -1.0)
    x = (a * signs).astype(np.float32)
    rq = ((np.arange(D) % 16) * 0.25 - 1.0).astype(np.float32)
    code, n_o, rho = orc.encode(x[None], np.eye(D, dtype=np.float32), np.zeros((1, D), np.float32),
                                np.zeros(1, np.int32))
    assert rho[0] == 1.0
    qb, vl, dl, sq, nq2 = orc.quantize(rq, np.zeros(D, np.float32), 3, 0, 0)
    ip, pc = orc.ip(code[0], qb, D)
    est, _ = orc.estimate(ip, pc, D, float(n_o[0]), float(rho[0]), vl, dl, sq, nq2)
    exact = float(((x.astype(np.float64) - rq.astype(np.float64)) ** 2).sum())
    assert est == pytest.approx(exact, rel=1e-12)


# --------------------------------------------------------------------------
# End-to-end search and its sharded semantics
# --------------------------------------------------------------------------
def _mixture(seed, n, D, ncent, nq):
    rng = np.random.default_rng(seed)
    mu = rng.standard_normal((ncent, D)) * 2
    X = (mu[rng.integers(0, ncent, n)] + rng.standard_normal((n, D))).astype(np.float32)
    Q = (mu[rng.integers(0, ncent, nq)] + rng.standard_normal((nq, D))).astype(np.float32)
    return X, Q


def _np_knn(X, Q, k):
    X64 = X.astype(np.float64)
    ids, ds = [], []
    for q in Q.astype(np.float64):
        row = ((X64 - q) ** 2).sum(-1)
        o = np.lexsort((np.arange(X.shape[0]), row))[:k]
        ids.append(o)
        ds.append(row[o])
    return np.stack(ids), np.stack(ds)


def test_bruteforce_matches_numpy(orc):
    X, Q = _mixture(30, 3000, 24, 10, 20)
    X[7] = X[8]  # exact tie -> lower id first
    Q[0] = X[7]
    ids, d = orc.bruteforce(X, Q, 5)
    rid, rd = _np_knn(X, Q, 5)
    assert np.array_equal(ids, rid)
    assert np.allclose(d, rd, rtol=1e-12, atol=0)
    assert ids[0, 0] == 7 and ids[0, 1] == 8


def test_exhaustive_search_is_exact_knn(orc):
    """nprobe = nlist and M >= N reduce the method to exact kNN."""
    X, Q = _mixture(31, 2000, 40, 12, 15)
    idx = orc.OracleIndex(X, 12, seed=4)
    ids, d = idx.search(Q, 10, 12, 2000)
    rid, rd = _np_knn(X, Q, 10)
    assert np.array_equal(ids, rid)
    assert np.allclose(d, rd.astype(np.float32), rtol=1e-6)
    # also with the lower-bound rank key: exhaustive M is still exact
    ids2, _ = idx.search(Q, 10, 12, 2000, rank_key=1)
    assert np.array_equal(ids2, rid)


def test_recall_and_monotonicity(orc):
    """Recall@10 vs brute force on a CFG1-shaped mixture (scaled to N = 20k so
    the CPU suite stays fast), monotone in nprobe and M."""
    X, Q = _mixture(32, 20000, 128, 64, 40)
    idx = orc.OracleIndex(X, 64, seed=42, max_iter=10)
    gt, _ = _np_knn(X, Q, 10)

    def recall(ids):
        return np.mean([len(set(a) & set(b)) / 10 for a, b in zip(ids, gt)])

    r = {}
    for nprobe in (1, 4, 16):
        for M in (10, 100):
            ids, _ = idx.search(Q, 10, nprobe, M)
            r[(nprobe, M)] = recall(ids)
    assert r[(16, 100)] >= 0.9
    assert r[(1, 100)] <= r[(4, 100)] <= r[(16, 100)]
    assert r[(16, 10)] <= r[(16, 100)]


def test_sharded_semantics(orc):
    """G = 1 equals single; per-shard top-M is a superset of the global top-M,
    so the merged top-k is elementwise no farther; the exhaustive
    result is invariant to G."""
    X, Q = _mixture(33, 6000, 32, 16, 25)
    single = orc.OracleIndex(X, 16, seed=8, max_iter=10)
    base = dict(P=single.P, Cr=single.Cr)
    k, nprobe, M = 10, 4, 20

    def shard_search(G, nprobe, M):
        outs_i, outs_d = [], []
        for g in range(G):
            lo, hi = (6000 * g) // G, (6000 * (g + 1)) // G
            a = single.assign[lo:hi]
            order = np.argsort(a, kind="stable")
            off = np.concatenate([[0], np.cumsum(np.bincount(a, minlength=16))]).astype(np.int64)
            codes, n_o, rho = orc.encode(X[lo:hi], base["P"], base["Cr"], a)
            ids, d = orc.search(Q, base["P"], base["Cr"], off, (order + lo).astype(np.int64), codes[order],
                                n_o[order], rho[order], X[lo:hi], k, nprobe, M, 8, id_offset=lo)
            outs_i.append(ids)
            outs_d.append(d)
        return orc.merge_topk(np.stack(outs_i), np.stack(outs_d))

    ids1, d1 = single.search(Q, k, nprobe, M)
    g1i, g1d = shard_search(1, nprobe, M)
    assert np.array_equal(ids1, g1i) and np.array_equal(d1, g1d)
    for G in (2, 3):
        gi, gd = shard_search(G, nprobe, M)
        assert np.all(gd <= d1 + 1e-6 * np.abs(d1))
        ei, _ = shard_search(G, 16, 6000)
        ex, _ = single.search(Q, k, 16, 6000)
        assert np.array_equal(ei, ex)


def test_merge_topk(orc):
    rng = np.random.default_rng(40)
    G, nq, k = 3, 7, 5
    ids = rng.permutation(1000)[: G * nq * k].reshape(G, nq, k).astype(np.int64)
    d = rng.integers(0, 20, (G, nq, k)).astype(np.float32)  # many exact ties
    d.sort(-1)
    oi, od = orc.merge_topk(ids, d)
    for q in range(nq):
        allid = ids[:, q].ravel()
        alld = d[:, q].ravel()
        o = np.lexsort((allid, alld))[:k]
        assert np.array_equal(oi[q], allid[o]) and np.array_equal(od[q], alld[o])


def test_padding_when_fewer_candidates(orc):
    """Fewer than k candidates in the probed lists -> (-1, +inf) padding (R#22)."""
    X, Q = _mixture(34, 300, 16, 30, 5)
    idx = orc.OracleIndex(X, 30, seed=2, max_iter=5)
    sizes = np.diff(idx.list_off)
    ids, d = idx.search(Q, 50, 1, 50)
    for q in range(5):
        j = orc.probe(orc.rotate(Q[q:q + 1], idx.P)[0].astype(np.float32), idx.Cr, 1)[0]
        n = int(sizes[j])
        if n < 50:
            assert np.all(ids[q, n:] == -1) and np.all(np.isinf(d[q, n:]))
            assert np.all(ids[q, :n] >= 0)


def test_rerank_is_restricted_bruteforce(orc):
    """Fine ranking over a candidate set = brute force restricted to it;
    over all ids it is exact kNN (numpy, direct subtraction)."""
    X, Q = _mixture(35, 1500, 20, 6, 12)
    allc = np.tile(np.arange(1500, dtype=np.int64), (12, 1))
    ids, d = orc.rerank(Q, X, allc, 7)
    rid, rd = _np_knn(X, Q, 7)
    assert np.array_equal(ids, rid) and np.allclose(d, rd.astype(np.float32), rtol=1e-6)
    sub = np.stack([np.random.default_rng(q).choice(1500, 40, replace=False) for q in range(12)])
    sub[:, -3:] = -1  # skipped entries
    ids2, _ = orc.rerank(Q, X, sub, 5)
    for q in range(12):
        s = sub[q][sub[q] >= 0]
        dd = ((X[s].astype(np.float64) - Q[q].astype(np.float64)) ** 2).sum(1)
        assert np.array_equal(ids2[q], s[np.lexsort((s, dd))][:5])


# ------------------------------------------------- O-S5b, NEXT-4
def test_adaptive_rerank_special_cases(orc):
    """The bound-driven re-rank set (rerank_mode 1) against the modes it must
    reduce to: an infinite bound keeps every top-M candidate (= the fixed-M
    search); a zero bound keeps exactly the candidates whose estimate is <= the
    k-th smallest estimate (= the fixed search with M = k, no ties here)."""
    X, Q = _mixture(41, 3000, 32, 12, 20)
    idx = orc.OracleIndex(X, 12, seed=5, max_iter=8)
    k, M, nprobe = 10, 80, 4
    ref_i, ref_d = idx.search(Q, k, nprobe, M)
    nr = np.empty(20, np.int64)
    a_i, a_d = idx.search(Q, k, nprobe, M, rerank_mode=1, eps0=1e30, n_reranked=nr)
    assert np.array_equal(a_i, ref_i) and np.array_equal(a_d, ref_d) and np.all(nr == M)
    k_i, k_d = idx.search(Q, k, nprobe, k)
    z_i, z_d = idx.search(Q, k, nprobe, M, rerank_mode=1, eps0=0.0, n_reranked=nr)
    assert np.array_equal(z_i, k_i) and np.array_equal(z_d, k_d) and np.all(nr == k)


def test_adaptive_rerank_recall(orc):
    """At the paper's confidence (eps0 = 1.9) the adaptive set keeps the fixed-M
    result almost everywhere (a miss needs a bound violation at the boundary);
    k <= re-ranked <= M, and a tighter bound never re-ranks more."""
    X, Q = _mixture(42, 6000, 64, 16, 40)
    idx = orc.OracleIndex(X, 16, seed=6, max_iter=8)
    k, M, nprobe = 10, 200, 6
    ref_i, _ = idx.search(Q, k, nprobe, M)
    nr = np.empty(40, np.int64)
    a_i, _ = idx.search(Q, k, nprobe, M, rerank_mode=1, n_reranked=nr)
    agree = np.mean([len(set(a.tolist()) & set(b.tolist())) / k for a, b in zip(a_i, ref_i)])
    assert agree >= 0.99, agree
    assert np.all(nr >= k) and np.all(nr <= M)
    nr2 = np.empty(40, np.int64)
    idx.search(Q, k, nprobe, M, rerank_mode=1, eps0=0.5, n_reranked=nr2)
    assert np.all(nr2 <= nr)


# ------------------------------------------- qmode 1, NEXT-1
def test_fullq_search_exhaustive_and_more_accurate(orc):
    """The unquantized-query search (qmode 1): exhaustive probing with M >= N is
    exact kNN (numpy); its estimates of the true squared distances have a
    smaller error than the 4-bit query's (no query SQ is more precise)."""
    X, Q = _mixture(43, 1200, 64, 8, 10)
    idx = orc.OracleIndex(X, 8, seed=7, max_iter=8)
    ids, d = idx.search(Q, 5, 8, 1200, qmode=1)
    rid, rd = _np_knn(X, Q, 5)
    assert np.array_equal(ids, rid) and np.allclose(d, rd.astype(np.float32), rtol=1e-6)
    err = {}
    for qm in (0, 1):
        _, _, _, tids, test = idx.search(Q, 5, 8, 1200, qmode=qm, debug=True)
        e = []
        for q in range(10):
            v = tids[q] >= 0
            true = ((X[tids[q][v]].astype(np.float64) - Q[q].astype(np.float64)) ** 2).sum(1)
            e.append(np.abs(test[q][v] - true))
        err[qm] = np.concatenate(e).mean()
    assert err[1] < err[0], err
