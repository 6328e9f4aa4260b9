/*
 * oracle.c -- plain CPU oracle of the IVF-RaBitQ search hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): loaded by tests/, by
 * __graft_entry__.smoke() and by bench.py's cpu_baseline / --impl reference
 * legs, never by the product path.  No blocking, fusion or reordering beyond
 * what the paper's definitions state; fp64 everywhere except the quantizer,
 * whose fp32 sequence is pinned (reading R#11).  Compile with
 * -ffp-contract=off, without -ffast-math.
 *
 * Paper: arxiv 2605.16007.  Cited as P:Lnnn [section/equation].
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3"): 10 rounds of the 4x32 Philox S-box with the
 * published multipliers and Weyl key increments.  NS(2): "deterministic
 * counter-based (Philox, seeded)". */
void oracle_philox4x32_10(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]) {
    uint32_t k0 = key[0], k1 = key[1];
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------------ */
/* Haar rotation (R#5).  Gaussian entries by Box-Muller from Philox,
 * then Householder QR (textbook, Golub & Van Loan Alg. 5.2.1) in fp64 and a
 * column sign fix so that diag(R) > 0, which makes Q Haar-distributed. */
int oracle_haar_rotation(int D, uint64_t seed, double* P64, float* P32) {
    if (D < 1) return -1;
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    double* A = (double*)malloc(sizeof(double) * (size_t)D * D);
    double* V = (double*)calloc((size_t)D * D, sizeof(double)); /* Householder vectors, row k = v_k */
    if (!A || !V) { free(A); free(V); return -1; }
    for (int i = 0; i < D; ++i) {
        for (int j = 0; j < D; ++j) {
            const uint32_t ctr[4] = {(uint32_t)j, (uint32_t)i, 0u, 0x524F544Eu /* 'ROTN' */};
            uint32_t w[4];
            oracle_philox4x32_10(key, ctr, w);
            double u1 = ((double)(w[0] >> 8) + 0.5) * (1.0 / 16777216.0);
            double u2 = ((double)(w[1] >> 8) + 0.5) * (1.0 / 16777216.0);
            A[(size_t)i * D + j] = sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
        }
    }
    /* A <- H_{D-1} ... H_0 A = R */
    double* diagR = (double*)malloc(sizeof(double) * D);
    for (int k = 0; k < D; ++k) {
        double nx = 0.0;
        for (int i = k; i < D; ++i) nx += A[(size_t)i * D + k] * A[(size_t)i * D + k];
        nx = sqrt(nx);
        double* v = V + (size_t)k * D;
        if (nx == 0.0) { diagR[k] = 0.0; continue; }
        double x0 = A[(size_t)k * D + k];
        double alpha = (x0 >= 0.0) ? -nx : nx;
        for (int i = k; i < D; ++i) v[i] = A[(size_t)i * D + k];
        v[k] -= alpha;
        double nv = 0.0;
        for (int i = k; i < D; ++i) nv += v[i] * v[i];
        nv = sqrt(nv);
        if (nv == 0.0) { diagR[k] = x0; for (int i = k; i < D; ++i) v[i] = 0.0; continue; }
        for (int i = k; i < D; ++i) v[i] /= nv;
        for (int j = k; j < D; ++j) {
            double s = 0.0;
            for (int i = k; i < D; ++i) s += v[i] * A[(size_t)i * D + j];
            for (int i = k; i < D; ++i) A[(size_t)i * D + j] -= 2.0 * v[i] * s;
        }
        diagR[k] = A[(size_t)k * D + k];
    }
    /* Q = H_0 H_1 ... H_{D-1} I */
    for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) P64[(size_t)i * D + j] = (i == j) ? 1.0 : 0.0;
    for (int k = D - 1; k >= 0; --k) {
        const double* v = V + (size_t)k * D;
        for (int j = 0; j < D; ++j) {
            double s = 0.0;
            for (int i = k; i < D; ++i) s += v[i] * P64[(size_t)i * D + j];
            for (int i = k; i < D; ++i) P64[(size_t)i * D + j] -= 2.0 * v[i] * s;
        }
    }
    for (int j = 0; j < D; ++j)
        if (diagR[j] < 0.0)
            for (int i = 0; i < D; ++i) P64[(size_t)i * D + j] = -P64[(size_t)i * D + j];
    if (P32)
        for (size_t e = 0; e < (size_t)D * D; ++e) P32[e] = (float)P64[e];
    free(A); free(V); free(diagR);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* x' = P^T x (R#4). */
void oracle_rotate(const float* X, int64_t n, int D, const float* P, double* Xr) {
    for (int64_t v = 0; v < n; ++v)
        for (int i = 0; i < D; ++i) {
            double s = 0.0;
            for (int k = 0; k < D; ++k) s += (double)P[(size_t)k * D + i] * (double)X[(size_t)v * D + k];
            Xr[(size_t)v * D + i] = s;
        }
}

static double sqdist_fd(const float* a, const double* b, int D) {
    double s = 0.0;
    for (int i = 0; i < D; ++i) { double t = (double)a[i] - b[i]; s += t * t; }
    return s;
}

/* Nearest centroid, ties -> lowest id ("assign it to the
 * inverted list of its nearest centroid"). */
void oracle_assign(const float* X, int64_t n, int D, const double* C, int nlist, int32_t* assign) {
    for (int64_t v = 0; v < n; ++v) {
        double best = INFINITY; int arg = 0;
        for (int j = 0; j < nlist; ++j) {
            double d = sqdist_fd(X + (size_t)v * D, C + (size_t)j * D, D);
            if (d < best) { best = d; arg = j; }
        }
        assign[v] = arg;
    }
}

/* Lloyd k-means ("Run K-Means clustering on a training subset";
 * P:L304-305 phases 1-2; details R#6). */
int oracle_kmeans(const float* T, int64_t nt, int D, int nlist, const int64_t* init_rows,
                  const float* init_centroids, int max_iter, double* C, double* obj_trace) {
    if (nt < nlist || nlist < 1 || D < 1) return -1;
    for (int j = 0; j < nlist; ++j)
        for (int i = 0; i < D; ++i)
            C[(size_t)j * D + i] = init_centroids ? (double)init_centroids[(size_t)j * D + i]
                                                  : (double)T[(size_t)init_rows[j] * D + i];
    int32_t* a = (int32_t*)malloc(sizeof(int32_t) * nt);
    int32_t* prev = (int32_t*)malloc(sizeof(int32_t) * nt);
    double* dist = (double*)malloc(sizeof(double) * nt);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * nlist);
    for (int64_t t = 0; t < nt; ++t) prev[t] = -1;
    int it = 0;
    for (; it < max_iter; ++it) {
        double obj = 0.0;
        int changed = 0;
        for (int64_t t = 0; t < nt; ++t) {
            double best = INFINITY; int arg = 0;
            for (int j = 0; j < nlist; ++j) {
                double d = sqdist_fd(T + (size_t)t * D, C + (size_t)j * D, D);
                if (d < best) { best = d; arg = j; }
            }
            a[t] = arg; dist[t] = best; obj += best;
            if (arg != prev[t]) changed = 1;
        }
        if (obj_trace) obj_trace[it] = obj;
        if (!changed) { ++it; break; }
        /* update: centroid = mean of its members */
        memset(cnt, 0, sizeof(int64_t) * nlist);
        memset(C, 0, sizeof(double) * (size_t)nlist * D);
        for (int64_t t = 0; t < nt; ++t) {
            cnt[a[t]]++;
            for (int i = 0; i < D; ++i) C[(size_t)a[t] * D + i] += (double)T[(size_t)t * D + i];
        }
        for (int j = 0; j < nlist; ++j) {
            if (cnt[j] > 0) {
                for (int i = 0; i < D; ++i) C[(size_t)j * D + i] /= (double)cnt[j];
            } else {
                /* re-seed with the point farthest from its centroid (R#6) */
                int64_t far = 0; double fd = -1.0;
                for (int64_t t = 0; t < nt; ++t) if (dist[t] > fd) { fd = dist[t]; far = t; }
                for (int i = 0; i < D; ++i) C[(size_t)j * D + i] = (double)T[(size_t)far * D + i];
                dist[far] = -1.0; /* each empty cluster takes a distinct point */
            }
        }
        memcpy(prev, a, sizeof(int32_t) * nt);
    }
    free(a); free(prev); free(dist); free(cnt);
    return it;
}

/* ------------------------------------------------------------------------ */
/* Encode (Eq. 1, sign code of the rotated residual; NS factors
 * ||o_r - c|| and <obar, o>; R#7 sign(0) -> bit 1; R#9 n_o = 0 -> rho = 1). */
void oracle_encode(const float* X, int64_t n, int D, const float* P, const float* Cr,
                   const int32_t* assign, uint32_t* codes, float* n_o, float* rho_o) {
    const int W = (D + 31) / 32;
    double* xr = (double*)malloc(sizeof(double) * D);
    for (int64_t v = 0; v < n; ++v) {
        oracle_rotate(X + (size_t)v * D, 1, D, P, xr);
        const float* c = Cr + (size_t)assign[v] * D;
        uint32_t* code = codes + (size_t)v * W;
        for (int w = 0; w < W; ++w) code[w] = 0u;
        double n2 = 0.0, l1 = 0.0;
        for (int i = 0; i < D; ++i) {
            double r = xr[i] - (double)c[i];
            if (r >= 0.0) code[i >> 5] |= 1u << (i & 31);
            n2 += r * r;
            l1 += fabs(r);
        }
        double no = sqrt(n2);
        n_o[v] = (float)no;
        rho_o[v] = (no > 0.0) ? (float)(l1 / (sqrt((double)D) * no)) : 1.0f;
    }
    free(xr);
}

/* ------------------------------------------------------------------------ */
typedef struct { double d; int64_t id; } dkey_t;

static int cmp_dkey(const void* pa, const void* pb) {
    const dkey_t* a = (const dkey_t*)pa;
    const dkey_t* b = (const dkey_t*)pb;
    if (a->d < b->d) return -1;
    if (a->d > b->d) return 1;
    /* id -1 (padding) orders after every real id */
    uint64_t ia = (uint64_t)a->id, ib = (uint64_t)b->id;
    return (ia < ib) ? -1 : (ia > ib) ? 1 : 0;
}

/* Probing (R#17 ties -> lower list id). */
void oracle_probe(const float* qr, int D, const float* Cr, int nlist, int nprobe, int32_t* probes) {
    dkey_t* dk = (dkey_t*)malloc(sizeof(dkey_t) * nlist);
    for (int j = 0; j < nlist; ++j) {
        double s = 0.0;
        for (int i = 0; i < D; ++i) {
            double t = (double)qr[i] - (double)Cr[(size_t)j * D + i];
            s += t * t;
        }
        dk[j].d = s; dk[j].id = j;
    }
    qsort(dk, nlist, sizeof(dkey_t), cmp_dkey);
    for (int p = 0; p < nprobe; ++p) probes[p] = (int32_t)dk[p].id;
    free(dk);
}

/* ------------------------------------------------------------------------ */
/* 4-bit randomized query quantization, pinned fp32 sequence (NS(2); R#11,
 * R#12; "quantized relative to the centroid c of each probed
 * cluster").  volatile temporaries force each fp32 rounding. */
void oracle_quantize(const float* qr, const float* cr, int D, uint64_t seed, int32_t list_id,
                     int64_t qglobal, uint8_t* qbar, float* v_l_out, float* delta_out,
                     int32_t* S_q_out, double* nq2_out) {
    const uint64_t s = seed ^ 0x5241424954515155ull;
    const uint32_t key[2] = {(uint32_t)s, (uint32_t)(s >> 32)};
    float* r = (float*)malloc(sizeof(float) * D);
    double nq2 = 0.0;
    float vl = INFINITY, vr = -INFINITY;
    for (int i = 0; i < D; ++i) {
        volatile float ri = qr[i] - cr[i];
        r[i] = ri;
        nq2 += (double)ri * (double)ri;
        if (ri < vl) vl = ri;
        if (ri > vr) vr = ri;
    }
    volatile float range = vr - vl;
    volatile float delta = range / 15.0f;
    int32_t Sq = 0;
    uint32_t w[4] = {0, 0, 0, 0};
    for (int i = 0; i < D; ++i) {
        int q = 0;
        if (delta != 0.0f) {
            if ((i & 3) == 0) {
                const uint32_t ctr[4] = {(uint32_t)(i >> 2), (uint32_t)list_id, (uint32_t)qglobal,
                                         0x51554E54u /* 'QUNT' */};
                oracle_philox4x32_10(key, ctr, w);
            }
            float u = (float)(w[i & 3] >> 8) * (1.0f / 16777216.0f);
            volatile float diff = r[i] - vl;
            volatile float t = diff / delta;
            volatile float y = t + u;
            q = (int)floorf(y);
            if (q > 15) q = 15;
        }
        qbar[i] = (uint8_t)q;
        Sq += q;
    }
    *v_l_out = vl;
    *delta_out = delta;
    *S_q_out = Sq;
    *nq2_out = nq2;
    free(r);
}

/* <b, qbar> (Eq. 3 in 0/1 form) by a plain per-dimension loop. */
int64_t oracle_ip(const uint32_t* code, const uint8_t* qbar, int D, int64_t* pc) {
    int64_t ip = 0, p = 0;
    for (int i = 0; i < D; ++i) {
        int64_t b = (code[i >> 5] >> (i & 31)) & 1u;
        ip += b * (int64_t)qbar[i];
        p += b;
    }
    if (pc) *pc = p;
    return ip;
}

/* NS(4): est = n_o^2 + ||r_q||^2 - 2 n_o <o,q>_est n_q, with the unbiased
 * <o,q> estimate <xbar, qbar>/(n_q <obar,o>) (R#1); the bound is the
 * O(1/sqrt(D)) error bound at eps0 (R#14). */
void oracle_estimate(int64_t ip, int64_t pc, int D, double n_o, double rho_o, double v_l,
                     double delta, int64_t S_q, double nq2, double eps0, double* est, double* bound) {
    double X = (2.0 * delta * (double)ip + 2.0 * v_l * (double)pc - delta * (double)S_q
                - (double)D * v_l) / sqrt((double)D);
    *est = n_o * n_o + nq2 - 2.0 * n_o * X / rho_o;
    if (bound) {
        double one_m = 1.0 - rho_o * rho_o;
        if (one_m < 0.0) one_m = 0.0;
        *bound = (D > 1) ? 2.0 * n_o * sqrt(nq2) * eps0 * sqrt(one_m) / (rho_o * sqrt((double)D - 1.0))
                         : 0.0;
    }
}

void oracle_estimate_fullq(const uint32_t* code, const double* rq, int D, double n_o, double rho_o,
                           double eps0, double* est, double* bound) {
    double X = 0.0, nq2 = 0.0;
    for (int i = 0; i < D; ++i) {
        double b = (double)((code[i >> 5] >> (i & 31)) & 1u);
        X += (2.0 * b - 1.0) / sqrt((double)D) * rq[i];
        nq2 += rq[i] * rq[i];
    }
    *est = n_o * n_o + nq2 - 2.0 * n_o * X / rho_o;
    if (bound) {
        double one_m = 1.0 - rho_o * rho_o;
        if (one_m < 0.0) one_m = 0.0;
        *bound = (D > 1) ? 2.0 * n_o * sqrt(nq2) * eps0 * sqrt(one_m) / (rho_o * sqrt((double)D - 1.0))
                         : 0.0;
    }
}

/* ------------------------------------------------------------------------ */
static int cmp_double(const void* pa, const void* pb) {
    const double a = *(const double*)pa, b = *(const double*)pb;
    return (a > b) - (a < b);
}

typedef struct { double key; int64_t id; double est; double bound; } cand_t;

static int cmp_cand(const void* pa, const void* pb) {
    const cand_t* a = (const cand_t*)pa;
    const cand_t* b = (const cand_t*)pb;
    if (a->key < b->key) return -1;
    if (a->key > b->key) return 1;
    return (a->id < b->id) ? -1 : (a->id > b->id) ? 1 : 0;
}

/* The three-stage pipeline of P:L239-246 (probe, coarse top-M, exact
 * re-rank top-k) with the NS estimator; see oracle.h for the steps. */
int oracle_search(const float* Q, int64_t nq, int D, const float* P, const float* Cr, int nlist,
                  const int64_t* list_off, const int64_t* list_ids, const uint32_t* codes,
                  const float* n_o, const float* rho_o, const float* X, int64_t id_offset,
                  int k, int nprobe, int M, uint64_t seed, int64_t qid_base, int rank_key,
                  double eps0, const float* qr_in, const int32_t* probes_in, int num_threads,
                  int64_t* ids, float* dists, int32_t* probes_out, int64_t* topm_ids,
                  double* topm_est, int rerank_mode, int64_t* n_reranked, int qmode) {
    if (nq < 0 || D < 1 || nlist < 1 || k < 1 || M < k || nprobe < 1 || nprobe > nlist) return -1;
    if (qmode != 0 && qmode != 1) return -1;
    if (rerank_mode != 0 && (rerank_mode != 1 || rank_key != 0)) return -1;
    const int W = (D + 31) / 32;
#ifdef _OPENMP
    if (num_threads <= 0) num_threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(num_threads)
#endif
    for (int64_t qi = 0; qi < nq; ++qi) {
        const float* q = Q + (size_t)qi * D;
        float* qr = (float*)malloc(sizeof(float) * D);
        int32_t* probes = (int32_t*)malloc(sizeof(int32_t) * nprobe);
        uint8_t* qbar = (uint8_t*)malloc(D);
        /* O-S1: q' = P^T q in fp64, rounded to fp32 */
        if (qr_in) {
            memcpy(qr, qr_in + (size_t)qi * D, sizeof(float) * D);
        } else {
            for (int i = 0; i < D; ++i) {
                double s = 0.0;
                for (int kk = 0; kk < D; ++kk) s += (double)P[(size_t)kk * D + i] * (double)q[kk];
                qr[i] = (float)s;
            }
        }
        /* O-S2: probe */
        if (probes_in) memcpy(probes, probes_in + (size_t)qi * nprobe, sizeof(int32_t) * nprobe);
        else oracle_probe(qr, D, Cr, nlist, nprobe, probes);
        if (probes_out) memcpy(probes_out + (size_t)qi * nprobe, probes, sizeof(int32_t) * nprobe);
        /* O-S3/O-S4: coarse ranking over every vector of every probed list */
        int64_t total = 0;
        for (int p = 0; p < nprobe; ++p) total += list_off[probes[p] + 1] - list_off[probes[p]];
        cand_t* cand = (cand_t*)malloc(sizeof(cand_t) * (total > 0 ? total : 1));
        int64_t nc = 0;
        double* rq = (double*)malloc(sizeof(double) * D);
        for (int p = 0; p < nprobe; ++p) {
            const int j = probes[p];
            float vl, delta; int32_t Sq; double nq2;
            if (qmode == 0)
                oracle_quantize(qr, Cr + (size_t)j * D, D, seed, j, qid_base + qi, qbar, &vl, &delta, &Sq, &nq2);
            else /* O-S3' (NEXT-1): the unquantized residual r_q = q' - c' */
                for (int i = 0; i < D; ++i) rq[i] = (double)qr[i] - (double)Cr[(size_t)j * D + i];
            for (int64_t s = list_off[j]; s < list_off[j + 1]; ++s) {
                double est, bound;
                if (qmode == 0) {
                    int64_t pc;
                    int64_t ip = oracle_ip(codes + (size_t)s * W, qbar, D, &pc);
                    oracle_estimate(ip, pc, D, (double)n_o[s], (double)rho_o[s], (double)vl, (double)delta,
                                    Sq, nq2, eps0, &est, &bound);
                } else {
                    oracle_estimate_fullq(codes + (size_t)s * W, rq, D, (double)n_o[s], (double)rho_o[s], eps0,
                                          &est, &bound);
                }
                cand[nc].key = (rank_key == 1) ? est - bound : est;
                cand[nc].est = est;
                cand[nc].bound = bound;
                cand[nc].id = list_ids[s];
                ++nc;
            }
        }
        /* O-S5: top-M by (key, id) (R#16, R#17) */
        qsort(cand, nc, sizeof(cand_t), cmp_cand);
        int64_t m = nc < M ? nc : M;
        if (topm_ids) {
            for (int64_t i = 0; i < M; ++i) {
                topm_ids[(size_t)qi * M + i] = (i < m) ? cand[i].id : -1;
                topm_est[(size_t)qi * M + i] = (i < m) ? cand[i].est : INFINITY;
            }
        }
        /* O-S5b (rerank_mode 1, NEXT-4): bound-driven re-rank set.  With the
         * error bound of Eq. (2)'s estimator (NS(4)), d lies in [est - bound,
         * est + bound] at the bound's confidence; tau = the k-th smallest
         * est + bound of the top-M; only candidates with est - bound <= tau can
         * be in the top-k, the others are not re-ranked. */
        uint8_t* keep = (uint8_t*)malloc(m > 0 ? (size_t)m : 1);
        for (int64_t i = 0; i < m; ++i) keep[i] = 1;
        if (rerank_mode == 1 && m > k) {
            double* ub = (double*)malloc(sizeof(double) * (size_t)m);
            for (int64_t i = 0; i < m; ++i) ub[i] = cand[i].est + cand[i].bound;
            qsort(ub, m, sizeof(double), cmp_double);
            const double tau = ub[k - 1];
            for (int64_t i = 0; i < m; ++i) keep[i] = (cand[i].est - cand[i].bound <= tau);
            free(ub);
        }
        /* O-S6: exact squared L2 on the raw vectors, top-k by (d, id) (R#19) */
        dkey_t* fk = (dkey_t*)malloc(sizeof(dkey_t) * (m > 0 ? m : 1));
        int64_t mr = 0;
        for (int64_t i = 0; i < m; ++i) {
            if (!keep[i]) continue;
            const float* x = X + (size_t)(cand[i].id - id_offset) * D;
            double s = 0.0;
            for (int d = 0; d < D; ++d) { double t = (double)q[d] - (double)x[d]; s += t * t; }
            fk[mr].d = s; fk[mr].id = cand[i].id; ++mr;
        }
        if (n_reranked) n_reranked[qi] = mr;
        free(keep);
        m = mr;
        qsort(fk, m, sizeof(dkey_t), cmp_dkey);
        for (int i = 0; i < k; ++i) {
            ids[(size_t)qi * k + i] = (i < m) ? fk[i].id : -1;
            dists[(size_t)qi * k + i] = (i < m) ? (float)fk[i].d : INFINITY;
        }
        free(fk); free(cand); free(qbar); free(probes); free(qr); free(rq);
    }
    return 0;
}

/* Fine ranking of a given candidate set. */
void oracle_rerank(const float* Q, int64_t nq, int D, const float* X, int64_t id_offset,
                   const int64_t* cand, int M, int k, int64_t* ids, float* dists) {
    dkey_t* fk = (dkey_t*)malloc(sizeof(dkey_t) * (M > 0 ? M : 1));
    for (int64_t qi = 0; qi < nq; ++qi) {
        const float* q = Q + (size_t)qi * D;
        int m = 0;
        for (int c = 0; c < M; ++c) {
            int64_t id = cand[(size_t)qi * M + c];
            if (id < 0) continue;
            const float* x = X + (size_t)(id - id_offset) * D;
            double s = 0.0;
            for (int d = 0; d < D; ++d) { double t = (double)q[d] - (double)x[d]; s += t * t; }
            fk[m].d = s; fk[m].id = id; ++m;
        }
        qsort(fk, m, sizeof(dkey_t), cmp_dkey);
        for (int i = 0; i < k; ++i) {
            ids[(size_t)qi * k + i] = (i < m) ? fk[i].id : -1;
            dists[(size_t)qi * k + i] = (i < m) ? (float)fk[i].d : INFINITY;
        }
    }
    free(fk);
}

/* Global top-k over the union of per-shard top-k lists (R#20). */
void oracle_merge_topk(const int64_t* in_ids, const float* in_d, int G, int64_t nq, int k,
                       int64_t* out_ids, float* out_d) {
    dkey_t* buf = (dkey_t*)malloc(sizeof(dkey_t) * (size_t)G * k);
    for (int64_t qi = 0; qi < nq; ++qi) {
        int n = 0;
        for (int g = 0; g < G; ++g)
            for (int i = 0; i < k; ++i) {
                size_t e = ((size_t)g * nq + qi) * k + i;
                buf[n].d = (double)in_d[e]; buf[n].id = in_ids[e]; ++n;
            }
        qsort(buf, n, sizeof(dkey_t), cmp_dkey);
        for (int i = 0; i < k; ++i) {
            out_ids[(size_t)qi * k + i] = buf[i].id;
            out_d[(size_t)qi * k + i] = (float)buf[i].d;
        }
    }
    free(buf);
}

/* Exact kNN ("the exact nearest neighbor search problem"). */
void oracle_bruteforce(const float* X, int64_t n, int D, const float* Q, int64_t nq, int k,
                       int num_threads, int64_t* ids, double* dists) {
#ifdef _OPENMP
    if (num_threads <= 0) num_threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(num_threads)
#endif
    for (int64_t qi = 0; qi < nq; ++qi) {
        dkey_t* best = (dkey_t*)malloc(sizeof(dkey_t) * (k + 1));
        int nb = 0;
        const float* q = Q + (size_t)qi * D;
        for (int64_t v = 0; v < n; ++v) {
            const float* x = X + (size_t)v * D;
            double s = 0.0;
            for (int d = 0; d < D; ++d) { double t = (double)q[d] - (double)x[d]; s += t * t; }
            dkey_t e = {s, v};
            if (nb == k && cmp_dkey(&e, &best[k - 1]) >= 0) continue;
            int pos = (nb < k) ? nb++ : k - 1;
            while (pos > 0 && cmp_dkey(&e, &best[pos - 1]) < 0) { best[pos] = best[pos - 1]; --pos; }
            best[pos] = e;
        }
        for (int i = 0; i < k; ++i) {
            ids[(size_t)qi * k + i] = (i < nb) ? best[i].id : -1;
            dists[(size_t)qi * k + i] = (i < nb) ? best[i].d : INFINITY;
        }
        free(best);
    }
}
