/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle of the IVF-RaBitQ
 * search hot path (arxiv 2605.16007, "Ascend-RaBitQ").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code with the CUDA path (paper_2605_16007_b200/csrc) and the
 * CUDA path never includes, links or calls it.
 *
 * Citations: "P:Lnnn" = line nnn of the paper text, with section
 * or equation; "NS" = BASELINE.json north_star; "R#n" = reading n of the
 * ambiguity ledger in DESIGN.md.
 *
 * Conventions (shared with the C-ABI contract, include/rabitq.h):
 *   - matrices are row-major; vectors are rows;
 *   - rotation: x' = P^T x, i.e. row form x'^T = x^T P   (R#4);
 *   - codes: W = ceil(D/32) uint32 words per vector, bit i of the code is
 *     bit (i & 31) of word (i >> 5) (LSB first), bit = [r_i >= 0] (P:L202,
 *     R#7, R#8); pad bits are 0;
 *   - all floating point is fp64 unless a step pins fp32 (the quantizer,
 *     R#11), compiled with -ffp-contract=off and no -ffast-math.
 *
 * Parity status of each function (pins live in tests/test_oracle_*.py):
 *   every function is pinned EXCEPT oracle_kmeans' exact centroids, which
 *   are "parity unpinned" (float summation order; only its invariants are
 *   checked, and the GPU path's k-means is never compared against it).
 */
#ifndef RABITQ_ORACLE_H
#define RABITQ_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Philox4x32-10 (Salmon et al., SC'11), the counter-based generator NS(2)
 * names.  out = Philox(key, ctr). */
void oracle_philox4x32_10(const uint32_t key[2], const uint32_t ctr[4], uint32_t out[4]);

/* Haar-random orthogonal P ("random orthogonal rotation", R#5):
 * standard normals from Philox (key = seed, ctr = (j, i, 0, 'ROTN')) by
 * Box-Muller, Householder QR in fp64, columns sign-fixed so diag(R) > 0.
 * Writes P64 (fp64) and P32 (the same values rounded to fp32). */
int oracle_haar_rotation(int D, uint64_t seed, double* P64, float* P32);

/* x'_i = sum_k P[k][i] x_k in fp64 (R#4).  X [n x D] fp32 in,
 * Xr [n x D] fp64 out. */
void oracle_rotate(const float* X, int64_t n, int D, const float* P, double* Xr);

/* Lloyd k-means in the ORIGINAL space, fp64 (
 * defaults R#6): init = rows init_rows[0..nlist) of T (or init_centroids
 * when non-NULL), assignment argmin ||t - c||^2 (direct subtraction, ties ->
 * lowest id), mean update, an empty cluster is re-seeded with the point
 * farthest from its assigned centroid, stop after max_iter iterations or
 * when no assignment changes.  Returns the number of iterations run.
 * obj_trace (nullable, length max_iter) receives the objective after each
 * assignment step.  C [nlist x D] fp64 out. */
int oracle_kmeans(const float* T, int64_t nt, int D, int nlist, const int64_t* init_rows,
                  const float* init_centroids, int max_iter, double* C, double* obj_trace);

/* Nearest-centroid assignment in fp64, ties -> lowest id. */
void oracle_assign(const float* X, int64_t n, int D, const double* C, int nlist, int32_t* assign);

/* RaBitQ encode (Eq. 1; NS factors): for row v with list a = assign[v]
 *   r_o = P^T x - c'_a  (fp64; c' = P^T c given as fp32 Cr, P:L324 restructuring)
 *   b_i = [r_o,i >= 0]; n_o = ||r_o||; rho_o = ||r_o||_1 / (sqrt(D) n_o), := 1 if n_o = 0
 * codes [n x W] uint32; n_o, rho_o rounded to fp32 (what the index stores). */
void oracle_encode(const float* X, int64_t n, int D, const float* P, const float* Cr,
                   const int32_t* assign, uint32_t* codes, float* n_o, float* rho_o);

/* IVF probing: d_j = ||q' - c'_j||^2 by direct
 * subtraction in fp64; the nprobe smallest by (d_j, j) ascending. */
void oracle_probe(const float* qr, int D, const float* Cr, int nlist, int nprobe, int32_t* probes);

/* Randomized 4-bit query quantization for one (query, list) pair (NS(2),
 * P:L213, R#2, R#10-12).  The pinned fp32 sequence:
 *   r_i = fl32(q'_i - c'_i); v_l = min r; v_r = max r;
 *   Delta = fl32(fl32(v_r - v_l) / 15);
 *   Delta == 0 -> qbar_i = 0, else
 *   qbar_i = min(15, floor(fl32(fl32(fl32(r_i - v_l) / Delta) + u_i)))
 *   u_i = (Philox(key, (i>>2, list_id, qglobal, 0x51554E54))[i&3] >> 8) * 2^-24
 *   key = (lo, hi) of (seed ^ 0x5241424954515155)
 *   S_q = sum qbar (int); nq2 = sum r_i^2 in fp64.
 * qbar [D] out. */
void oracle_quantize(const float* qr, const float* cr, int D, uint64_t seed, int32_t list_id,
                     int64_t qglobal, uint8_t* qbar, float* v_l, float* delta, int32_t* S_q,
                     double* nq2);

/* <b, qbar> and popcount(b) by plain per-dimension loops (Eq. 3,
 * 0/1 form). */
int64_t oracle_ip(const uint32_t* code, const uint8_t* qbar, int D, int64_t* pc);

/* Unbiased estimator of ||o_r - q||^2 and its error bound (NS(4), R#1, R#14):
 *   X     = (2 Delta ip + 2 v_l pc - Delta S_q - D v_l) / sqrt(D)   (= <xbar, qbar>)
 *   est   = n_o^2 + nq2 - 2 n_o X / rho_o
 *   bound = 2 n_o n_q eps0 sqrt(1 - rho_o^2) / (rho_o sqrt(D - 1))  (0 when D = 1)
 * all in fp64 from the stored fp32 n_o, rho_o. */
void oracle_estimate(int64_t ip, int64_t pc, int D, double n_o, double rho_o, double v_l,
                     double delta, int64_t S_q, double nq2, double eps0, double* est, double* bound);

/* Full-precision-query estimator variant: X = <xbar, r_q> exactly (used by
 * the estimator pins as the "exact-query" reference and as NEXT-1). */
void oracle_estimate_fullq(const uint32_t* code, const double* rq, int D, double n_o, double rho_o,
                           double eps0, double* est, double* bound);

/* The whole search hot path for nq queries over one index (shard), the
 * paper's three stages with the NS steps:
 *   O-S1 q' = P^T q (fp64, rounded to fp32)     [qr_in overrides]
 *   O-S2 probes                                  [probes_in overrides]
 *   O-S3 quantize per (q, list)                  (Philox ctr uses qid_base + qi)
 *   O-S4 ip, est, bound for every vector of every probed list
 *   O-S5 top-M by (key, id), key = est (rank_key 0) or est - bound (rank_key 1)
 *   qmode 1 (NEXT-1): no query quantization, est from <x-bar, r_q> with the exact
 *        residual (oracle_estimate_fullq) instead of O-S3/O-S4's 4-bit form
 *   O-S5b rerank_mode 1 (NEXT-4, rank_key 0 only): keep the top-M candidates
 *        with est - bound <= tau, tau = k-th smallest est + bound; 0: keep all
 *   O-S6 exact squared L2 on raw vectors (fp64), top-k by (d, id); pad (-1, +inf)
 *        n_reranked [nq] (nullable): candidates re-ranked per query
 * Index arrays are in list order: list_off [nlist+1], list_ids [n] (global
 * ids), codes [n x W], n_o/rho_o [n].  Raw vectors X [n x D] are indexed by
 * local row = id - id_offset.  Outputs ids/dists [nq x k].  Optional debug
 * outputs (nullable): probes_out [nq x nprobe], topm_ids/topm_est [nq x M]
 * (padded -1 / +inf).  OpenMP over queries (num_threads <= 0: runtime default).
 * Returns 0, or -1 on bad arguments. */
int oracle_search(const float* Q, int64_t nq, int D, const float* P, const float* Cr, int nlist,
                  const int64_t* list_off, const int64_t* list_ids, const uint32_t* codes,
                  const float* n_o, const float* rho_o, const float* X, int64_t id_offset,
                  int k, int nprobe, int M, uint64_t seed, int64_t qid_base, int rank_key,
                  double eps0, const float* qr_in, const int32_t* probes_in, int num_threads,
                  int64_t* ids, float* dists, int32_t* probes_out, int64_t* topm_ids,
                  double* topm_est, int rerank_mode, int64_t* n_reranked, int qmode);

/* Fine ranking of given candidates (O-S6): exact squared L2 in fp64
 * between q and the raw vectors X[cand - id_offset] (cand = -1 skipped),
 * top-k by (d, id), padded (-1, +inf).  cand [nq x M] -> ids/dists [nq x k]. */
void oracle_rerank(const float* Q, int64_t nq, int D, const float* X, int64_t id_offset,
                   const int64_t* cand, int M, int k, int64_t* ids, float* dists);

/* Merge G per-shard top-k lists into the global top-k by (d, id) (P:L405-407,
 * NS "merges top-k"; R#20).  in_* [G x nq x k] -> out_* [nq x k]. */
void oracle_merge_topk(const int64_t* in_ids, const float* in_d, int G, int64_t nq, int k,
                       int64_t* out_ids, float* out_d);

/* Exact kNN by brute force in fp64, ties -> lower id. */
void oracle_bruteforce(const float* X, int64_t n, int D, const float* Q, int64_t nq, int k,
                       int num_threads, int64_t* ids, double* dists);

#ifdef __cplusplus
}
#endif
#endif
