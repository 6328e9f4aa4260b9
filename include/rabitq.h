/*
 * rabitq.h -- C ABI of the B200-native IVF-RaBitQ search hot path
 *             (librabitq.so, built from paper_2605_16007_b200/csrc).
 *
 * The calls follow the paper's problem statement (arxiv 2605.16007, PAPER.md):
 *   - P:L147-150 [sec 2.1.1]  corpus X of N vectors in R^D, query q, distance d
 *   - P:L156-159 [sec 2.1.2]  index construction: k-means -> nList centroids,
 *                             each vector to the list of its nearest centroid
 *   - P:L161-163 [sec 2.1.2]  query processing: top-nProbe nearest lists
 *   - P:L197-209 [sec 2.2.1]  RaBitQ rotation P, sign codes (Eq. 1), per-vector
 *                             constants (here ||o_r - c|| and <obar, o>, BASELINE.json north_star)
 *   - P:L211-234 [sec 2.2.2]  code x query inner products (Eq. 3) -> estimator
 *   - P:L239-246 [sec 2.2.3]  probe -> coarse top-M -> exact re-rank top-K
 *   - P:L397-407 [sec 3.4]    lists sharded across devices, results aggregated
 * and BASELINE.json north_star (rabitq_build(X, nlist, seed),
 * rabitq_search(Q, k, nprobe, n_rerank) -> ids, distances).
 *
 * General conventions
 *   - Every call returns a rabitq_status; on failure rabitq_last_error()
 *     returns a thread-local message.  No C++ exception crosses this ABI.
 *   - Pointers to vectors/results may be HOST or DEVICE memory (classified
 *     with cudaPointerGetAttributes); device pointers must live on the
 *     index's device.  Layouts are row-major and contiguous.
 *   - The caller owns every array it passes in; the index owns everything it
 *     allocates (released by rabitq_free).
 *   - Rotation convention: x' = P^T x (row form x'^T = x^T P); P is stored
 *     row-major fp32 [D x D].  Codes: W = ceil(D/32) uint32 words per vector,
 *     bit i = bit (i & 31) of word (i >> 5), 1 <=> rotated residual >= 0.
 *   - Distances returned are exact SQUARED L2 in fp32; per query the k
 *     results are ascending by (distance, id); missing results are padded
 *     with id = -1, distance = +INF.
 *   - Determinism: results are a pure function of (index contents, Q, k,
 *     nprobe, n_rerank, query_id_base, rank_key); they do not depend on the
 *     scan path, work partition, stream or batch split.  The randomized
 *     query quantizer draws from Philox4x32-10 with counter
 *     (dim/4, list id, query_id_base + query row, 'QUNT') and key
 *     seed ^ 0x5241424954515155 (R#12).
 */
#ifndef RABITQ_H
#define RABITQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RABITQ_OK = 0,
    RABITQ_ERR_INVALID_ARGUMENT = 1, /* sizes / parameters out of range                 */
    RABITQ_ERR_INVALID_DATA = 2,     /* non-finite input vectors                          */
    RABITQ_ERR_OUT_OF_MEMORY = 3,    /* device allocation failed; nothing is leaked       */
    RABITQ_ERR_CUDA = 4,             /* CUDA runtime / kernel error (message has details) */
    RABITQ_ERR_NCCL = 5,             /* NCCL error in a collective call                   */
    RABITQ_ERR_UNSUPPORTED = 6,      /* no usable sm_100 device, or option not supported  */
    RABITQ_ERR_INTERNAL = 7
} rabitq_status;

typedef struct rabitq_index rabitq_index; /* opaque; owns device memory */
typedef struct rabitq_comm rabitq_comm;   /* opaque; an NCCL communicator + rank info */

/* ---------------------------------------------------------------- build -- */
typedef struct {
    int32_t kmeans_iters;         /* Lloyd iterations, 0 -> 25 (R#6)                    */
    int64_t train_size;           /* k-means training rows, 0 -> min(n, 256 * nlist)             */
    const float* init_centroids;  /* nullable [nlist x d] ORIGINAL-space initial centroids       */
    int32_t borrow_vectors;       /* 0: copy X for re-rank (X may be freed after build);
                                     1: borrow X (must be a DEVICE pointer outliving the index)  */
    int64_t id_offset;            /* global id of row 0 (sharded builds); ids = id_offset + row  */
    const float* rotation;        /* nullable [d x d]: use this P instead of generating it       */
    const float* centroids_rot;   /* nullable [nlist x d] ROTATED centroids c' = P^T c: skip
                                     k-means (sharded builds take rank 0's centroids)            */
    int32_t device;               /* CUDA device ordinal, -1 -> current device                   */
} rabitq_build_opts;

/* Build an IVF-RaBitQ index over X [n x d] fp32:
 * Haar-random P (seeded fp64 QR on the host), k-means in the rotated space
 * on the GPU, nearest-centroid assignment, sign codes of r_o = P^T x - c'
 * and the factors n_o = ||r_o|| = ||o_r - c|| and rho_o = <obar, o> =
 * ||r_o||_1 / (sqrt(d) n_o) (1 if n_o = 0).  Lists hold ids ascending.
 * nlist = 0 means AUTO ceil(sqrt(n)).
 * Errors: d < 1, nlist < 0, n < nlist, n >= 2^32 -> INVALID_ARGUMENT;
 * non-finite X -> INVALID_DATA.  On failure *out = NULL (no partial index). */
rabitq_status rabitq_build(const float* X, int64_t n, int32_t d, int32_t nlist, uint64_t seed,
                           rabitq_index** out);
rabitq_status rabitq_build_ex(const float* X, int64_t n, int32_t d, int32_t nlist, uint64_t seed,
                              const rabitq_build_opts* opts, rabitq_index** out);
void rabitq_build_opts_default(rabitq_build_opts* opts);

/* --------------------------------------------------------------- search -- */
typedef enum { RABITQ_SCAN_AUTO = 0, RABITQ_SCAN_POPC = 1, RABITQ_SCAN_IMMA = 2 } rabitq_scan_path;
typedef enum { RABITQ_RANK_EST = 0, RABITQ_RANK_LOWER_BOUND = 1 } rabitq_rank_key;
typedef enum { RABITQ_RERANK_FIXED = 0, RABITQ_RERANK_BOUND = 1 } rabitq_rerank_mode;

/* Optional capture of the intermediate stages (parity harness).  Every
 * non-NULL member is filled (host or device memory); sizes in brackets. */
typedef struct {
    float* qrot;           /* [nq x d]            q' = P^T q (stage S1)                       */
    int32_t* probes;       /* [nq x nprobe]       probed lists, ascending (d, list) (S2-S3)   */
    uint8_t* qbar;         /* [nq x nprobe x d]   4-bit quantized query per (q, probe) (S4)   */
    float* qscal;          /* [nq x nprobe x 4]   v_l, Delta, ||r_q||^2, S_q (as float) (S4)  */
    int64_t* topm_ids;     /* [nq x n_rerank]     coarse top-M ids, ascending (key, id) (S8)  */
    float* topm_est;       /* [nq x n_rerank]     their estimated distances                  */
    float* topm_bound;     /* [nq x n_rerank]     their error bounds                          */
    float* tau;            /* [nq]                pruning threshold seeded from nearest lists */
    int32_t* survivors;    /* [nq]                candidates kept by the threshold            */
    int32_t* retries;      /* [1]                 overflow re-scans performed                 */
    /* Scan dump (single internal batch only): for every flattened work item i
     * (pair p = (q, probe) in query-major order, 32-slot block b of list
     * probes[p]; items of pair p are [off_p, off_p + ceil(size/32)), off_p the
     * exclusive prefix sum) and lane l, entry i*32 + l holds the integer inner
     * product <b, qbar> (-1 for pad slots) and the estimate of slot 32 b + l
     * of the list.  DEVICE memory, capacity scan_dump_cap entries. */
    int32_t* scan_ip;
    float* scan_est;
    int64_t scan_dump_cap;
} rabitq_debug;

/* Optional per-call measurement (host memory), filled when the call returns.
 * Stage times come from CUDA events recorded on the call's stream around each
 * stage (summed over internal query batches). */
#define RABITQ_NSTAGES 8
typedef struct {
    float stage_ms[RABITQ_NSTAGES]; /* 0 rotate, 1 probe GEMM+select, 2 quantize, 3 plan,
                                       4 threshold seed, 5 scan (+estimator), 6 overflow
                                       re-scans, 7 top-M select + exact re-rank         */
    int64_t pairs;                  /* (query, vector) pairs scanned by the first scan   */
    int64_t survivors;              /* candidates kept by the threshold, all queries     */
    int64_t max_survivors;          /* largest per-query survivor count                  */
    int32_t retries;                /* overflow re-scans                                 */
    int32_t kernel_launches;        /* librabitq kernels launched by this call           */
    int32_t scan_path_used;         /* 1 popc, 2 imma (CUDA-core survivor test), 3 imma with
                                       the folded tensor-core survivor test             */
    int32_t batches;                /* internal query batches                            */
    int64_t reranked;               /* candidates whose exact distance was taken (rerank 1) */
    float dense_ms;                 /* the dense nearest-list re-rank block (tgemm_dist1), which runs on
                                       the side stream beside stages 2-5 (not in stage_ms)             */
} rabitq_profile;

typedef struct {
    int32_t scan_path;       /* rabitq_scan_path; AUTO picks by workload                       */
    int32_t rank_key;        /* rabitq_rank_key; default EST (R#15)                  */
    float eps0;              /* error-bound confidence, 0 -> 1.9 (R#14)                        */
    int64_t query_id_base;   /* global index of Q row 0 (Philox counter)                       */
    int32_t cap_per_query;   /* survivor buffer per query, 0 -> auto (max(8192, 16M)); clamped to
                                >= 2 n_rerank; overflowing queries are re-scanned with a tighter
                                threshold until they fit                                       */
    int32_t seed_max;        /* size of the per-query sample of probed vectors that seeds the
                                pruning threshold, 0 -> auto: d <= 128 on the tensor
                                cores 8192 vectors of the nearest lists; else about 20 P / T,
                                capped at 16384 (P = probed vectors, T = target survivors).
                                Results never depend on it                                     */
    void* stream;            /* cudaStream_t to run on (NULL -> the index's stream); outputs
                                in device memory are valid after that stream synchronizes     */
    rabitq_debug* debug;     /* nullable                                                       */
    rabitq_profile* profile; /* nullable, host memory                                          */
    int32_t rerank;          /* 0: re-rank the n_rerank best estimates (default);
                                1: bound-driven: of those, only the ones with
                                est - bound <= the k-th smallest est + bound (bound = the
                                estimator's error bound at eps0, NS(4)); changes results when a
                                bound is violated at the boundary.  Requires rank_key EST. */
    int32_t query_bits;      /* 0 or 4: the 4-bit randomized query (NS(2), default); 32: the
                                unquantized query: the estimator
                                takes <x-bar, r_q> from r_q in 24-bit fixed point (error <= 1e-6
                                n_o n_q), no Philox draws; grouped tensor-core scan only (d <= 1024,
                                scan_path AUTO or IMMA), UNSUPPORTED otherwise */
    uint32_t variant;        /* 0 (default) or an OR of RABITQ_VARIANT_*: alternative execution
                                paths of the same computation (parity tests prove them
                                bit-identical to the default); never changes results        */
    const int32_t* probes_in;/* nullable [nq x nprobe] (host or device): the probed lists of each
                                query, e.g. from rabitq_probe; stage S2-S3 is
                                skipped.  Ids outside [0, nlist) -> INVALID_ARGUMENT.  Results
                                equal the default search when these are rabitq_probe's lists */
    int32_t query_split;     /* rabitq_search_sharded only: 0 every rank probes every query;
                                1 rank g probes queries [g c, (g+1) c), c = ceil(nq / G), and
                                the probe lists are all-gathered (one ncclAllGather of
                                nq x nprobe int32) -- the probe GEMM is split G ways
                                (SURVEY 8(e)); results are identical                          */
    int32_t graph;           /* 1: latency mode for a single-batch call without
                                debug / profile / rerank / probes_in: the whole path is captured
                                once as a CUDA graph (no host synchronisation inside; sizes from
                                host bounds) and replayed per call -- one input copy, one graph
                                launch, one output copy, one synchronisation; a batch whose
                                survivor buffers overflowed is re-run on the normal path, so
                                results are identical.  Graphs are cached per index and shape. */
} rabitq_search_opts;

/* rabitq_search_opts.variant bits (results are identical with any of them) */
#define RABITQ_VARIANT_RADIX_PROBE 1u        /* probe top-nprobe by the radix select only        */
#define RABITQ_VARIANT_EXPAND_IN_KERNEL 2u   /* grouped scan expands the codes into TMEM itself
                                                 (ignores the index's expanded-code copy)        */
#define RABITQ_VARIANT_NO_DENSE_RERANK 4u    /* exact gather of every re-rank candidate          */
#define RABITQ_VARIANT_GENERIC_SCAN 8u       /* d <= 128: the generic grouped scan kernel instead
                                                 of the small-K one                              */
#define RABITQ_VARIANT_UNIFORM_SEED 16u      /* d <= 128, tensor-core scan: threshold from a uniform
                                                 prefix sample of every probed list (the d > 128
                                                 seeding, also used when list sizes are skewed)
                                                 instead of the nearest lists; implies NO_FOLD   */
#define RABITQ_VARIANT_NO_FOLD 32u           /* d <= 128, tensor-core scan: survivor test on the
                                                 CUDA cores (scan_small_kernel) instead of the
                                                 tensor-core folded test (scan_fold_kernel, which
                                                 runs with the nearest-list threshold only)      */
#define RABITQ_VARIANT_FOLD_INPLACE 64u      /* folded scan: 2 deferred records per CTA instead of
                                                 32768, so that nearly every flagged pair takes the
                                                 region-full path (keys computed in place)        */

/* Search nq queries Q [nq x d] fp32: rotate, probe the nprobe
 * nearest lists, 4-bit Philox-randomized query quantization per (q, list),
 * 1-bit code scan with the unbiased estimator + error bound, per-query
 * top-n_rerank, exact-L2 re-rank from the fp32 vectors in HBM, top-k.
 * ids [nq x k] int64 (global ids), dists [nq x k] fp32 squared L2.
 * nprobe = 0 means AUTO ceil(0.05 nlist).  nq = 0 is OK (no work).
 * Errors: k < 1, n_rerank < k, nprobe > nlist, nq < 0 -> INVALID_ARGUMENT;
 * non-finite Q -> INVALID_DATA.  On failure outputs are unspecified and the
 * index is unchanged.  Synchronous w.r.t. host output buffers. */
rabitq_status rabitq_search(const rabitq_index* idx, const float* Q, int64_t nq, int32_t k,
                            int32_t nprobe, int32_t n_rerank, int64_t* ids, float* dists);
rabitq_status rabitq_search_ex(const rabitq_index* idx, const float* Q, int64_t nq, int32_t k,
                               int32_t nprobe, int32_t n_rerank, const rabitq_search_opts* opts,
                               int64_t* ids, float* dists);
void rabitq_search_opts_default(rabitq_search_opts* opts);

/* Stages S1-S3 only: rotate Q [nq x d] and
 * write each query's nprobe nearest lists, ascending by (distance, list id),
 * to probes [nq x nprobe] int32 (host or device).  stream: cudaStream_t or NULL
 * (the index's stream); synchronous w.r.t. host buffers.  nprobe = 0 means AUTO.
 * Errors: nprobe > nlist, nq < 0 -> INVALID_ARGUMENT; non-finite Q ->
 * INVALID_DATA. */
rabitq_status rabitq_probe(const rabitq_index* idx, const float* Q, int64_t nq, int32_t nprobe, int32_t* probes,
                           void* stream);

/* ----------------------------------------------------- info / export -- */
typedef struct {
    int32_t d, W, nlist, device;
    int64_t n, id_offset, max_list;
    int64_t bytes_codes, bytes_factors, bytes_ids, bytes_vectors, bytes_total;
    int32_t vectors_borrowed;
    /* derived copies built when they fit (both included in bytes_total):
     * the codes expanded to s8 {0, -1} (the grouped tensor-core scan's A operand,
     * loaded by TMA) and the vectors in slot order minus their centroid (the
     * dense re-rank block); 0 when absent */
    int64_t bytes_codes8, bytes_slot_vectors;
} rabitq_index_info_t;
rabitq_status rabitq_index_info(const rabitq_index* idx, rabitq_index_info_t* out);

/* Copies the index into caller buffers (host or device); NULL members are
 * skipped.  Arrays are in LIST order (list j = [list_off[j], list_off[j+1])). */
typedef struct {
    float* rotation;      /* [d x d]        P                                   */
    float* centroids;     /* [nlist x d]    c' = P^T c                          */
    int64_t* list_off;    /* [nlist + 1]                                        */
    int64_t* ids;         /* [n]            global ids, ascending within a list */
    uint32_t* codes;      /* [n x W]                                            */
    float* n_o;           /* [n]            ||o_r - c||                         */
    float* rho;           /* [n]            <obar, o>                           */
} rabitq_export_t;
rabitq_status rabitq_index_export(const rabitq_index* idx, rabitq_export_t* out);

void rabitq_free(rabitq_index* idx); /* NULL is a no-op */
const char* rabitq_last_error(void);
const char* rabitq_version(void);

/* Device self-check of an arithmetic identity the search path relies on
 * (diagnostics; no index needed).  what = 1: the quantizer's reciprocal
 * division (search.cu div_rcp_rn, R#11: t = fl(x / Delta) must equal the IEEE
 * quotient) against __fdiv_rn on n seeded random (x, Delta) pairs drawn from
 * the quantizer's domain (Delta > 0 normal, 0 <= x / Delta <= 15.01) plus
 * arbitrary bit patterns with quotients in range.  *mismatches (host) receives
 * the number of differing quotients.  Runs on the current CUDA device.
 * Errors: what unknown or mismatches NULL -> INVALID_ARGUMENT. */
rabitq_status rabitq_selftest(int32_t what, uint64_t n, uint64_t seed, uint64_t* mismatches);

/* ------------------------------------------ multi-GPU -- */
/* One process per GPU.  Rank 0 calls rabitq_comm_unique_id, the id travels
 * through the caller's process group (e.g. torch.distributed), every rank
 * calls rabitq_comm_init.  A sharded index is one rabitq_index per rank over
 * the rank's contiguous id slice (build with opts.id_offset, shared rotation
 * and centroids).  rabitq_search_sharded is collective: identical Q, k,
 * nprobe, n_rerank on every rank; each rank searches its shard, the per-rank
 * top-k (dist, id) are exchanged with ncclAllGather over NVLink and merged by
 * (dist, id); every rank returns the same global result. */
rabitq_status rabitq_comm_unique_id(uint8_t uid[128]);
rabitq_status rabitq_comm_init(const uint8_t uid[128], int32_t rank, int32_t world, int32_t device,
                               rabitq_comm** out);
void rabitq_comm_free(rabitq_comm* comm);
rabitq_status rabitq_search_sharded(const rabitq_index* shard, rabitq_comm* comm, const float* Q,
                                    int64_t nq, int32_t k, int32_t nprobe, int32_t n_rerank,
                                    const rabitq_search_opts* opts, int64_t* ids, float* dists);

/* Merge G per-shard top-k lists in_ids/in_d [G x nq x k] (DEVICE memory)
 * into out_ids/out_d [nq x k] (DEVICE) by (dist, id) on `stream`. */
rabitq_status rabitq_merge_topk(const int64_t* in_ids, const float* in_d, int32_t G, int64_t nq,
                                int32_t k, int64_t* out_ids, float* out_d, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RABITQ_H */
