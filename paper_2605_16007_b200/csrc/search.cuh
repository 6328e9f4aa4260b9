// search.cuh -- argument blocks shared by the scan kernels (popc: search.cu,
// tcgen05 IMMA: scan_imma.cu) and the host orchestration.
#pragma once
#include <nvtx3/nvToolsExt.h>

#include "index.cuh"

namespace rabitq {

struct ColC {      // per grouped row (query, list) constants of the grouped scan epilogue
    float a, b, K; // PairC a, b, K (estimator)
    float U;       // fast survivor test: A - f t <= U, U = tau - ||r_q||^2 + rounding margin
    float nq2;     // ||r_q||^2
    float tau;     // threshold of the column's query
    int q;         // query (-1: empty column)
    int pair;      // (query, probe) pair index
};

// Column constants of the grouped scan as stored (global and shared memory):
// two grouped rows per 64-byte record, so that the fast test of columns 2p,
// 2p + 1 takes (-a, b) and (-K, U) of both with two 16-byte loads, already
// paired for the packed FP32 ops (FFMA2 / FADD2)
struct ColPair {
    float na[2], b[2], nK[2], U[2];
    float nq2[2], tau[2];
    int q[2], pair[2];
};

struct ScanArgs {
    const int32_t* probes;     // [npairs] list of each (q, probe) pair
    int64_t npairs;
    int nprobe;
    const int64_t* item_off;   // [npairs + 1] exclusive scan of 32-slot blocks per pair
    const int64_t* list_off;
    const int64_t* slot_off;
    const uint32_t* codes;
    const float2* fac;
    const float* g1;
    const uint32_t* rows;
    const uint4* planes;       // [npairs][W] {plane0..3} per 32-dim word
    const float4* qscal;       // [npairs] {v_l, Delta, ||r_q||^2, S_q}
    const float* tau;          // [nq] float threshold
    const uint64_t* tau64;     // [nq] 64-bit (key, row) threshold (retry)
    const int* flags;          // [nq] retry flags
    int* cnt;                  // [nq] survivors appended
    uint64_t* buf;             // [nq x cap] survivor keys (orderable key << 32 | row)
    int cap;
    int D, W;
    float eps0;
    int32_t* dump_ip;          // debug: [items x 32] ip per (item, lane)
    float* dump_est;
    int64_t dump_cap;
    // grouped tcgen05 path (scan_imma.cu)
    int nlist;
    int Dp;                    // D rounded up to 32 (K of the int8 MMA)
    const int64_t* gstart;     // [nlist + 1] first grouped row of each list's pairs (multiple of 16)
    const int64_t* gcount;     // [nlist] grouped rows of each list (its region is rounded up to 16 rows)
    int64_t nrows;             // grouped rows allocated (qbar8 / gpair / column constants)
    const int32_t* gpair;      // [npairs] pair index of each grouped row
    const uint8_t* qbar8;      // [(npairs + 128) x Dp] quantized queries, grouped by list
    const int64_t* list_items; // [nlist + 1] prefix of (128-vector tile, 128-query group) items
    const uint16_t* pcnt;      // [nslots] popcount of each code
    const uint8_t* codes8;     // [nslots + 128][Dp] expanded codes (nullable: expanded in the kernel)
    int64_t nslots;
    const ColPair* gcolp;      // [nrows / 2] column constants in grouped order
    const float* list_amax;    // [nlist] max n_o^2 of each list (fast-test margin)
    long long* trace;          // diagnostics (RABITQ_SCAN_TRACE): clock64 stamps of CTA 0, [trace_n][16]
    int trace_n;
    // dense key dump (threshold-seeding sample scan): key of every scanned pair
    // at dense_keys[dense_base[q] + dense_off[pair] + v]
    uint32_t* dense_keys;
    const int64_t* dense_base;  // [nq] first key of each query
    const int64_t* dense_off;   // [npairs] offset of each (query, probe) pair within its query
    int full;                   // 1: unquantized query (NEXT-1), 4 digit rows per pair (npairs = rows)
    int small;                  // 1: Dp <= 128 may take the small-K scan (scan_small_kernel)
    int f8;                     // 1: e4m3 operands (.kind::f8f6f4): Dp <= 128, 4-bit query (codes8 / qbar8 bytes)
    int64_t items_bound;        // upper bound on the grouping's work items (small-K item table)
    int fold;                   // 1: the small-K main scan tests survivors on the tensor cores (scan_fold_kernel)
    long long* fold_tl;         // diagnostics (-DRABITQ_DIAG, RABITQ_FOLD_TIMELINE): clock64 stamps of CTA 0, [16][1024]
    uint4* fold_defer;          // folded scan: per-CTA regions of deferred flagged records (set by scan_imma)
    int fold_defer_cap;         // records per CTA
    int fold_diag;              // diagnostics (-DRABITQ_DIAG, RABITQ_FOLD_DIAG): 1 no slow path, 2 no row ip
};

template <typename T>
struct WBuf {  // stream-ordered workspace buffer
    T* p = nullptr;
    cudaStream_t st = nullptr;
    void alloc(size_t count, cudaStream_t s) {
        st = s;
        if (count) RQ_CUDA(cudaMallocAsync(&p, count * sizeof(T), s));
    }
    ~WBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

// list grouping of the (query, probe) pairs for the grouped scan
struct Groups {
    WBuf<int64_t> gcount, gstart, list_items, itemc;
    WBuf<int32_t> gfill, gpos, gpair;
    WBuf<uint8_t> qbar8;
    int Dp = 0;
    int64_t nrows = 0;  // grouped rows allocated (each list's region padded to 16 rows)
    bool ta = false;    // A operand = the index's expanded codes by TMA (else expanded in the kernel)
    int64_t n = 0;  // grouped pairs
    int rows = 1;   // B rows per pair (4: the unquantized query's digit rows, NEXT-1)
};
void prepare_groups(const rabitq_index* idx, const int32_t* probes, int64_t n, const int32_t* sub, Groups& g,
                    cudaStream_t st, int& launches, int rows, bool ta);
int64_t regroup_flagged(const rabitq_index* idx, const int32_t* probes, int64_t npairs, int nprobe, const int* flags,
                        int max_rank, const Groups& full, Groups& sub, cudaStream_t st, int& launches);
bool imma_wanted(const rabitq_index* idx, int64_t npairs, int scan_path);
int64_t item_bound(const rabitq_index* idx, int64_t rows, int64_t max_group);
// build time: idx->codes8 (the grouped scan's A operand, loaded by TMA) when it fits
void expand_codes(rabitq_index* idx, cudaStream_t st);
cudaStream_t side_stream(const rabitq_index* idx);

struct RerankArgs {
    const int* cnt;
    const uint64_t* buf;
    int cap, M, k, D;
    const float* Q;            // [nq x D] unrotated queries (device)
    const float* X;            // [n x D] vectors (device)
    int64_t id_offset;
    int64_t* ids;
    float* dists;
    int64_t* topm_ids;
    float* topm_est;
    float* topm_bound;
    int rank_key;
    float eps0;
    const uint32_t* slot_of_row;
    const int64_t* slot_off;
    int nlist;
    const int32_t* probes;
    int nprobe;
    const float4* qscal;
    const float* g1;
    const int32_t* order;      // [nq] block -> query (queries sharing their nearest list run together)
    // dense re-rank of the nearest list (nullable): distance of query q to the v-th
    // vector of its nearest list at dense_d[dpos[q] + v] (dpos[q] < 0: not covered)
    const float* dense_d;
    const int64_t* dpos;
    const int64_t* list_off;
    const float* n_o;          // [nslots] ||o - c|| (the dense distances' error scale)
    // row staging for the exact gather: each warp streams its candidates' rows
    // into a private ring of `slots` shared-memory rows by bulk async copies
    // (0: register loads; needs D % 4 == 0, D <= 1024, 16-byte aligned X)
    int slots;
    // bound-driven re-rank set (NEXT-4): keep est - bound <= k-th smallest est + bound
    int adaptive;
    unsigned long long* reranked;  // [1] candidates kept, summed over queries (adaptive only)
};

struct SearchCfg {
    int scan_path = 0;   // 0 auto, 1 popc, 2 imma
    int rank_key = 0;
    float eps0 = 1.9f;
    int cap = 0;
    int seed_max = 0;
    int refine_rank = 0;  // > 0: refine tau with a tensor-core pass over each query's nearest lists
    int rerank = 0;       // 1: bound-driven re-rank set (NEXT-4)
    int full = 0;         // 1: unquantized query (NEXT-1), grouped tensor-core scan
    uint32_t variant = 0; // result-invariant execution variants (rabitq_search_opts.variant)
    const int32_t* probes_in = nullptr;  // DEVICE [nq x nprobe]: skip S2-S3 (query-split probing)
    // latency mode (NEXT-2, CUDA-graph capturable): no host synchronisation -- sizes from host-side
    // bounds, no side stream, one overflow check whose counters go to `flags_out` (host pinned, 8 ints:
    // [0] non-finite Q, [1] queries that need a re-scan); the caller re-runs the batch normally if set
    bool latency = false;
    int* flags_out = nullptr;
};

struct DebugOut {  // device-or-host pointers (cudaMemcpyDefault), all nullable
    float* qrot = nullptr;
    int32_t* probes = nullptr;
    uint8_t* qbar = nullptr;   // written by the quantize kernel directly: must be DEVICE
    float4* qscal = nullptr;
    int64_t* topm_ids = nullptr;  // DEVICE
    float* topm_est = nullptr;    // DEVICE
    float* topm_bound = nullptr;  // DEVICE
    float* tau = nullptr;
    int32_t* survivors = nullptr;
    int32_t* scan_ip = nullptr;   // DEVICE [scan_dump_cap]
    float* scan_est = nullptr;    // DEVICE
    int64_t scan_dump_cap = 0;
};

struct SearchStats {
    bool timing = false;       // record CUDA events per stage (rabitq_profile)
    float stage_ms[8] = {};
    int64_t pairs = 0;
    int64_t survivors = 0;
    int64_t max_survivors = 0;
    int retries = 0;
    int64_t reranked = 0;  // rerank 1: candidates re-ranked
    float dense_ms = 0.f;  // the dense re-rank block (side stream), when timing
    int launches = 0;
    int used_imma = 0;
    int batches = 0;
};

// per-stage CUDA events on the call's stream (rabitq_profile)
// and NVTX ranges named after the stages (host-side ranges around each stage's
// enqueue; visible to nsys / ncu --nvtx)
struct StageTimer {
    cudaEvent_t ev[9] = {};
    bool on = false;
    int open = -1;  // NVTX range currently pushed
    cudaStream_t st = nullptr;
    StageTimer(bool enable, cudaStream_t s) : on(enable), st(s) {
        if (on)
            for (auto& e : ev) RQ_CUDA(cudaEventCreate(&e));
    }
    void mark(int i) {
        static const char* kNames[8] = {"rabitq:S1 rotate",      "rabitq:S2-S3 probe",  "rabitq:S4 quantize",
                                        "rabitq:S5 plan",        "rabitq:S8a seed",     "rabitq:S6-S7 scan",
                                        "rabitq:overflow rescan", "rabitq:S8b-S9 select+rerank"};
        if (open >= 0) nvtxRangePop();
        open = -1;
        if (i < 8) {
            nvtxRangePushA(kNames[i]);
            open = i;
        }
        if (on) RQ_CUDA(cudaEventRecord(ev[i], st));
    }
    void accumulate(float* ms) {
        if (!on) return;
        RQ_CUDA(cudaEventSynchronize(ev[8]));
        for (int i = 0; i < 8; ++i) {
            float t = 0.0f;
            RQ_CUDA(cudaEventElapsedTime(&t, ev[i], ev[i + 1]));
            ms[i] += t;
        }
    }
    ~StageTimer() {
        if (open >= 0) nvtxRangePop();
        if (on)
            for (auto& e : ev) cudaEventDestroy(e);
    }
};
void rotate_probe(const rabitq_index* idx, const float* Q, int64_t nq, int nprobe, uint32_t variant, float* Qr,
                  int32_t* probes, cudaStream_t st, int& L, StageTimer* tm, bool latency = false);
void search_batch(const rabitq_index* idx, const float* Q, int64_t nq, int k, int nprobe, int M,
                  const SearchCfg& cfg, int64_t qid_base, int64_t* ids, float* dists, const DebugOut& dbg,
                  cudaStream_t st, SearchStats* stats);
void scan_imma(const ScanArgs& a, bool lb, bool dump, bool retry, cudaStream_t st, bool dense = false);
// list_items of a grouping for other list sizes (sample-scan view)
void group_items(const rabitq_index* idx, const int64_t* list_off, const Groups& g, WBuf<int64_t>& itemc,
                 WBuf<int64_t>& items, cudaStream_t st, int& launches);
uint64_t selftest_div(uint64_t n, uint64_t seed, cudaStream_t st);
void scan_popc_entry(const ScanArgs& a, bool lb, bool retry, bool dump, cudaStream_t st);
void check_probes(const int32_t* probes, int64_t n, int nlist, cudaStream_t st);
void probe_only(const rabitq_index* idx, const float* Q, int64_t nq, int nprobe, uint32_t variant, int32_t* probes,
                cudaStream_t st);
void merge_topk(const int64_t* in_ids, const float* in_d, int G, int64_t nq, int k, int64_t* out_ids,
                float* out_d, cudaStream_t st);

}  // namespace rabitq
