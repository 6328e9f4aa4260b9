// scan_imma.cu -- the grouped coarse scan on the 5th-generation tensor cores
// (NS(3) "when queries are grouped by shared list, a dense int8 tcgen05
// contraction of +-1 codes against quantized queries").
//
// Eq. (3) turns the per-pair bit count into an inner product, so
// for list j the inner products of ALL its vectors with ALL queries probing
// it form one integer matrix product
//        S[v, c] = sum_i b[v, i] * qbar[c, i]      (b in {0,1}, qbar in 0..15)
// A = codes of a 128-vector tile expanded bit -> byte in shared memory,
// B = the int8 quantized queries of up to 128 pairs grouped on that list,
// D = S in TMEM (int32, exact), K = D rounded up to 32.  The epilogue reads
// S back with tcgen05.ld and applies the same estimator + threshold as the
// popc scan (rabitq_est), so both paths produce bit-identical keys.
//
// Work item = (list, group of <= NG queries, range of <= 8 vector tiles); one
// persistent CTA per SM strides over the items.  The group's int8 query rows
// (B, every K chunk, 128-byte swizzle) are loaded ONCE per item by TMA and stay
// resident in shared memory (NG = 256 for D <= 512, 128 at D = 960); producer
// warps expand each 128-vector code tile (A) chunk by chunk into a 4-stage
// ring; a single thread issues the UMMAs into one of two TMEM accumulators
// (2 x 256 columns) while 8 epilogue warps drain the other.  UMMA N is the
// group size rounded up to 16, so empty columns cost nothing.
//
// This ignores query boundaries for scheduling and re-opens the
// list grouping the paper rejected for its NPU pipeline: on B200 it
// turns the bandwidth-bound scan into tensor-core work.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>

#include "search.cuh"
#include "tc.cuh"

namespace rabitq {
namespace {

constexpr int kTM = 128;                   // vectors per tile (UMMA M)
constexpr int kTN = 256;                   // grouped-row padding (>= max group size)
constexpr int kKC = 128;                   // bytes of K per chunk (one 128-byte swizzle row of B)
constexpr int kChunkCols = kKC / 4;        // TMEM columns of one A chunk (4 int8 per column)
constexpr int kMaxChunks = 8;              // Dp <= 1024
constexpr int kMaxSlots = 8;               // A ring slots in TMEM
constexpr int kBRes = 192 * 1024;          // resident query operand (all K chunks of one group)
constexpr int kMaxNG = 224;                // 2 NG accumulator columns + >= 2 A slots <= 512
constexpr int kBoxRows = 16;               // TMA box = 16 query rows x 128 bytes (group width granularity)
constexpr int kTilesPerItem = 8;           // vector tiles per work item (B loaded once per item)
constexpr int kProdWarps = 4;              // thread r expands code row r into TMEM lane r
constexpr int kMmaWarp = kProdWarps;       // warp 4 issues the UMMAs (and owns TMEM)
constexpr int kLoadWarp = kProdWarps + 1;  // warp 5 streams the query operand (TMA)
constexpr int kEpiWarp0 = kProdWarps + 2;  // warps 6..13
constexpr int kEpiWarps = 16;              // 4 per TMEM lane quarter, columns interleaved in chunks of kEC
constexpr int kEC = 16;                    // accumulator columns per epilogue step
constexpr int kNT = (kEpiWarp0 + kEpiWarps) * 32;  // 704 threads (80 registers)
constexpr int kTmemCols = 512;
constexpr int kPF = 8;                     // code-word prefetch ring (chunks in flight per producer thread)
constexpr int kSmemLimit = 227 * 1024;

// A operand by TMA (expanded codes in HBM, `ta`): A stages of one K chunk of a
// 128-vector tile in shared memory instead of the TMEM A slots and producers
constexpr int kAStage = kTM * kKC;  // 16 KB
constexpr int kMinAStages = 3;

// queries per group: all K chunks of a group fit the resident B region, and
// the double-buffered accumulator leaves TMEM room for >= 2 A slots (ta: B
// resident + >= 3 A stages + column constants fit shared memory; N <= 256)
__host__ __device__ inline int group_cols(int Dp, bool ta, int ngmax = kTN, int minst = kMinAStages) {
    const int nch = (Dp + kKC - 1) / kKC;
    if (ta) {
        int n = ngmax;
        while (n > kBoxRows && nch * n * kKC + minst * kAStage + 2 * n * (int)sizeof(ColC) + 2048 > kSmemLimit)
            n -= kBoxRows;
        return n;
    }
    int n = (kBRes / (nch * kKC)) / kBoxRows * kBoxRows;
    return n > kMaxNG ? kMaxNG : n;
}

// shared-memory / TMEM plan of one launch (host and device agree); slots = TMEM
// A slots, or (ta) shared-memory A stages
struct SmemPlan {
    int nchunks, NG, slots;
    uint32_t acc_cols, off_colc, off_raw, total;
};
__host__ __device__ inline SmemPlan smem_plan(int Dp, bool ta, int ngmax = kTN, int minst = kMinAStages) {
    SmemPlan p;
    p.nchunks = (Dp + kKC - 1) / kKC;
    p.NG = group_cols(Dp, ta, ngmax, minst);
    p.acc_cols = (uint32_t)((p.NG + 31) & ~31);  // per accumulator buffer
    const uint32_t bres = (uint32_t)(p.nchunks * p.NG * kKC);
    p.off_colc = bres;  // [2][NG / 2] ColPair
    if (ta) {
        p.off_raw = (p.off_colc + 2u * p.NG * (uint32_t)sizeof(ColC) + 1023u) & ~1023u;  // A stages, 1024-aligned
        int st = (int)(((uint32_t)kSmemLimit - 1024u - p.off_raw) / (uint32_t)kAStage);
        p.slots = st < kMaxSlots ? st : kMaxSlots;
        p.total = p.off_raw + (uint32_t)(p.slots * kAStage) + 1024u;
        return p;
    }
    int slots = (kTmemCols - 2 * (int)p.acc_cols) / kChunkCols;
    p.slots = slots < kMaxSlots ? slots : kMaxSlots;
    p.off_raw = p.off_colc + 2u * p.NG * (uint32_t)sizeof(ColC);  // [kPF][128 rows][4 words]
    p.total = p.off_raw + (uint32_t)(kPF * kTM * 16) + 1024u;
    return p;
}

// warp roles: (ta) no producers, a second loader warp streams A
__host__ __device__ constexpr int mma_warp(bool ta) { return ta ? 0 : kProdWarps; }
__host__ __device__ constexpr int load_warp(bool ta) { return mma_warp(ta) + 1; }
__host__ __device__ constexpr int loada_warp(bool ta) { return mma_warp(ta) + 2; }
__host__ __device__ constexpr int epi_warp0(bool ta) { return ta ? 3 : kProdWarps + 2; }
__host__ __device__ constexpr int n_threads(bool ta) { return (epi_warp0(ta) + kEpiWarps) * 32; }

struct Item {
    int j;
    int64_t L, t0, slot_base, grow0;
    int ntiles, ncols, ncols16, nboxes;
};

// item = (list, group of <= NG queries, range of <= kTilesPerItem vector tiles)
__device__ __forceinline__ Item decode_item(const ScanArgs& a, int NG, int64_t item) {
    int64_t lo = 0, hi = a.nlist;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(a.list_items + mid) <= item) lo = mid;
        else hi = mid;
    }
    Item it;
    it.j = (int)lo;
    it.L = __ldg(a.list_off + lo + 1) - __ldg(a.list_off + lo);
    const int64_t gs = __ldg(a.gstart + lo);
    const int64_t G = __ldg(a.gstart + lo + 1) - gs;
    const int64_t ntl = (it.L + kTM - 1) / kTM;
    const int64_t nti = (ntl + kTilesPerItem - 1) / kTilesPerItem;
    const int64_t local = item - __ldg(a.list_items + lo);
    const int64_t g = local / nti, ti = local % nti;
    it.t0 = ti * kTilesPerItem;
    const int64_t nt = ntl - it.t0;
    it.ntiles = (int)(nt < kTilesPerItem ? nt : kTilesPerItem);
    it.slot_base = __ldg(a.slot_off + lo);
    it.grow0 = gs + g * NG;
    const int64_t rem = G - g * NG;
    it.ncols = (int)(rem < NG ? rem : NG);
    it.ncols16 = (it.ncols + 15) & ~15;
    it.nboxes = (it.ncols + kBoxRows - 1) / kBoxRows;
    return it;
}

// 32 code bits -> 32 bytes in {0, -1} (s8), K order permuted: output byte
// k = 4 s + t (s = 0..7, t = 0..3) holds code bit 8 t + 7 - s, the sign bit of
// byte t of (x << s), replicated by PRMT.  The quantizer writes the query rows
// in the same K order, so the contraction is unchanged:
//   sum_k A[k] B[k] = - sum_i b_i qbar_i = -ip.
__device__ __forceinline__ uint32_t sgnrep(uint32_t y) {
    uint32_t r;
    asm("prmt.b32 %0, %1, 0, 0xBA98;" : "=r"(r) : "r"(y));
    return r;
}
__device__ __forceinline__ void expand32(uint32_t x, uint4& lo, uint4& hi) {
    lo.x = sgnrep(x);
    lo.y = sgnrep(x * 2u);
    lo.z = sgnrep(x * 4u);
    lo.w = sgnrep(x * 8u);
    hi.x = sgnrep(x * 16u);
    hi.y = sgnrep(x * 32u);
    hi.z = sgnrep(x * 64u);
    hi.w = sgnrep(x * 128u);
}

// fused estimator from the accumulator (acc = -ip: s8 codes in {0, -1}).
// 0x4B400000 + n is the float 1.5 2^23 + n exactly for |n| < 2^22, so ipn = -ip
// exactly; the rest is rabitq_est's arithmetic (a ip = (-a)(-ip) exactly).
__device__ __forceinline__ float est_of(uint32_t acc, const ColC& cc, float2 fac, float pcf) {
    const float ipn = __fsub_rn(__int_as_float(0x4B400000 + (int)acc), 12582912.0f);
    const float tt = __fmaf_rn(-cc.a, ipn, __fmaf_rn(cc.b, pcf, -cc.K));
    return __fmaf_rn(-fac.y, tt, __fadd_rn(fac.x, cc.nq2));
}

// Column constants in shared memory, two columns per 64-byte record so that
// the fast test of columns 2p, 2p+1 takes (-a, b) and (-K, U) of both with two
// 16-byte loads, already paired for the packed FP32 ops (FFMA2 / FADD2)
struct ColPair {
    float na[2], b[2], nK[2], U[2];
    float nq2[2], tau[2];
    int q[2], pair[2];
};
__device__ __forceinline__ void colp_put(ColPair* cp, int c, const ColC& x) {
    ColPair& P = cp[c >> 1];
    const int h = c & 1;
    P.na[h] = -x.a;
    P.b[h] = x.b;
    P.nK[h] = -x.K;
    P.U[h] = x.U;
    P.nq2[h] = x.nq2;
    P.tau[h] = x.tau;
    P.q[h] = x.q;
    P.pair[h] = x.pair;
}
__device__ __forceinline__ ColC colp_get(const ColPair* cp, int c) {  // negations are exact
    const ColPair& P = cp[c >> 1];
    const int h = c & 1;
    ColC x;
    x.a = -P.na[h];
    x.b = P.b[h];
    x.K = -P.nK[h];
    x.U = P.U[h];
    x.nq2 = P.nq2[h];
    x.tau = P.tau[h];
    x.q = P.q[h];
    x.pair = P.pair[h];
    return x;
}

// the same estimator from a float ipn (= -ip): est_of(acc) == est_ipn(exact float of acc)
__device__ __forceinline__ float est_ipn(float ipn, const ColC& cc, float2 fac, float pcf) {
    const float tt = __fmaf_rn(-cc.a, ipn, __fmaf_rn(cc.b, pcf, -cc.K));
    return __fmaf_rn(-fac.y, tt, __fadd_rn(fac.x, cc.nq2));
}
__device__ __forceinline__ float acc_f(uint32_t acc) {  // exact int32 -> float, |acc| < 2^22
    return __fsub_rn(__int_as_float(0x4B400000 + (int)acc), 12582912.0f);
}
// NEXT-1: -sum_i b_i X_i from the four 6-bit digit accumulators (|acc_k| < 2^16)
__device__ __forceinline__ float ipn_full(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
    return __fmaf_rn(262144.0f, acc_f(a3), __fmaf_rn(4096.0f, acc_f(a2), __fmaf_rn(64.0f, acc_f(a1), acc_f(a0))));
}

// eps0 n_q of a column (lower-bound rank key, R#15)
#define epsnq_of(cc) __fmul_rn(a.eps0, sqrtf((cc).nq2))

// clock stamps of CTA 0 (RABITQ_SCAN_TRACE diagnostics): row idx, column slot
// (compiled in with -DRABITQ_SCAN_TRACE only; the stamps cost issue slots)
#ifdef RABITQ_SCAN_TRACE
#define RQ_TR(slot, idx)                                                                            \
    do {                                                                                            \
        if (a.trace && blockIdx.x == 0 && (int64_t)(idx) < a.trace_n) a.trace[(int64_t)(idx) * 16 + (slot)] = clock64(); \
    } while (0)
#else
#define RQ_TR(slot, idx) \
    do {                 \
    } while (0)
#endif

// position of one K chunk in a CTA's work sequence (items strided by the grid)
struct Pos {
    int64_t item;
    Item it;
    int t, c;
};
__device__ __forceinline__ void pos_next(const ScanArgs& a, int NG, int nchunks, int64_t total, Pos& p) {
    if (++p.c < nchunks) return;
    p.c = 0;
    if (++p.t < p.it.ntiles) return;
    p.t = 0;
    p.item += gridDim.x;
    if (p.item < total) p.it = decode_item(a, NG, p.item);
}

// Warp-specialised persistent kernel, one CTA per SM.  TMEM (512 columns):
// two int32 accumulators of acc_cols columns + a ring of A slots (32 columns =
// one 128-byte K chunk of a 128-vector code tile each).
//   warps 0-3  producers: thread r expands code row r chunk by chunk (PRMT, see
//              expand32) straight into TMEM lane r of the next A slot
//              (tcgen05.st; code words prefetched two chunks ahead)
//   warp 4     MMA issuer: 4 UMMA (A from TMEM, B from shared memory, K = 32
//              each) per chunk into one of two accumulators per vector tile;
//              tcgen05.commit frees A slots, publishes accumulators and frees
//              each B chunk after the item's last tile used it
//   warp 5     query loader: TMA of the group's int8 query rows (B, resident per
//              item), chunk c of the next item as soon as chunk c is free
//   warps 6-13 epilogue: tcgen05.ld the int32 inner products, fused
//              estimator (+ bound), threshold, survivor append
template <bool kLB, bool kDump, bool kRetry, bool kDense, bool kTA, bool kFull>
__global__ __launch_bounds__(n_threads(kTA), 1) void scan_imma_kernel(const __grid_constant__ CUtensorMap tmapB,
                                                                      const __grid_constant__ CUtensorMap tmapA,
                                                                      ScanArgs a) {
    constexpr int kMmaWarp = mma_warp(kTA), kLoadWarp = load_warp(kTA), kLoadAWarp = loada_warp(kTA),
                  kEpiWarp0 = epi_warp0(kTA);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    const SmemPlan sp = smem_plan(a.Dp, kTA, a.ngmax, a.minst);
    uint8_t* Bres = smem;                                        // [nchunks][NG rows][128 B], 128-byte swizzle
    ColPair* colc = reinterpret_cast<ColPair*>(smem + sp.off_colc);  // [2][NG / 2]
    __shared__ __align__(8) uint64_t full_bar[kMaxSlots], empty_bar[kMaxSlots], accf_bar[2], acce_bar[2],
        bfull_bar[kMaxChunks], bfree_bar[kMaxChunks];
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nchunks = sp.nchunks, NG = sp.NG, nsl = sp.slots;
    if (warp == kMmaWarp) tc::tmem_alloc(&tmem_base_s, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s < nsl; ++s) {
            tc::mbar_init(&full_bar[s], 1);
            tc::mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&accf_bar[b], 1);
            tc::mbar_init(&acce_bar[b], kEpiWarps);
        }
        for (int c = 0; c < nchunks; ++c) {
            tc::mbar_init(&bfull_bar[c], 1);
            tc::mbar_init(&bfree_bar[c], 1);
        }
        tc::prefetch_tmap(&tmapB);
        if (kTA) tc::prefetch_tmap(&tmapA);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base_s;
    const uint32_t tmemA = tmem + 2u * sp.acc_cols;  // A slot s at columns tmemA + 32 s

    const int64_t total = a.list_items[a.nlist];
    const int bchunk = NG * kKC;  // bytes of one K chunk of the resident B

    if (!kTA && warp < kProdWarps) {
        // ================= producers =================
        const int r = tid;  // tile row = vector = TMEM lane
        const int W = a.W;
        const uint32_t lane_addr = (uint32_t)(warp * 32) << 16;
        uint32_t* raw = reinterpret_cast<uint32_t*>(smem + sp.off_raw);  // [kPF][128][4]
        // this thread's 4 code words of chunk p -> ring entry e (async, zero-filled past W)
        auto issue = [&](const Pos& p, int e) {
            if (p.item < total) {
                const int64_t slot = p.it.slot_base + (p.it.t0 + p.t) * kTM + r;  // slot_base multiple of 32
                const uint32_t* src = a.codes + (size_t)(slot >> 5) * W * 32 + (slot & 31);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int wd = 4 * p.c + k;
                    tc::cp_async4(raw + (e * kTM + r) * 4 + k, src + (size_t)min(wd, W - 1) * 32, wd < W ? 4u : 0u);
                }
            }
            tc::cp_async_commit();  // (possibly empty) group per chunk keeps the wait count uniform
        };
        Pos pf{(int64_t)blockIdx.x, Item{}, 0, 0};
        if (pf.item < total) pf.it = decode_item(a, NG, pf.item);
        Pos cur = pf;
        for (int i = 0; i < kPF - 1; ++i) {
            issue(pf, i);
            pos_next(a, NG, nchunks, total, pf);
        }
        int s = 0, e = 0;
        uint32_t u = 0;
        for (uint32_t gc = 0; cur.item < total; ++gc) {
            issue(pf, (e + kPF - 1) % kPF);  // kPF - 1 chunks ahead
            pos_next(a, NG, nchunks, total, pf);
            tc::cp_async_wait<kPF - 1>();  // this thread's words of chunk gc have landed
            const uint4 wv = *reinterpret_cast<const uint4*>(raw + (e * kTM + r) * 4);
            if (tid == 0) RQ_TR(0, gc);
            if (u > 0) tc::mbar_wait_backoff(&empty_bar[s], (u - 1) & 1);
            tc::fence_after_sync();
            if (tid == 0) RQ_TR(1, gc);
            const uint32_t dst = tmemA + (uint32_t)(s * kChunkCols) + lane_addr;
            uint4 lo, hi;
            expand32(wv.x, lo, hi);
            tc::tmem_st8(dst, lo, hi);
            expand32(wv.y, lo, hi);
            tc::tmem_st8(dst + 8, lo, hi);
            expand32(wv.z, lo, hi);
            tc::tmem_st8(dst + 16, lo, hi);
            expand32(wv.w, lo, hi);
            tc::tmem_st8(dst + 24, lo, hi);
            tc::tmem_st_wait();
            tc::fence_before_sync();
            if (tid == 0) RQ_TR(2, gc);
            tc::named_barrier(2, kProdWarps * 32);  // slot written by all 128 rows
            if (tid == 0) {
                tc::mbar_arrive(&full_bar[s]);
                RQ_TR(4, gc);
            }
            if (++s == nsl) {
                s = 0;
                ++u;
            }
            if (++e == kPF) e = 0;
            pos_next(a, NG, nchunks, total, cur);
        }
        tc::cp_async_wait<0>();
    } else if (warp == kMmaWarp) {
        // ================= MMA issuer =================
        uint32_t gc = 0, tcnt = 0, ic = 0, u = 0;
        int s = 0;
        const uint64_t bdesc0 = tc::smem_desc_sw128(tc::smem_u32(Bres));
        for (int64_t item = blockIdx.x; item < total; item += gridDim.x, ++ic) {
            const Item it = decode_item(a, NG, item);
            const uint32_t idesc = tc::idesc_i8(kTM, it.ncols16, /*a_signed=*/true);
            for (int t = 0; t < it.ntiles; ++t, ++tcnt) {
                const int b = tcnt & 1;
                const uint32_t ub = tcnt >> 1;
                if (lane == 0) RQ_TR(11, tcnt);
                if (ub > 0) tc::mbar_wait_backoff(&acce_bar[b], (ub - 1) & 1);
                if (lane == 0) RQ_TR(12, tcnt);
                tc::fence_after_sync();
                const uint32_t dacc = tmem + (uint32_t)b * sp.acc_cols;
                for (int c = 0; c < nchunks; ++c, ++gc) {
                    const int nks = min(kKC, a.Dp - c * kKC) / 32;
                    if (lane == 0) RQ_TR(7, gc);
                    if (t == 0) tc::mbar_wait(&bfull_bar[c], ic & 1);
                    tc::mbar_wait(&full_bar[s], u & 1);
                    tc::fence_after_sync();
                    if (lane == 0) RQ_TR(9, gc);
                    {
                        const uint64_t bd = bdesc0 + (uint64_t)((c * bchunk) >> 4);
                        if constexpr (kTA) {
                            // A stage s (TMA, 128-byte swizzle) free once these retire
                            const uint64_t ad = tc::smem_desc_sw128(tc::smem_u32(smem + sp.off_raw + s * kAStage));
                            tc::mma_i8_ss_chunk(dacc, ad, bd, idesc, c > 0 ? 1u : 0u, nks, &empty_bar[s]);
                        } else if (a.experiment & 2) {  // diagnostics: skip the UMMAs
                            const uint32_t aaddr = tmemA + (uint32_t)(s * kChunkCols);
                            if (c == 0) tc::mma_i8_ts_warp(dacc, aaddr, bd, idesc, 0u);
                            tc::commit_warp(&empty_bar[s]);
                        } else {
                            // nks UMMAs + commit: A slot s free once these retire
                            const uint32_t aaddr = tmemA + (uint32_t)(s * kChunkCols);
                            tc::mma_i8_ts_chunk(dacc, aaddr, bd, idesc, c > 0 ? 1u : 0u, nks, &empty_bar[s]);
                        }
                        if (t == it.ntiles - 1) tc::commit_warp(&bfree_bar[c]);  // B chunk c free for the next item
                        if (c == nchunks - 1) tc::commit_warp(&accf_bar[b]);     // accumulator b complete
                        if (lane == 0) RQ_TR(10, gc);
                    }
                    if (++s == nsl) {
                        s = 0;
                        ++u;
                    }
                }
            }
        }
    } else if (warp == kLoadWarp) {
        // ================= query operand loader =================
        if (lane == 0) {
            uint32_t ic = 0;
            for (int64_t item = blockIdx.x; item < total; item += gridDim.x, ++ic) {
                const Item it = decode_item(a, NG, item);
                for (int c = 0; c < nchunks; ++c) {
                    if (ic > 0) tc::mbar_wait_backoff(&bfree_bar[c], (ic - 1) & 1);  // previous item done with chunk c
                    tc::mbar_arrive_expect_tx(&bfull_bar[c], (uint32_t)(it.nboxes * kBoxRows * kKC));
                    for (int bx = 0; bx < it.nboxes; ++bx)
                        tc::tma_load_2d(Bres + c * bchunk + bx * kBoxRows * kKC, &tmapB, &bfull_bar[c], c * kKC,
                                        (int)(it.grow0 + bx * kBoxRows));
                }
            }
        }
    } else if (kTA && warp == kLoadAWarp) {
        // ================= code operand loader (A by TMA) =================
        if (lane == 0) {
            uint32_t gc = 0;
            for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
                const Item it = decode_item(a, NG, item);
                for (int t = 0; t < it.ntiles; ++t) {
                    const int row0 = (int)(it.slot_base + (it.t0 + t) * kTM);
                    for (int c = 0; c < nchunks; ++c, ++gc) {
                        const int s = (int)(gc % nsl);
                        const uint32_t u = gc / nsl;
                        if (u > 0) tc::mbar_wait_backoff(&empty_bar[s], (u - 1) & 1);
                        tc::mbar_arrive_expect_tx(&full_bar[s], (uint32_t)kAStage);
                        tc::tma_load_2d(smem + sp.off_raw + s * kAStage, &tmapA, &full_bar[s], c * kKC, row0);
                    }
                }
            }
        }
    } else {
        // ================= epilogue =================
        const int e = warp - kEpiWarp0;     // 0..7
        const int quarter = warp & 3;       // TMEM lanes this warp may access: 32 * (warp % 4) ..
        const int part = e >> 2;            // interleaved kEC-column chunks: part, part + kEpiWarps / 4, ...
        const int r = quarter * 32 + lane;  // tile row = vector
        const int et = e * 32 + lane;       // index among the epilogue threads (>= NG)
        uint32_t ic = 0, tcnt = 0;
        int64_t item = blockIdx.x;
        Item it{};
        ColC nextc;
        auto fetch_colc = [&](const Item& x) {  // one coalesced 32-byte load per column (NG <= 32 kEpiWarps)
            if (et < x.ncols) {
                nextc = a.gcolc[x.grow0 + et];
            } else {
                nextc.a = nextc.b = nextc.K = nextc.nq2 = 0.f;
                nextc.tau = -INFINITY;
                nextc.U = -INFINITY;
                nextc.q = -1;
                nextc.pair = -1;
            }
        };
        if (item < total) {
            it = decode_item(a, NG, item);
            fetch_colc(it);
            if (et < NG) colp_put(colc, et, nextc);
        }
        tc::named_barrier(1, kEpiWarps * 32);
        for (; item < total; item += gridDim.x, ++ic) {
            const ColPair* cb = colc + (ic & 1) * (NG / 2);
            // prefetch the next item's column constants (latency hidden by this item)
            const int64_t nitem = item + gridDim.x;
            Item nit{};
            if (nitem < total) {
                nit = decode_item(a, NG, nitem);
                fetch_colc(nit);
            }
            for (int t = 0; t < it.ntiles; ++t, ++tcnt) {
                const int b = tcnt & 1;
                const uint32_t ub = tcnt >> 1;
                const int64_t v = (it.t0 + t) * kTM + r;
                const bool vok = v < it.L;
                const int64_t slot = it.slot_base + v;
                const float2 fac = vok ? a.fac[slot] : make_float2(0.f, 0.f);
                const float pcf = vok ? (float)a.pcnt[slot] : 0.f;
                const float g1 = (kLB && vok) ? a.g1[slot] : 0.f;
                const uint32_t row = vok ? a.rows[slot] : 0u;
                if (e == 0 && lane == 0) RQ_TR(13, tcnt);
                tc::mbar_wait(&accf_bar[b], ub & 1);
                if (e == 0 && lane == 0) RQ_TR(14, tcnt);
                tc::fence_after_sync();
                // pass A (each of this warp's column chunks): fast test, ballots and the
                // chunk's counter atomics; pass B: the survivors' stores, after every
                // atomic of the tile is in flight (their latency overlaps the tests)
                constexpr int kMaxHC = (kTN / kEC + kEpiWarps / 4 - 1) / (kEpiWarps / 4);
                uint32_t hc_cols[kMaxHC], hc_bal[kMaxHC];
                int hc_base[kMaxHC];
                const int ncols_e = (a.experiment & 1) ? 0 : it.ncols;
#pragma unroll
                for (int k = 0; k < kMaxHC; ++k) hc_cols[k] = 0u;
#pragma unroll
                for (int k = 0; k < kMaxHC; ++k) {
                    const int hc = part + k * (kEpiWarps / 4);
                    if (hc * kEC >= ncols_e) break;
                    const int col0 = hc * kEC;
                    const uint32_t tcol = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)b * sp.acc_cols + col0;
                    uint32_t acc[kEC];
                    tc::tmem_ld16(tcol, acc);
                    // kFull: a pair is 4 consecutive digit columns, logical column = its first
                    constexpr int kStep = kFull ? 4 : 1;
                    auto est_at = [&](int i, const ColC& cc) -> float {
                        if constexpr (kFull) return est_ipn(ipn_full(acc[i], acc[i + 1], acc[i + 2], acc[i + 3]), cc, fac, pcf);
                        else return est_of(acc[i], cc, fac, pcf);
                    };
                    if constexpr (kDense) {
                        // sample scan: every key, coalesced (lanes = consecutive vectors);
                        // the column's absolute offset rides in (q, pair)
#pragma unroll
                        for (int i = 0; i < kEC; i += kStep) {
                            const ColC cc = colp_get(cb, col0 + i);
                            const float key = rank_key<kLB>(est_at(i, cc), epsnq_of(cc), g1);
                            const int64_t off = ((int64_t)(uint32_t)cc.pair << 32) | (uint32_t)cc.q;
                            if (vok && col0 + i < it.ncols) a.dense_keys[off + v] = f2o(key);
                        }
                        continue;
                    }
                    // phase 1: bit i of rowbits = this row may survive against column i.
                    // Main scan: fast test fma(-f, t, A) <= U (U = tau - ||r_q||^2 + a
                    // rounding margin), a superset of est <= tau; phase 3 stores the
                    // exact keys.  Re-scan / lower-bound key / dump: the exact key.
                    uint32_t rowbits = 0u;
                    if constexpr (!kLB && !kRetry && !kDump && !kFull) {
                        // packed: columns i, i + 1 per FADD2 / FFMA2, each lane rounded as
                        // fma(-a, ipn, fma(b, pcf, -K)), fma(-f, t, A) (empty columns: U = -inf)
                        const float2 pc2 = make_float2(pcf, pcf), nf2 = make_float2(-fac.y, -fac.y);
                        const float2 fx2 = make_float2(fac.x, fac.x), mg2 = make_float2(12582912.0f, 12582912.0f);
                        const float4* P0 = reinterpret_cast<const float4*>(cb + (col0 >> 1));  // col0 even
#pragma unroll
                        for (int i = 0; i < kEC; i += 2) {
                            const float4* P = P0 + 2 * i;  // record (col0 + i) / 2 = 4 float4
                            const float4 ab = P[0], ku = P[1];  // (-a0, -a1, b0, b1), (-K0, -K1, U0, U1)
                            const float2 ipn = fsub2(make_float2(__int_as_float(0x4B400000 + (int)acc[i]),
                                                                 __int_as_float(0x4B400000 + (int)acc[i + 1])), mg2);
                            const float2 inner = ffma2(make_float2(ab.z, ab.w), pc2, make_float2(ku.x, ku.y));
                            const float2 tt = ffma2(make_float2(ab.x, ab.y), ipn, inner);
                            const float2 v = ffma2(nf2, tt, fx2);
                            rowbits |= (v.x <= ku.z ? 1u : 0u) << i;
                            rowbits |= (v.y <= ku.w ? 1u : 0u) << (i + 1);
                        }
                    } else {
#pragma unroll
                    for (int i = 0; i < kEC; i += kStep) {
                        const ColC cc = colp_get(cb, col0 + i);
                        bool sv;
                        {
                            const float est = est_at(i, cc);
                            const float key = rank_key<kLB>(est, epsnq_of(cc), g1);
                            if constexpr (kDump) {
                                if (vok && col0 + i < it.ncols) {
                                    const int64_t di = (a.item_off[cc.pair] + (v >> 5)) * 32 + (v & 31);
                                    if (di < a.dump_cap) {
                                        a.dump_ip[di] = kFull ? 0 : -(int)acc[i];  // (full: ip exceeds int32)
                                        a.dump_est[di] = est;
                                    }
                                }
                            }
                            if constexpr (kRetry) {  // exact (key, row) <= tau64 (overflow / underflow re-scan)
                                const uint32_t ko = f2o(key), to = f2o(cc.tau);
                                sv = ko < to || (ko == to && row <= (uint32_t)cc.pair);
                            } else {
                                sv = key <= cc.tau;
                            }
                        }
                        rowbits |= sv ? (1u << i) : 0u;
                    }
                    }
                    if (!vok) rowbits = 0u;
                    const uint32_t cols = __reduce_or_sync(0xFFFFFFFFu, rowbits);
                    hc_cols[k] = cols;
                    hc_bal[k] = 0u;
                    hc_base[k] = 0;
                    if (cols) {
                        // phase 2 (surviving columns only): lane i takes column i's ballot,
                        // then one atomic per column, all issued together
                        uint32_t mybal = 0u;
                        for (uint32_t m = cols; m; m &= m - 1) {
                            const int i = __ffs(m) - 1;
                            const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (rowbits >> i) & 1u);
                            if (lane == i) mybal = bal;
                        }
                        hc_bal[k] = mybal;
                        if (mybal) hc_base[k] = atomicAdd(&a.cnt[colp_get(cb, col0 + (lane & (kEC - 1))).q], __popc(mybal));
                    }
                }
                if constexpr (!kDense) {
#pragma unroll
                    for (int k = 0; k < kMaxHC; ++k) {
                        const uint32_t cols = hc_cols[k];
                        if (!cols) continue;
                        // phase 3: survivors re-read their accumulator column and store
                        // (key, row); same arithmetic as phase 1, same key
                        const int col0 = (part + k * (kEpiWarps / 4)) * kEC;
                        const uint32_t tcol = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)b * sp.acc_cols + col0;
                        for (uint32_t m = cols; m; m &= m - 1) {
                            const int i = __ffs(m) - 1;
                            const uint32_t bal = __shfl_sync(0xFFFFFFFFu, hc_bal[k], i);
                            const int base = __shfl_sync(0xFFFFFFFFu, hc_base[k], i);
                            const uint32_t acci = tc::tmem_ld1(tcol + (uint32_t)i);
                            uint32_t acc1 = 0u, acc2 = 0u, acc3 = 0u;
                            if constexpr (kFull) {
                                acc1 = tc::tmem_ld1(tcol + (uint32_t)i + 1u);
                                acc2 = tc::tmem_ld1(tcol + (uint32_t)i + 2u);
                                acc3 = tc::tmem_ld1(tcol + (uint32_t)i + 3u);
                            }
                            if ((bal >> lane) & 1u) {
                                const ColC cc = colp_get(cb, col0 + i);
                                const float est = kFull ? est_ipn(ipn_full(acci, acc1, acc2, acc3), cc, fac, pcf)
                                                        : est_of(acci, cc, fac, pcf);
                                const float key = rank_key<kLB>(est, epsnq_of(cc), g1);
                                const int pos = base + __popc(bal & ((1u << lane) - 1u));
                                if (pos < a.cap) a.buf[(size_t)cc.q * a.cap + pos] = make_key(key, row);
                            }
                        }
                    }
                }
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&acce_bar[b]);  // accumulator b may be overwritten
                if (e == 0 && lane == 0) RQ_TR(15, tcnt);
            }
            // publish the next item's column constants into the other buffer (its
            // last readers finished item ic - 1 before the previous barrier)
            if (nitem < total && et < NG) colp_put(colc + ((ic + 1) & 1) * (NG / 2), et, nextc);
            tc::named_barrier(1, kEpiWarps * 32);
            it = nit;
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == kMmaWarp) tc::tmem_dealloc(tmem, kTmemCols);
}

// ------------------------------------------------- operand-swapped main scan
// The main scan (rank key EST, no dump / re-scan / dense mode, 4-bit query)
// with the roles of the operands swapped: the group's <= 128 quantized queries
// are the A operand, resident in TMEM for a whole item (K = Dp bytes = Dp / 4
// columns), and each 128-vector code tile is the B operand, streamed from the
// expanded codes by TMA through kSwB shared-memory stages.  D[query][vector]
// sits in TMEM with one query per lane, so the epilogue keeps the query's
// column constants in registers and reserves a lane's survivors of a 16-vector
// chunk with one counter atomic.  Same arithmetic per (query, vector) as
// scan_imma_kernel: identical keys and survivors.
constexpr int kSwNG = 128;        // queries per group (UMMA M)
constexpr int kSwB = 12;          // code stages (16 KB each)
constexpr int kSwEpi0 = 6;        // warps 0 loader, 1 MMA, 2-5 query writers, 6-21 epilogue
constexpr int kSwNT = (kSwEpi0 + kEpiWarps) * 32;
constexpr int kSwAcc = 128;       // accumulator columns per buffer (128 vectors)
__global__ __launch_bounds__(kSwNT, 1) void scan_swap_kernel(const __grid_constant__ CUtensorMap tmapC, ScanArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* stages = smem_raw + pad;  // [kSwB][128 vectors][128 bytes], 128-byte swizzle
    __shared__ __align__(8) uint64_t full_bar[kSwB], empty_bar[kSwB], accf_bar[2], acce_bar[2],
        afull_bar[kMaxChunks], afree_bar[kMaxChunks], vfull_bar[2];
    __shared__ __align__(16) float4 vconst[2][kTM / 2];  // per tile buffer: (f0, A0, f1, A1) per vector pair
    __shared__ __align__(16) float2 vpc[2][kTM / 2];     // (pcf0, pcf1)
    __shared__ uint32_t vrow[2][kTM];
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nchunks = (a.Dp + kKC - 1) / kKC;
    if (warp == 1) tc::tmem_alloc(&tmem_base_s, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s < kSwB; ++s) {
            tc::mbar_init(&full_bar[s], 1);
            tc::mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&accf_bar[b], 1);
            tc::mbar_init(&acce_bar[b], kEpiWarps);
        }
        for (int c = 0; c < kMaxChunks; ++c) {
            tc::mbar_init(&afull_bar[c], 4);  // one arrive per query-writer warp
            tc::mbar_init(&afree_bar[c], 1);
        }
        tc::prefetch_tmap(&tmapC);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base_s;
    const uint32_t tmemA = tmem + 2u * kSwAcc;  // the queries: Dp / 4 columns
    const int64_t total = a.list_items[a.nlist];

    if (warp == 0) {
        // ================= code tiles (B) by TMA =================
        if (lane == 0) {
            uint32_t gc = 0;
            for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
                const Item it = decode_item(a, kSwNG, item);
                for (int t = 0; t < it.ntiles; ++t) {
                    const int row0 = (int)(it.slot_base + (it.t0 + t) * kTM);
                    for (int c = 0; c < nchunks; ++c, ++gc) {
                        const int s = (int)(gc % kSwB);
                        const uint32_t u = gc / kSwB;
                        if (u > 0) tc::mbar_wait_backoff(&empty_bar[s], (u - 1) & 1);
                        tc::mbar_arrive_expect_tx(&full_bar[s], (uint32_t)kAStage);
                        tc::tma_load_2d(stages + s * kAStage, &tmapC, &full_bar[s], c * kKC, row0);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer =================
        uint32_t gc = 0, tcnt = 0, ic = 0;
        const uint32_t idesc = tc::idesc_i8(kSwNG, kTM, /*a_signed=*/false, /*b_signed=*/true);
        for (int64_t item = blockIdx.x; item < total; item += gridDim.x, ++ic) {
            const Item it = decode_item(a, kSwNG, item);
            for (int t = 0; t < it.ntiles; ++t, ++tcnt) {
                const int b = tcnt & 1;
                const uint32_t ub = tcnt >> 1;
                if (ub > 0) tc::mbar_wait_backoff(&acce_bar[b], (ub - 1) & 1);
                tc::fence_after_sync();
                const uint32_t dacc = tmem + (uint32_t)b * kSwAcc;
                for (int c = 0; c < nchunks; ++c, ++gc) {
                    const int s = (int)(gc % kSwB);
                    const int nks = min(kKC, a.Dp - c * kKC) / 32;
                    if (t == 0) tc::mbar_wait(&afull_bar[c], ic & 1);  // the item's query chunk c is in TMEM
                    tc::mbar_wait(&full_bar[s], (gc / kSwB) & 1);
                    tc::fence_after_sync();
                    const uint64_t bd = tc::smem_desc_sw128(tc::smem_u32(stages + s * kAStage));
                    tc::mma_i8_ts_chunk(dacc, tmemA + (uint32_t)(c * kChunkCols), bd, idesc, c > 0 ? 1u : 0u, nks,
                                        &empty_bar[s]);
                    if (t == it.ntiles - 1) tc::commit_warp(&afree_bar[c]);  // query chunk c free for the next item
                    if (c == nchunks - 1) tc::commit_warp(&accf_bar[b]);
                }
            }
        }
    } else if (warp < kSwEpi0) {
        // ================= queries (A) into TMEM =================
        const int qq = warp & 3;              // TMEM lane quarter of this warp
        const int r = qq * 32 + lane;         // query row of the group = TMEM lane
        const uint32_t lane_addr = (uint32_t)(qq * 32) << 16;
        uint32_t ic = 0;
        for (int64_t item = blockIdx.x; item < total; item += gridDim.x, ++ic) {
            const Item it = decode_item(a, kSwNG, item);
            const uint4* src = reinterpret_cast<const uint4*>(a.qbar8 + (size_t)(it.grow0 + r) * a.Dp);
            const bool ok = r < it.ncols;
            for (int c = 0; c < nchunks; ++c) {
                // chunk c (128 K bytes = 32 columns) once the previous item's last tile used it
                uint4 v[8];
                const int nq4 = min(kKC, a.Dp - c * kKC) / 16;  // 16-byte words in this chunk (4 or 8)
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    v[k] = (ok && k < nq4) ? __ldg(src + c * 8 + k) : make_uint4(0u, 0u, 0u, 0u);
                if (ic > 0) tc::mbar_wait_backoff(&afree_bar[c], (ic - 1) & 1);
                tc::fence_after_sync();
                const uint32_t dst = tmemA + lane_addr + (uint32_t)(c * kChunkCols);
                tc::tmem_st16(dst, v[0], v[1], v[2], v[3]);
                if (nq4 > 4) tc::tmem_st16(dst + 16, v[4], v[5], v[6], v[7]);
                tc::tmem_st_wait();
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&afull_bar[c]);
            }
        }
    } else {
        // ================= epilogue: lane = query, columns = vectors =================
        const int e = warp - kSwEpi0;
        const int quarter = warp & 3;
        const int part = e >> 2;              // column chunks part, part + 4 (16 vectors each)
        const int r = quarter * 32 + lane;    // query row of the group
        uint32_t tcnt = 0;
        for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
            const Item it = decode_item(a, kSwNG, item);
            const bool qok = r < it.ncols;
            ColC cc;
            if (qok) {
                cc = a.gcolc[it.grow0 + r];
            } else {
                cc.a = cc.b = cc.K = cc.nq2 = 0.f;
                cc.tau = cc.U = -INFINITY;
                cc.q = 0;
                cc.pair = -1;
            }
            const float2 nb_pc = make_float2(cc.b, cc.b), nK2 = make_float2(-cc.K, -cc.K);
            const float2 na2 = make_float2(-cc.a, -cc.a), mg2 = make_float2(12582912.0f, 12582912.0f);
            for (int t = 0; t < it.ntiles; ++t, ++tcnt) {
                const int b = tcnt & 1;
                const uint32_t ub = tcnt >> 1;
                const int64_t vbase = (it.t0 + t) * kTM;
                {
                    // the tile's vector constants in shared memory (double-buffered by tile
                    // parity; the barrier below also ends every warp's use of this buffer
                    // two tiles ago): (-f0, -f1, A0, A1), (pcf0, pcf1), rows
                    const int et = e * 32 + lane;
                    if (et < kTM / 2) {
                        const int64_t v0 = vbase + 2 * et;
                        const bool ok0 = v0 < it.L, ok1 = v0 + 1 < it.L;
                        const float2 f0 = ok0 ? __ldg(a.fac + it.slot_base + v0) : make_float2(0.f, 0.f);
                        const float2 f1 = ok1 ? __ldg(a.fac + it.slot_base + v0 + 1) : make_float2(0.f, 0.f);
                        vconst[b][et] = make_float4(-f0.y, -f1.y, f0.x, f1.x);
                        vpc[b][et] = make_float2(ok0 ? (float)__ldg(a.pcnt + it.slot_base + v0) : 0.f,
                                                 ok1 ? (float)__ldg(a.pcnt + it.slot_base + v0 + 1) : 0.f);
                    } else if (et < kTM / 2 + kTM) {
                        const int64_t v = vbase + (et - kTM / 2);
                        vrow[b][et - kTM / 2] = v < it.L ? __ldg(a.rows + it.slot_base + v) : 0u;
                    }
                    tc::named_barrier(1, kEpiWarps * 32);
                }
                tc::mbar_wait(&accf_bar[b], ub & 1);
                tc::fence_after_sync();
                uint32_t hc_bits[2];
                int hc_base[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int col0 = (part + 4 * k) * 16;
                    const uint32_t tcol = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)b * kSwAcc + col0;
                    uint32_t acc[16];
                    tc::tmem_ld16(tcol, acc);
                    uint32_t bits = 0u;
                    const int64_t nval = it.L - (vbase + col0);  // valid vectors from col0 on
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        const float4 vc = vconst[b][(col0 + i) >> 1];
                        const float2 pc = vpc[b][(col0 + i) >> 1];
                        const float2 ipn = fsub2(make_float2(__int_as_float(0x4B400000 + (int)acc[i]),
                                                             __int_as_float(0x4B400000 + (int)acc[i + 1])), mg2);
                        const float2 inner = ffma2(nb_pc, pc, nK2);
                        const float2 tt = ffma2(na2, ipn, inner);
                        const float2 vv = ffma2(make_float2(vc.x, vc.y), tt, make_float2(vc.z, vc.w));
                        bits |= (vv.x <= cc.U ? 1u : 0u) << i;
                        bits |= (vv.y <= cc.U ? 1u : 0u) << (i + 1);
                    }
                    if (nval < 16) bits &= nval > 0 ? (1u << nval) - 1u : 0u;
                    if (!qok) bits = 0u;
                    hc_bits[k] = bits;
                    hc_base[k] = bits ? atomicAdd(&a.cnt[cc.q], __popc(bits)) : 0;
                }
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const uint32_t bits = hc_bits[k];
                    uint32_t cols = __reduce_or_sync(0xFFFFFFFFu, bits);
                    const int col0 = (part + 4 * k) * 16;
                    const uint32_t tcol = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)b * kSwAcc + col0;
                    for (; cols; cols &= cols - 1) {
                        const int i = __ffs(cols) - 1;
                        const uint32_t acci = tc::tmem_ld1(tcol + (uint32_t)i);
                        if ((bits >> i) & 1u) {
                            const int c = col0 + i;
                            const float4 vc = vconst[b][c >> 1];
                            const float2 pc = vpc[b][c >> 1];
                            const float2 fac = (c & 1) ? make_float2(vc.w, -vc.y) : make_float2(vc.z, -vc.x);
                            const float key = est_of(acci, cc, fac, (c & 1) ? pc.y : pc.x);
                            const int pos = hc_base[k] + __popc(bits & ((1u << i) - 1u));
                            if (pos < a.cap) a.buf[(size_t)cc.q * a.cap + pos] = make_key(key, vrow[b][c]);
                        }
                    }
                }
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&acce_bar[b]);
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, kTmemCols);
}

// ------------------------------------------------------------ list grouping
// pairs to group: all (sub == nullptr) or the listed pair indices
// rows = grouped B rows per pair (1; 4 for the unquantized query's digit rows)
__global__ void group_count_kernel(const int32_t* __restrict__ probes, const int32_t* __restrict__ sub, int64_t n,
                                   int64_t* __restrict__ gcount, int rows) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)&gcount[probes[sub ? sub[i] : i]], (unsigned long long)rows);
}

__global__ void group_fill_kernel(const int32_t* __restrict__ probes, const int32_t* __restrict__ sub, int64_t n,
                                  const int64_t* __restrict__ gstart, int32_t* __restrict__ gfill,
                                  int32_t* __restrict__ gpos, int32_t* __restrict__ gpair, int rows) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int p = sub ? sub[i] : (int)i;
        const int j = probes[p];
        const int64_t pos = gstart[j] + atomicAdd(&gfill[j], rows);
        gpos[i] = (int32_t)pos;  // first of the pair's rows
        for (int r = 0; r < rows; ++r) gpair[pos + r] = (int32_t)p;
    }
}

// copy the int8 query rows of the listed pairs from the full grouping into a sub grouping
// (`rows` consecutive rows of Dp bytes per pair)
__global__ void gather_rows_kernel(const int32_t* __restrict__ sub, int64_t n, const int32_t* __restrict__ gpos_full,
                                   const uint8_t* __restrict__ q8_full, const int32_t* __restrict__ gpos_sub,
                                   uint8_t* __restrict__ q8_sub, int Dp, int rows) {
    const int per = rows * Dp / 16;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * per; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / per;
        const int k = (int)(e % per);
        const uint4 v = reinterpret_cast<const uint4*>(q8_full + (size_t)gpos_full[sub[i]] * Dp)[k];
        reinterpret_cast<uint4*>(q8_sub + (size_t)gpos_sub[i] * Dp)[k] = v;
    }
}

// pairs of the flagged (overflowed) queries, or (flags == nullptr) the pairs of
// probe rank < max_rank (each query's nearest lists)
__global__ void compact_flagged_kernel(const int* __restrict__ flags, int max_rank, int64_t npairs, int nprobe,
                                       int32_t* __restrict__ sub, int* __restrict__ n) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs; p += (int64_t)gridDim.x * blockDim.x) {
        const bool take = flags ? flags[p / nprobe] != 0 : (p % nprobe) < max_rank;
        if (take) sub[atomicAdd(n, 1)] = (int32_t)p;
    }
}

// column constants of every grouped row (one 32-byte record per (query, list) pair)
// (re-scan: tau / pair carry the 64-bit (key, row) threshold instead)
__global__ void colc_kernel(const int32_t* __restrict__ gpair, int64_t npairs, int nprobe, int D,
                            const float4* __restrict__ qscal, const float* __restrict__ tau,
                            const uint64_t* __restrict__ tau64, float eps0, const int64_t* __restrict__ dbase,
                            const int64_t* __restrict__ doff, const int32_t* __restrict__ probes,
                            const float* __restrict__ list_amax, ColC* __restrict__ gcolc) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < npairs; g += (int64_t)gridDim.x * blockDim.x) {
        const int p = gpair[g];
        const int q = p / nprobe;
        const PairC pc = pair_consts(qscal[p], D);
        ColC cc;
        cc.a = pc.a;
        cc.b = pc.b;
        cc.K = pc.K;
        cc.nq2 = pc.nq2;
        cc.q = q;
        if (dbase) {  // dense key dump: absolute offset of the pair's keys in (q, pair)
            const int64_t off = dbase[q] + doff[p];
            cc.tau = INFINITY;
            cc.q = (int)(uint32_t)off;
            cc.pair = (int)(uint32_t)(off >> 32);
        } else if (tau64) {
            cc.tau = o2f((uint32_t)(tau64[q] >> 32));
            cc.pair = (int)(uint32_t)tau64[q];
        } else {
            cc.tau = tau[q];
            cc.pair = p;
        }
        // fast test bound: for est = RN(RN(A + nq2) - f t) <= tau, the fused
        // RN(A - f t) exceeds tau - nq2 by at most a few ulps of A + nq2 + |tau|
        if (cc.tau == INFINITY || cc.tau == -INFINITY) {
            cc.U = cc.tau;
        } else {
            const float amax = list_amax[probes[p]];
            const float mag = __fadd_rn(__fadd_rn(amax, pc.nq2), fabsf(cc.tau));
            cc.U = __fadd_rn(__fsub_rn(cc.tau, pc.nq2), __fmul_rn(4.76837158e-7f, mag));  // 2^-21
        }
        gcolc[g] = cc;
    }
}

__global__ void list_items_kernel(int nlist, const int64_t* __restrict__ list_off, const int64_t* __restrict__ gcount,
                                  int NG, int64_t* __restrict__ items) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= nlist; j += gridDim.x * blockDim.x) {
        if (j == nlist) {
            items[j] = 0;
            continue;
        }
        const int64_t L = list_off[j + 1] - list_off[j];
        const int64_t G = gcount[j];
        const int64_t ntl = (L + kTM - 1) / kTM;
        items[j] = ((ntl + kTilesPerItem - 1) / kTilesPerItem) * ((G + NG - 1) / NG);
    }
}

// codes -> s8 {0, -1} rows in the K order of expand32 (the TMEM A operand the
// producers would build), slot-major, 128 zero pad rows
__global__ void expand_codes_kernel(const uint32_t* __restrict__ codes, int64_t nslots, int W,
                                    uint4* __restrict__ out) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (nslots + kTM) * W;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / W;
        const int w = (int)(e % W);
        uint4 lo = make_uint4(0u, 0u, 0u, 0u), hi = lo;
        if (s < nslots) expand32(__ldg(codes + ((s >> 5) * W + w) * 32 + (s & 31)), lo, hi);
        out[2 * e] = lo;
        out[2 * e + 1] = hi;
    }
}

__global__ void list_items_gstart_kernel(int nlist, const int64_t* __restrict__ list_off,
                                         const int64_t* __restrict__ gstart, int NG, int64_t* __restrict__ items) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= nlist; j += gridDim.x * blockDim.x) {
        if (j == nlist) {
            items[j] = 0;
            continue;
        }
        const int64_t L = list_off[j + 1] - list_off[j];
        const int64_t G = gstart[j + 1] - gstart[j];
        const int64_t ntl = (L + kTM - 1) / kTM;
        items[j] = ((ntl + kTilesPerItem - 1) / kTilesPerItem) * ((G + NG - 1) / NG);
    }
}

}  // namespace

// largest group (B columns) of the TMA-A scan: fewer columns leave shared memory
// for more A stages in flight (diagnostics: RABITQ_TA_NGMAX, multiple of 32)
int ta_ngmax() {
    const char* env = getenv("RABITQ_TA_NGMAX");
    const int v = env ? atoi(env) : kTN;
    return std::max(kBoxRows, std::min(kTN, v / kBoxRows * kBoxRows));
}

// fewest A stages of the TMA-A scan (the group shrinks to make room; 16-column steps)
int ta_minstages() {
    const char* env = getenv("RABITQ_TA_MINSTAGES");
    const int v = env ? atoi(env) : kMinAStages;
    return std::max(2, std::min(kMaxSlots, v));
}

const uint8_t* codes8_of(const rabitq_index* idx) {
    const char* env = getenv("RABITQ_CODES8");  // "0": expand in the kernel (diagnostics / tests)
    return (env && env[0] == '0') ? nullptr : idx->codes8;
}

void expand_codes(rabitq_index* idx, cudaStream_t st) {
    const size_t bytes = (size_t)(idx->nslots + kTM) * 32 * idx->W;
    RQ_CUDA(cudaMalloc(&idx->codes8, bytes));
    expand_codes_kernel<<<4096, 256, 0, st>>>(idx->codes, idx->nslots, idx->W, reinterpret_cast<uint4*>(idx->codes8));
    RQ_CHECK_LAUNCH();
}

bool imma_wanted(const rabitq_index* idx, int64_t npairs, int scan_path) {
    if (scan_path == RABITQ_SCAN_POPC) return false;
    if (idx->W > 4 * kMaxChunks) return false;  // B chunks (D <= 1024)
    if (scan_path == RABITQ_SCAN_IMMA) return true;
    // AUTO: the tensor-core path pays once lists are shared by a few queries and
    // the batch amortizes its fixed cost, and at any batch for long codes
    // (measured, CFG2 D = 960: batch 64 0.75 vs 1.26 ms per search, 256: 1.12 vs
    // 3.48; CFG3 D = 96: batch 64 popc 0.66 vs 1.12 ms, 256 (4 pairs per list):
    // tensor cores 1.47 vs 1.95 ms; CFG1, 1600 pairs: popc 0.29 vs 0.42 ms)
    return npairs >= (int64_t)8 * idx->nlist || (npairs >= (int64_t)4 * idx->nlist && npairs >= 8192) ||
           idx->W >= 16;
}

void prepare_groups(const rabitq_index* idx, const int32_t* probes, int64_t n, const int32_t* sub, Groups& g,
                    cudaStream_t st, int& launches, int rows) {
    const int nlist = idx->nlist;
    g.Dp = ((idx->D + 31) / 32) * 32;
    g.n = n;
    g.rows = rows;
    g.gcount.alloc((size_t)nlist + 1, st);
    g.gstart.alloc((size_t)nlist + 1, st);
    g.itemc.alloc((size_t)nlist + 1, st);
    g.list_items.alloc((size_t)nlist + 1, st);
    g.gfill.alloc((size_t)nlist, st);
    g.gpos.alloc((size_t)n, st);
    g.gpair.alloc((size_t)n * rows + kTN, st);
    g.qbar8.alloc(((size_t)n * rows + kTN) * g.Dp, st);
    RQ_CUDA(cudaMemsetAsync(g.gcount.p, 0, ((size_t)nlist + 1) * sizeof(int64_t), st));
    RQ_CUDA(cudaMemsetAsync(g.gfill.p, 0, (size_t)nlist * sizeof(int32_t), st));
    RQ_CUDA(cudaMemsetAsync(g.gpair.p + n * rows, 0, kTN * sizeof(int32_t), st));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 2048));
    group_count_kernel<<<grid, 256, 0, st>>>(probes, sub, n, g.gcount.p, rows);
    RQ_CHECK_LAUNCH();
    size_t tb = 0;
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, g.gcount.p, g.gstart.p, nlist + 1, st));
    size_t tb2 = 0;
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, g.itemc.p, g.list_items.p, nlist + 1, st));
    WBuf<uint8_t> tmp;
    tmp.alloc(std::max(tb, tb2), st);
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, g.gcount.p, g.gstart.p, nlist + 1, st));
    group_fill_kernel<<<grid, 256, 0, st>>>(probes, sub, n, g.gstart.p, g.gfill.p, g.gpos.p, g.gpair.p, rows);
    RQ_CHECK_LAUNCH();
    list_items_kernel<<<(nlist + 256) / 256, 256, 0, st>>>(nlist, idx->list_off, g.gcount.p,
                                                           group_cols(g.Dp, codes8_of(idx) != nullptr, ta_ngmax(), ta_minstages()),
                                                           g.itemc.p);
    RQ_CHECK_LAUNCH();
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, g.itemc.p, g.list_items.p, nlist + 1, st));
    launches += 7;
}

void group_items(const rabitq_index* idx, const int64_t* list_off, const Groups& g, WBuf<int64_t>& itemc,
                 WBuf<int64_t>& items, cudaStream_t st, int& launches) {
    const int nlist = idx->nlist;
    itemc.alloc((size_t)nlist + 1, st);
    items.alloc((size_t)nlist + 1, st);
    list_items_kernel<<<(nlist + 256) / 256, 256, 0, st>>>(nlist, list_off, g.gcount.p,
                                                           group_cols(g.Dp, codes8_of(idx) != nullptr, ta_ngmax(), ta_minstages()), itemc.p);
    RQ_CHECK_LAUNCH();
    size_t tb = 0;
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, itemc.p, items.p, nlist + 1, st));
    WBuf<uint8_t> tmp;
    tmp.alloc(tb, st);
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, itemc.p, items.p, nlist + 1, st));
    launches += 3;
}

int64_t regroup_flagged(const rabitq_index* idx, const int32_t* probes, int64_t npairs, int nprobe, const int* flags,
                        int max_rank, const Groups& full, Groups& sub, cudaStream_t st, int& launches) {
    WBuf<int32_t> list;
    list.alloc((size_t)npairs, st);
    WBuf<int> cnt;
    cnt.alloc(1, st);
    RQ_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), st));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((npairs + 255) / 256, 2048));
    compact_flagged_kernel<<<grid, 256, 0, st>>>(flags, max_rank, npairs, nprobe, list.p, cnt.p);
    RQ_CHECK_LAUNCH();
    int n = 0;
    RQ_CUDA(cudaMemcpyAsync(&n, cnt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    RQ_CUDA(cudaStreamSynchronize(st));
    if (n == 0) return 0;
    prepare_groups(idx, probes, n, list.p, sub, st, launches, full.rows);
    const int per = full.rows * full.Dp / 16;
    gather_rows_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(((int64_t)n * per + 255) / 256, 4096)), 256,
                         0, st>>>(list.p, n, full.gpos.p, full.qbar8.p, sub.gpos.p, sub.qbar8.p, full.Dp, full.rows);
    RQ_CHECK_LAUNCH();
    launches += 2;
    return n;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        RQ_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        RQ_REQUIRE(p && q == cudaDriverEntryPointSuccess, RABITQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

void scan_imma(const ScanArgs& a_in, bool lb, bool dump, bool retry, cudaStream_t st, bool dense) {
    ScanArgs a = a_in;  // a.npairs = grouped rows (all pairs, or the re-scan's sub list)
    WBuf<ColC> gcolc;
    gcolc.alloc((size_t)a.npairs + kTN, st);
    colc_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((a.npairs + 255) / 256, 2048)), 256, 0, st>>>(
        a.gpair, a.npairs, a.nprobe, a.D, a.qscal, a.tau, retry ? a.tau64 : nullptr, a.eps0,
        dense ? a.dense_base : nullptr, dense ? a.dense_off : nullptr, a.probes, a.list_amax, gcolc.p);
    RQ_CHECK_LAUNCH();
    a.gcolc = gcolc.p;
    int dev = 0, sms = 148;
    RQ_CUDA(cudaGetDevice(&dev));
    RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // B = grouped int8 query rows [(npairs + kTN) x Dp]; TMA box 128 bytes x 32 rows, 128-byte swizzle
    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {(cuuint64_t)a.Dp, (cuuint64_t)(a.npairs + kTN)};
    const cuuint64_t gstride[1] = {(cuuint64_t)a.Dp};
    const cuuint32_t box[2] = {(cuuint32_t)kKC, (cuuint32_t)kBoxRows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = get_encode()(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.qbar8), gdim, gstride,
                               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RQ_REQUIRE(cr == CUDA_SUCCESS, RABITQ_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
    // A = expanded codes [(nslots + 128) x Dp] when the index has them: TMA box 128 bytes x 128 rows
    const bool ta = a.codes8 != nullptr;
    CUtensorMap tmapA;
    std::memset(&tmapA, 0, sizeof(tmapA));
    if (ta) {
        const cuuint64_t adim[2] = {(cuuint64_t)a.Dp, (cuuint64_t)(a.nslots + kTM)};
        const cuuint64_t astride[1] = {(cuuint64_t)a.Dp};
        const cuuint32_t abox[2] = {(cuuint32_t)kKC, (cuuint32_t)kTM};
        cr = get_encode()(&tmapA, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.codes8), adim, astride, abox,
                          estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        RQ_REQUIRE(cr == CUDA_SUCCESS, RABITQ_ERR_CUDA, "cuTensorMapEncodeTiled (A) failed: " + std::to_string((int)cr));
    }
    a.ngmax = ta_ngmax();
    a.minst = ta_minstages();
    // operand-swapped main scan (queries resident in TMEM, code tiles streamed
    // through 12 stages): opt-in (RABITQ_SWAP=1), bit-identical but slower as
    // built (CFG2 scan 4.47 vs 3.66 ms, CFG3 7.37 vs 4.86 ms): groups of 128
    // queries (TMEM holds the queries and both 128-column accumulators) mean
    // more tile passes than the 160 / 256-column groups of scan_imma_kernel
    const char* sw_env = getenv("RABITQ_SWAP");
    if (ta && !lb && !dump && !retry && !dense && !a.full && sw_env && sw_env[0] == '1' && a.experiment == 0 &&
        a.Dp <= 1024) {
        WBuf<int64_t> itemc, items;
        itemc.alloc((size_t)a.nlist + 1, st);
        items.alloc((size_t)a.nlist + 1, st);
        list_items_gstart_kernel<<<(a.nlist + 256) / 256, 256, 0, st>>>(a.nlist, a.list_off, a.gstart, kSwNG,
                                                                       itemc.p);
        RQ_CHECK_LAUNCH();
        size_t tb = 0;
        RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, itemc.p, items.p, a.nlist + 1, st));
        WBuf<uint8_t> tmp;
        tmp.alloc(tb, st);
        RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, itemc.p, items.p, a.nlist + 1, st));
        ScanArgs s = a;
        s.list_items = items.p;
        const size_t smem = (size_t)kSwB * kAStage + 1024;
        RQ_CUDA(cudaFuncSetAttribute(scan_swap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        scan_swap_kernel<<<sms, kSwNT, smem, st>>>(tmapA, s);
        RQ_CHECK_LAUNCH();
        return;
    }
    const SmemPlan plan = smem_plan(a.Dp, ta, a.ngmax, a.minst);
    RQ_REQUIRE(plan.slots >= 2 && plan.total <= (uint32_t)kSmemLimit, RABITQ_ERR_INTERNAL,
               "grouped scan: TMEM / shared-memory plan does not fit");
    const size_t smem = plan.total;
    const int grid = sms;
#define RQ_IMMA6(LB, DP, RT, DN, TA, FU)                                                                       \
    do {                                                                                                        \
        RQ_CUDA(cudaFuncSetAttribute(scan_imma_kernel<LB, DP, RT, DN, TA, FU>,                                  \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));                  \
        scan_imma_kernel<LB, DP, RT, DN, TA, FU><<<grid, n_threads(TA), smem, st>>>(tmap, tmapA, a);            \
    } while (0)
#define RQ_IMMA5(LB, DP, RT, DN, TA)                   \
    do {                                               \
        if (a.full) RQ_IMMA6(LB, DP, RT, DN, TA, true);  \
        else RQ_IMMA6(LB, DP, RT, DN, TA, false);        \
    } while (0)
#define RQ_IMMA4(LB, DP, RT, DN)                \
    do {                                        \
        if (ta) RQ_IMMA5(LB, DP, RT, DN, true); \
        else RQ_IMMA5(LB, DP, RT, DN, false);   \
    } while (0)
#define RQ_IMMA(LB, DP, RT) RQ_IMMA4(LB, DP, RT, false)
    if (dense) {
        if (lb) RQ_IMMA4(true, false, false, true);
        else RQ_IMMA4(false, false, false, true);
    } else if (dump) {
        if (lb) RQ_IMMA(true, true, false);
        else RQ_IMMA(false, true, false);
    } else if (retry) {
        if (lb) RQ_IMMA(true, false, true);
        else RQ_IMMA(false, false, true);
    } else {
        if (lb) RQ_IMMA(true, false, false);
        else RQ_IMMA(false, false, false);
    }
#undef RQ_IMMA
#undef RQ_IMMA4
#undef RQ_IMMA5
#undef RQ_IMMA6
    RQ_CHECK_LAUNCH();
}

}  // namespace rabitq
