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
#include <cuda_fp16.h>
#include <cuda_fp8.h>

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
    const int64_t G = __ldg(a.gcount + lo);
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

// the same bytes as e4m3: -1.0 (0xB8) / 0 (the .kind::f8f6f4 A operand, D <= 128)
__device__ __forceinline__ void to_e4m3(uint4& lo, uint4& hi) {
    lo.x &= 0xB8B8B8B8u; lo.y &= 0xB8B8B8B8u; lo.z &= 0xB8B8B8B8u; lo.w &= 0xB8B8B8B8u;
    hi.x &= 0xB8B8B8B8u; hi.y &= 0xB8B8B8B8u; hi.z &= 0xB8B8B8B8u; hi.w &= 0xB8B8B8B8u;
}

// fused estimator from the accumulator (acc = -ip: s8 codes in {0, -1}).
// 0x4B400000 + n is the float 1.5 2^23 + n exactly for |n| < 2^22, so ipn = -ip
// exactly; the rest is rabitq_est's arithmetic (a ip = (-a)(-ip) exactly).
// kF8 (e4m3 operands, f32 accumulator, D <= 128): the accumulator is -ip as an
// exact float already (integers of magnitude <= 15 D < 2^11)
template <bool kF8 = false>
__device__ __forceinline__ float acc_ipn(uint32_t acc) {
    if constexpr (kF8) return __uint_as_float(acc);
    else return __fsub_rn(__int_as_float(0x4B400000 + (int)acc), 12582912.0f);
}
template <bool kF8 = false>
__device__ __forceinline__ float est_of(uint32_t acc, const ColC& cc, float2 fac, float pcf) {
    const float ipn = acc_ipn<kF8>(acc);
    const float tt = __fmaf_rn(-cc.a, ipn, __fmaf_rn(cc.b, pcf, -cc.K));
    return __fmaf_rn(-fac.y, tt, __fadd_rn(fac.x, cc.nq2));
}

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
template <bool kLB, bool kDump, bool kRetry, bool kDense, bool kTA, bool kFull, bool kF8>
__global__ __launch_bounds__(n_threads(kTA), 1) void scan_imma_kernel(const __grid_constant__ CUtensorMap tmapB,
                                                                      const __grid_constant__ CUtensorMap tmapA,
                                                                      ScanArgs a) {
    constexpr int kMmaWarp = mma_warp(kTA), kLoadWarp = load_warp(kTA), kLoadAWarp = loada_warp(kTA),
                  kEpiWarp0 = epi_warp0(kTA);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    const SmemPlan sp = smem_plan(a.Dp, kTA);
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
            if (kF8) to_e4m3(lo, hi);
            tc::tmem_st8(dst, lo, hi);
            expand32(wv.y, lo, hi);
            if (kF8) to_e4m3(lo, hi);
            tc::tmem_st8(dst + 8, lo, hi);
            expand32(wv.z, lo, hi);
            if (kF8) to_e4m3(lo, hi);
            tc::tmem_st8(dst + 16, lo, hi);
            expand32(wv.w, lo, hi);
            if (kF8) to_e4m3(lo, hi);
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
            const uint32_t idesc = tc::idesc_scan<kF8>(kTM, it.ncols16);
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
                            tc::mma_i8_ss_chunk<kF8>(dacc, ad, bd, idesc, c > 0 ? 1u : 0u, nks, &empty_bar[s]);
                        } else {
                            // nks UMMAs + commit: A slot s free once these retire
                            const uint32_t aaddr = tmemA + (uint32_t)(s * kChunkCols);
                            tc::mma_i8_ts_chunk<kF8>(dacc, aaddr, bd, idesc, c > 0 ? 1u : 0u, nks, &empty_bar[s]);
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
                nextc = colp_get(a.gcolp, (int)(x.grow0 + et));
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
                const int ncols_e = it.ncols;
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
                        else return est_of<kF8>(acc[i], cc, fac, pcf);
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
                            const float2 ipn = kF8 ? make_float2(__uint_as_float(acc[i]), __uint_as_float(acc[i + 1]))
                                                   : fsub2(make_float2(__int_as_float(0x4B400000 + (int)acc[i]),
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
                                        a.dump_ip[di] = kFull ? 0 : (int)-acc_ipn<kF8>(acc[i]);  // (full: ip exceeds int32)
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
                                                        : est_of<kF8>(acci, cc, fac, pcf);
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

// ------------------------------------------------- folded survivor test
// (scan_fold_kernel, D <= 128).  For f = fac.y > 0 and a = 2 Delta > 0 the fast
// test A - f (a ip + b pc - K) <= U  (A = n_o^2, U = tau - ||r_q||^2) is
//     T = ip + pc y1 + y2 + alpha y3 + beta y4 >= 0,
//     y1 = b / a, y2 = -K / a, y3 = -1 / a, y4 = U / a (column),
//     alpha = A / f, beta = 1 / f, pc (row),
// a sum of rank-1 products: the tensor cores compute E = T - ip as a K = 16
// tf32 contraction (each factor split hi + lo, the three significant
// products kept: relative error ~2^-21 per term) into a second accumulator,
// and the epilogue tests E - acc >= 0 (acc = -ip, exact).  The margins make
// the test conservative: every pair whose est (scan arithmetic, fp32) is <= tau
// has T >= c S > 0 in exact arithmetic (S = sum of the terms' magnitudes,
// c = 2^-16 >> the fp32 / tf32 / accumulation errors), so it is flagged;
// flagged pairs then get their exact key as before.  Rows with f <= 0 (n_o = 0)
// and columns without a finite positive a or a finite tau always pass (or, tau
// = -inf, never): their keys are computed exactly.
constexpr float kFoldC = 1.52587890625e-05f;  // 2^-16
constexpr float kFoldBig = 1.8446744073709552e19f;  // 2^64
// X / BX layout: 16 tf32 per row, canonical K-major without swizzle: row r,
// 4-float chunk c at (r / 8) 512 + c 128 + (r % 8) 16 bytes
__device__ __forceinline__ void fold_col_put(float* gext, int64_t g, float y1, float y2, float y3, float y4,
                                             float pad) {
    const float y1h = tc::tf32_rna(y1), y2h = tc::tf32_rna(y2), y3h = tc::tf32_rna(y3), y4h = tc::tf32_rna(y4);
    const float y1l = tc::tf32_rna(__fsub_rn(y1, y1h)), y2l = tc::tf32_rna(__fsub_rn(y2, y2h));
    const float y3l = tc::tf32_rna(__fsub_rn(y3, y3h)), y4l = tc::tf32_rna(__fsub_rn(y4, y4h));
    (void)pad;
    float4* o = reinterpret_cast<float4*>(gext + (g >> 3) * 128 + (g & 7) * 4);
    o[0] = make_float4(y1h, y1l, y2h, y2l);    // x pc, pc, 1, 1  (all negated by the caller: D = -ip - E)
    o[8] = make_float4(y3h, y3l, y3h, y4h);    // x alpha_h, alpha_h, alpha_l, beta_h
    o[16] = make_float4(y4l, y4h, 0.f, 0.f);   // x beta_h, beta_l
    o[24] = make_float4(0.f, 0.f, 0.f, 0.f);
}
// fold_col_put(-kFoldBig, ...) puts -2^64 into y1 x pc; a pad / force column
// uses y2 instead (multiplied by 1 in every row):
__device__ __forceinline__ void fold_col_const(float* gext, int64_t g, float e) {
    float4* o = reinterpret_cast<float4*>(gext + (g >> 3) * 128 + (g & 7) * 4);
    o[0] = make_float4(0.f, 0.f, e, 0.f);
    o[8] = make_float4(0.f, 0.f, 0.f, 0.f);
    o[16] = make_float4(0.f, 0.f, 0.f, 0.f);
    o[24] = make_float4(0.f, 0.f, 0.f, 0.f);
}
__device__ __forceinline__ void fold_col(float* gext, int64_t g, const ColC& cc, int Dp) {
    const float a = cc.a, tau = cc.tau;
    const bool fin = isfinite(a) && isfinite(cc.b) && isfinite(cc.K) && isfinite(cc.nq2);
    if (tau == -INFINITY) {
        fold_col_const(gext, g, kFoldBig);  // nothing is <= -inf (D = -ip - E > 0)
        return;
    }
    if (!(a > 0.f) || !fin || !isfinite(tau)) {
        fold_col_const(gext, g, -kFoldBig);  // every pair is flagged (exact keys decide)
        return;
    }
    const float ia = __frcp_rn(a);
    const float y1 = __fmul_rn(cc.b, ia), kp = __fmul_rn(cc.K, ia);
    const float m = __fmul_rn(kFoldC, __fadd_rn(__fmul_rn(15.f, (float)Dp),
                                                __fadd_rn(__fmul_rn(2.f * (float)Dp, fabsf(y1)), __fmul_rn(2.f, fabsf(kp)))));
    const float y2 = __fadd_rn(-kp, m);
    const float y3 = -__fmul_rn(1.f - kFoldC, ia);
    const float u = __fadd_rn(__fsub_rn(tau, cc.nq2), __fmul_rn(kFoldC, __fadd_rn(cc.nq2, fabsf(tau))));
    const float y4 = __fmul_rn(u, ia);
    fold_col_put(gext, g, -y1, -y2, -y3, -y4, 0.f);  // the accumulator holds -ip - E
}

// column constants of every grouped row (one half of a 64-byte ColPair record
// per (query, list) pair; pad rows (gpair < 0) are left untouched: every
// consumer masks columns past the group's size)
// (re-scan: tau / pair carry the 64-bit (key, row) threshold instead)
__global__ void colc_kernel(const int32_t* __restrict__ gpair, int64_t nrows, int nprobe, int D,
                            const float4* __restrict__ qscal, const float* __restrict__ tau,
                            const uint64_t* __restrict__ tau64, float eps0, const int64_t* __restrict__ dbase,
                            const int64_t* __restrict__ doff, const int32_t* __restrict__ probes,
                            const float* __restrict__ list_amax, ColPair* __restrict__ gcolp,
                            float* __restrict__ gext, int Dp) {
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < nrows; g += (int64_t)gridDim.x * blockDim.x) {
        const int p = gpair[g];
        if (p < 0) {
            if (gext) fold_col_const(gext, g, kFoldBig);  // pad column: never flagged (D > 0)
            continue;
        }
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
        colp_put(gcolp, (int)g, cc);
        if (gext) fold_col(gext, g, cc, Dp);
    }
}

__global__ void pad_rows_kernel(int nlist, const int64_t* __restrict__ gcount, int64_t* __restrict__ gsz) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= nlist; j += gridDim.x * blockDim.x)
        gsz[j] = j == nlist ? 0 : (gcount[j] + kBoxRows - 1) / kBoxRows * kBoxRows;
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
                                    uint4* __restrict__ out, bool f8) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (nslots + kTM) * W;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = e / W;
        const int w = (int)(e % W);
        uint4 lo = make_uint4(0u, 0u, 0u, 0u), hi = lo;
        if (s < nslots) expand32(__ldg(codes + ((s >> 5) * W + w) * 32 + (s & 31)), lo, hi);
        if (f8) to_e4m3(lo, hi);
        out[2 * e] = lo;
        out[2 * e + 1] = hi;
    }
}

// ----------------------------------------------------- small-K grouped scan
// Dp <= 128 (CFG1, CFG3, CFG4, CFG5): one tile pass is a single K chunk, at
// most 4 UMMAs of M = 128, so the epilogue -- one TMEM read, the estimator
// and the threshold test per (query, vector) pair -- sets the pace.
// scan_imma_kernel above keeps all 16 epilogue warps on one tile with two
// accumulators and an item-wide barrier, which serialised every tile's
// latency chain (CFG4: 13.5 ms, issue active 47 %; ncu: 10 % of the stall
// samples on the per-tile row loads, 7 % on the tail, 8 % of the
// instructions in decode_item's binary search).  Here:
//  * the unit of epilogue work is (tile, block of <= 64 group columns): one
//    of 8 TMEM accumulator slots of 64 columns, up to 8 units in flight; each
//    of the 24 epilogue warps takes the next unit of its TMEM lane quarter
//    from a shared counter (6 warps per quarter), so a wide group keeps every
//    warp busy and a slow unit does not stall the others;
//  * the unit's per-vector constants (n_o^2 and f, popcount, row id, g1) are
//    staged in shared memory by bulk copies next to the accumulator slot;
//  * items (list, group of <= 256 queries, <= 8 tiles) come from a table
//    built once per launch and are taken dynamically (one atomic per item, no
//    tail) through a shared-memory ring of item records and their column
//    constants; the query operand (B) is double-buffered per item;
//  * every wait suspends in hardware (mbarrier.try_wait), no polling loops.
// Same per-pair arithmetic as scan_imma_kernel (est_of, the fast test), so the
// keys and survivors are bit-identical (tested).
constexpr int kSkNG = 256;                                   // group columns (B rows)
constexpr int kSkUW = 64;                                    // unit width (accumulator slot columns)
constexpr int kSkRI = 6;                                     // item ring
constexpr int kSkSA = 5;                                     // A stages (16 KB)
constexpr int kSkUS = kTmemCols / kSkUW;                     // 8 units in flight
constexpr int kSkEpi0 = 3;                                   // warps 0 sched + B, 1 A + row constants, 2 MMA
constexpr int kSkEpiW = 24;                                  // epilogue warps (6 per TMEM lane quarter)
constexpr int kSkNT = (kSkEpi0 + kSkEpiW) * 32;              // 864 threads (72 registers)
constexpr uint32_t kSkBStage = kSkNG * kKC;                  // 32 KB
constexpr uint32_t kSkCStage = kSkNG / 2 * sizeof(ColPair);  // 8 KB
struct SkRows {                                              // one unit's per-vector constants
    float2 fac[kTM];
    uint32_t rows[kTM];
    uint16_t pcnt[kTM];
};
constexpr uint32_t kSkOffA = 2 * kSkBStage;
constexpr uint32_t kSkOffC = kSkOffA + kSkSA * kAStage;
constexpr uint32_t kSkOffR = kSkOffC + kSkRI * kSkCStage;
constexpr uint32_t kSkSmem = kSkOffR + kSkUS * sizeof(SkRows) + 1024;  // + alignment slack

// item record: x = first slot of the list, y = its vectors (or sample prefix),
// z = first grouped row of the group, w = ncols | ntiles << 9 | t0 << 13 (t0 =
// first tile of the item in the list); w = 0 ends the work.  One warp per list.
__global__ void item_table_kernel(int nlist, const int64_t* __restrict__ list_off,
                                  const int64_t* __restrict__ slot_off, const int64_t* __restrict__ gstart,
                                  const int64_t* __restrict__ gcount, const int64_t* __restrict__ list_items,
                                  int4* __restrict__ items) {
    const int lane = threadIdx.x & 31;
    for (int j = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); j < nlist;
         j += (int)(((int64_t)gridDim.x * blockDim.x) >> 5)) {
        const int64_t i0 = list_items[j], ni = list_items[j + 1] - i0;
        if (ni == 0) continue;
        const int64_t L = list_off[j + 1] - list_off[j];
        const int64_t G = gcount[j];
        const int64_t ntl = (L + kTM - 1) / kTM;
        const int64_t nti = (ntl + kTilesPerItem - 1) / kTilesPerItem;
        const int sb = (int)slot_off[j], gs = (int)gstart[j];
        for (int64_t l = lane; l < ni; l += 32) {
            const int64_t g = l / nti, ti = l % nti;
            const int t0 = (int)(ti * kTilesPerItem);
            const int nt = (int)(ntl - t0 < kTilesPerItem ? ntl - t0 : kTilesPerItem);
            const int nc = (int)(G - g * kSkNG < kSkNG ? G - g * kSkNG : kSkNG);
            items[i0 + l] = make_int4(sb, (int)L, gs + (int)(g * kSkNG), nc | nt << 9 | t0 << 13);
        }
    }
}

// kMode: 0 main scan (fast test, survivors), 1 re-scan (exact (key, row) <=
// tau64), 2 dense key dump (threshold sample); kDump (main scan): also write
// every pair's ip and estimate to the debug dump (exact test path)
template <bool kLB, int kMode, bool kDump>
__global__ __launch_bounds__(kSkNT, 1) void scan_small_kernel(const __grid_constant__ CUtensorMap tmapB,
                                                              const __grid_constant__ CUtensorMap tmapA,
                                                              ScanArgs a, const int4* __restrict__ items,
                                                              int* __restrict__ sched) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;  // [2] B | [kSkSA] A | [kSkRI] column constants | [kSkUS] unit rows
    ColPair* colc = reinterpret_cast<ColPair*>(smem + kSkOffC);
    SkRows* urows = reinterpret_cast<SkRows*>(smem + kSkOffR);
    __shared__ int4 rec[kSkRI];
    __shared__ uint32_t next_unit[4];  // epilogue: next unit of each TMEM lane quarter
    __shared__ __align__(8) uint64_t ifull[kSkRI], iempty[kSkRI], bfull[2], bfree[2], afull[kSkSA], aempty[kSkSA],
        accf[kSkUS], acce[kSkUS], rowf[kSkUS];
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 2) tc::tmem_alloc(&tmem_base_s, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s < kSkRI; ++s) {
            tc::mbar_init(&ifull[s], 1);
            tc::mbar_init(&iempty[s], 2 + kSkEpiW);  // A loader, MMA warp, every epilogue warp
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&bfull[b], 1);
            tc::mbar_init(&bfree[b], 1);
        }
        for (int s = 0; s < kSkSA; ++s) {
            tc::mbar_init(&afull[s], 1);
            tc::mbar_init(&aempty[s], 1);
        }
        for (int k = 0; k < kSkUS; ++k) {
            tc::mbar_init(&accf[k], 1);
            tc::mbar_init(&acce[k], 4);  // the 4 warps of the unit's warpgroup
            tc::mbar_init(&rowf[k], 1);
        }
        for (int q = 0; q < 4; ++q) next_unit[q] = 0u;
        tc::prefetch_tmap(&tmapB);
        tc::prefetch_tmap(&tmapA);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base_s;
    const int64_t nitems = a.list_items[a.nlist];

    if (warp == 0) {
        // ============ scheduler: item records, column constants, query operand (B) ============
        if (lane == 0) {
            for (uint32_t i = 0;; ++i) {
                const int s = (int)(i % kSkRI);
                if (i >= (uint32_t)kSkRI) tc::mbar_wait(&iempty[s], ((i / kSkRI) - 1) & 1);
                const int64_t id = atomicAdd(sched, 1);
                if (id >= nitems) {
                    rec[s] = make_int4(0, 0, 0, 0);
                    tc::mbar_arrive(&ifull[s]);
                    break;
                }
                const int4 r = __ldg(items + id);
                rec[s] = r;
                const int nc = r.w & 511;
                const uint32_t cb = (uint32_t)(((nc + 15) & ~15) / 2) * (uint32_t)sizeof(ColPair);
                tc::mbar_arrive_expect_tx(&ifull[s], cb);
                tc::bulk_load(colc + s * (kSkNG / 2), a.gcolp + r.z / 2, cb, &ifull[s]);
                const int b = (int)(i & 1u);
                if (i >= 2) tc::mbar_wait(&bfree[b], ((i >> 1) - 1) & 1);
                const int nb = (nc + kBoxRows - 1) / kBoxRows;
                tc::mbar_arrive_expect_tx(&bfull[b], (uint32_t)(nb * kBoxRows * kKC));
                for (int bx = 0; bx < nb; ++bx)
                    tc::tma_load_2d(smem + b * kSkBStage + bx * kBoxRows * kKC, &tmapB, &bfull[b], 0,
                                    r.z + bx * kBoxRows);
            }
        }
    } else if (warp == 1) {
        // ============ code operand (A) by TMA ============
        if (lane == 0) {
            uint32_t tcnt = 0, ucnt = 0;
            for (uint32_t i = 0;; ++i) {
                const int s = (int)(i % kSkRI);
                tc::mbar_wait(&ifull[s], (i / kSkRI) & 1);
                const int4 r = rec[s];
                tc::mbar_arrive(&iempty[s]);
                if (r.w == 0) break;
                const int nt = (r.w >> 9) & 15, t0 = (int)((uint32_t)r.w >> 13);
                const int nu = ((r.w & 511) + kSkUW - 1) / kSkUW;
                for (int t = 0; t < nt; ++t, ++tcnt) {
                    const int st = (int)(tcnt % kSkSA);
                    if (tcnt >= (uint32_t)kSkSA) tc::mbar_wait(&aempty[st], ((tcnt / kSkSA) - 1) & 1);
                    tc::mbar_arrive_expect_tx(&afull[st], (uint32_t)kAStage);
                    tc::tma_load_2d(smem + kSkOffA + st * kAStage, &tmapA, &afull[st], 0, r.x + (t0 + t) * kTM);
                    // the tile's per-vector constants, once per unit, as each unit slot frees up
                    // (issued right behind the tile's code operand: measured faster than a
                    // separate loader warp, whose copies queue behind code tiles issued ahead)
                    const int v0 = (t0 + t) * kTM;
                    const int nv = r.y - v0 < kTM ? r.y - v0 : kTM;
                    const uint32_t ncp = (uint32_t)((nv + 31) & ~31);  // whole 32-slot blocks of the list
                    const int64_t s0 = (int64_t)r.x + v0;
                    for (int u = 0; u < nu; ++u, ++ucnt) {
                        const int k = (int)(ucnt % kSkUS);
                        if (ucnt >= (uint32_t)kSkUS) tc::mbar_wait(&acce[k], ((ucnt / kSkUS) - 1) & 1);
                        SkRows& R = urows[k];
                        tc::mbar_arrive_expect_tx(&rowf[k], ncp * 14u);
                        tc::bulk_load(R.fac, a.fac + s0, ncp * 8u, &rowf[k]);
                        tc::bulk_load(R.pcnt, a.pcnt + s0, ncp * 2u, &rowf[k]);
                        tc::bulk_load(R.rows, a.rows + s0, ncp * 4u, &rowf[k]);
                    }
                }
            }
        }
    } else if (warp == 2) {
        // ============ MMA issuer: per unit nks UMMAs (N <= 64) into slot ucnt % 8 ============
        uint32_t tcnt = 0, ucnt = 0;
        const int nks = a.Dp / 32;
        for (uint32_t i = 0;; ++i) {
            const int s = (int)(i % kSkRI);
            tc::mbar_wait(&ifull[s], (i / kSkRI) & 1);
            const int4 r = rec[s];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&iempty[s]);
            if (r.w == 0) break;
            const int nc = r.w & 511, nt = (r.w >> 9) & 15;
            const int nu = (nc + kSkUW - 1) / kSkUW;
            const int b = (int)(i & 1u);
            tc::mbar_wait(&bfull[b], (i >> 1) & 1);
            tc::fence_after_sync();
            const uint32_t bbase = tc::smem_u32(smem + b * kSkBStage);
            for (int t = 0; t < nt; ++t, ++tcnt) {
                const int as = (int)(tcnt % kSkSA);
                tc::mbar_wait(&afull[as], (tcnt / kSkSA) & 1);
                tc::fence_after_sync();
                const uint64_t adesc = tc::smem_desc_sw128(tc::smem_u32(smem + kSkOffA + as * kAStage));
                for (int u = 0; u < nu; ++u, ++ucnt) {
                    const int k = (int)(ucnt % kSkUS);
                    if (ucnt >= (uint32_t)kSkUS) {
                        tc::mbar_wait(&acce[k], ((ucnt / kSkUS) - 1) & 1);
                        tc::fence_after_sync();
                    }
                    const int w = nc - u * kSkUW < kSkUW ? nc - u * kSkUW : kSkUW;
                    const uint32_t idesc = tc::idesc_f8(kTM, (w + 15) & ~15);
                    // B rows [64 u, 64 u + w): 64 rows = 8 swizzle atoms further
                    const uint64_t bdesc = tc::smem_desc_sw128(bbase + (uint32_t)(u * kSkUW * kKC));
                    tc::mma_i8_ss_chunk<true>(tmem + (uint32_t)(k * kSkUW), adesc, bdesc, idesc, 0u, nks, &accf[k]);
                }
                tc::commit_warp(&aempty[as]);                // the tile's code operand is free
                if (t == nt - 1) tc::commit_warp(&bfree[b]);  // the item's query operand is free
            }
        }
    } else if (warp >= kSkEpi0) {
        // ============ epilogue: 32 rows (the warp's TMEM lane quarter) x a unit's columns ============
        // Units are taken dynamically, per lane quarter: the 4 warps of quarter q
        // share a counter, so a unit that takes long (many survivors) holds up
        // neither the other quarters nor the other units; the MMA fills units in
        // order and blocks only when it wraps around to a slot still in use.
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t rowf_s = tc::smem_u32(rowf), accf_s = tc::smem_u32(accf), acce_s = tc::smem_u32(acce);
        uint32_t i = 0, u0 = 0;  // item cursor and its first unit
        int4 R = make_int4(0, 0, 0, 0);
        int nu = 0, nut = -1;     // nut < 0: item i not read yet
        for (;;) {
            uint32_t uc = 0;
            if (lane == 0) uc = atomicAdd(&next_unit[quarter], 1u);
            uc = __shfl_sync(0xFFFFFFFFu, uc, 0);
            bool done = false;
            for (;;) {  // advance to the item holding unit uc, releasing the items passed
                if (nut < 0) {
                    tc::mbar_wait(&ifull[i % kSkRI], (i / kSkRI) & 1);
                    R = rec[i % kSkRI];
                    if (R.w == 0) {
                        done = true;
                        break;
                    }
                    nu = ((R.w & 511) + kSkUW - 1) / kSkUW;
                    nut = ((R.w >> 9) & 15) * nu;
                }
                if (uc < u0 + (uint32_t)nut) break;
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&iempty[i % kSkRI]);
                u0 += (uint32_t)nut;
                ++i;
                nut = -1;
            }
            if (done) break;
            const int s = (int)(i % kSkRI);
            const int nc = R.w & 511, t0 = (int)((uint32_t)R.w >> 13);
            const int x = (int)(uc - u0);
            // x / nu for nu in 1..4 without an integer division (x < 32 * 4)
            const int t = nu == 1 ? x : nu == 2 ? x >> 1 : nu == 4 ? x >> 2 : (x * 43) >> 7, u = x - t * nu;
            const int64_t v = (int64_t)(t0 + t) * kTM + r;
            const bool vok = v < R.y;
            {
                {
                    const int k = (int)(uc % kSkUS);
                    const uint32_t ph = (uc / kSkUS) & 1;
                    const ColPair* cb = colc + s * (kSkNG / 2) + u * (kSkUW / 2);
                    const int w = nc - u * kSkUW < kSkUW ? nc - u * kSkUW : kSkUW;
                    tc::mbar_wait_s(rowf_s + 8u * k, ph);
                    const SkRows& RS = urows[k];
                    const float2 fac = vok ? RS.fac[r] : make_float2(0.f, 0.f);
                    const float pcf = vok ? (float)RS.pcnt[r] : 0.f;
                    const float g1 = (kLB && vok) ? __ldg(a.g1 + R.x + v) : 0.f;  // lower-bound key only
                    const uint32_t row = vok ? RS.rows[r] : 0u;
                    tc::mbar_wait_s(accf_s + 8u * k, ph);
                    tc::fence_after_sync();
                    const uint32_t tbase = lane_base + (uint32_t)(k * kSkUW);
                    constexpr int kH = kSkUW / kEC;  // 16-column chunks per unit
                    uint32_t hc_cols[kH], hc_bal[kH];
                    int hc_base[kH];
#pragma unroll
                    for (int h = 0; h < kH; ++h) {
                        hc_cols[h] = 0u;
                        hc_bal[h] = 0u;
                        hc_base[h] = 0;
                        const int col0 = h * kEC;
                        if (col0 < w) {
                            uint32_t acc[kEC];
                            tc::tmem_ld16(tbase + (uint32_t)col0, acc);
                            if constexpr (kMode == 2) {
                                // sample scan: every key, coalesced (lanes = consecutive vectors)
                                if (vok) {
#pragma unroll
                                    for (int i2 = 0; i2 < kEC; ++i2) {
                                        if (col0 + i2 < w) {
                                            const ColC cc = colp_get(cb, col0 + i2);
                                            const float key = rank_key<kLB>(est_of<true>(acc[i2], cc, fac, pcf), epsnq_of(cc), g1);
                                            const int64_t off = ((int64_t)(uint32_t)cc.pair << 32) | (uint32_t)cc.q;
                                            a.dense_keys[off + v] = f2o(key);
                                        }
                                    }
                                }
                            } else {
                                uint32_t rowbits = 0u;
                                if constexpr (!kLB && kMode == 0 && !kDump) {
                                    // fast test, two columns per packed op: v = fma(-f, fma(-a, ipn,
                                    // fma(b, pcf, -K)), A) <= U <=> U - v >= 0 (sign bit clear; the
                                    // difference of two floats is never -0 when v > U).  Sign bits
                                    // are shifted in from the last column down (one SHF per column).
                                    const float2 pc2 = make_float2(pcf, pcf), nf2 = make_float2(-fac.y, -fac.y);
                                    const float2 fx2 = make_float2(fac.x, fac.x);
                                    const float4* P0 = reinterpret_cast<const float4*>(cb + (col0 >> 1));
                                    // two independent shift chains (columns 15..8 and 7..0) so the
                                    // dependent funnel shifts overlap
                                    uint32_t neg_hi = 0u, neg_lo = 0u;
#pragma unroll
                                    for (int i2 = kEC - 2; i2 >= 0; i2 -= 2) {
                                        const float4* P = P0 + 2 * i2;
                                        const float4 ab = P[0], ku = P[1];  // (-a0, -a1, b0, b1), (-K0, -K1, U0, U1)
                                        const float2 ipn = make_float2(__uint_as_float(acc[i2]), __uint_as_float(acc[i2 + 1]));
                                        const float2 inner = ffma2(make_float2(ab.z, ab.w), pc2, make_float2(ku.x, ku.y));
                                        const float2 tt = ffma2(make_float2(ab.x, ab.y), ipn, inner);
                                        const float2 vv = ffma2(nf2, tt, fx2);
                                        const float2 dd = fsub2(make_float2(ku.z, ku.w), vv);
                                        uint32_t& neg = i2 >= kEC / 2 ? neg_hi : neg_lo;
                                        neg = __funnelshift_l(__float_as_uint(dd.y), neg, 1);  // (neg << 1) | sign
                                        neg = __funnelshift_l(__float_as_uint(dd.x), neg, 1);
                                    }
                                    rowbits = ~((neg_hi << (kEC / 2)) | neg_lo) & 0xFFFFu;
                                } else {
#pragma unroll
                                    for (int i2 = 0; i2 < kEC; ++i2) {
                                        const ColC cc = colp_get(cb, col0 + i2);
                                        const float est = est_of<true>(acc[i2], cc, fac, pcf);
                                        const float key = rank_key<kLB>(est, epsnq_of(cc), g1);
                                        if constexpr (kDump) {
                                            if (vok && col0 + i2 < w) {
                                                const int64_t di = (a.item_off[cc.pair] + (v >> 5)) * 32 + (v & 31);
                                                if (di < a.dump_cap) {
                                                    a.dump_ip[di] = (int)-acc_ipn<true>(acc[i2]);
                                                    a.dump_est[di] = est;
                                                }
                                            }
                                        }
                                        bool sv;
                                        if constexpr (kMode == 1) {  // exact (key, row) <= tau64
                                            const uint32_t ko = f2o(key), to = f2o(cc.tau);
                                            sv = ko < to || (ko == to && row <= (uint32_t)cc.pair);
                                        } else {
                                            sv = key <= cc.tau;
                                        }
                                        rowbits |= sv ? (1u << i2) : 0u;
                                    }
                                }
                                const int rem = w - col0;
                                if (rem < kEC) rowbits &= (1u << rem) - 1u;
                                if (!vok) rowbits = 0u;
                                const uint32_t cols = __reduce_or_sync(0xFFFFFFFFu, rowbits);
                                hc_cols[h] = cols;
                                if (cols) {
                                    uint32_t mybal = 0u;
                                    for (uint32_t m = cols; m; m &= m - 1) {
                                        const int i2 = __ffs(m) - 1;
                                        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (rowbits >> i2) & 1u);
                                        if (lane == i2) mybal = bal;
                                    }
                                    hc_bal[h] = mybal;
                                    if (mybal) hc_base[h] = atomicAdd(&a.cnt[colp_get(cb, col0 + (lane & (kEC - 1))).q], __popc(mybal));
                                }
                            }
                        }
                    }
                    if constexpr (kMode != 2) {
                        // survivors re-read their accumulator column and store (key, row)
#pragma unroll
                        for (int h = 0; h < kH; ++h) {
                            const uint32_t cols = hc_cols[h];
                            if (!cols) continue;
                            const int col0 = h * kEC;
                            for (uint32_t m = cols; m; m &= m - 1) {
                                const int i2 = __ffs(m) - 1;
                                const uint32_t bal = __shfl_sync(0xFFFFFFFFu, hc_bal[h], i2);
                                const int base = __shfl_sync(0xFFFFFFFFu, hc_base[h], i2);
                                const uint32_t acci = tc::tmem_ld1(tbase + (uint32_t)(col0 + i2));
                                if ((bal >> lane) & 1u) {
                                    const ColC cc = colp_get(cb, col0 + i2);
                                    const float key = rank_key<kLB>(est_of<true>(acci, cc, fac, pcf), epsnq_of(cc), g1);
                                    const int pos = base + __popc(bal & ((1u << lane) - 1u));
                                    if (pos < a.cap) a.buf[(size_t)cc.q * a.cap + pos] = make_key(key, row);
                                }
                            }
                        }
                    }
                    tc::fence_before_sync();
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive_s(acce_s + 8u * k);  // the slot (accumulator + rows) may be reused
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 2) tc::tmem_dealloc(tmem, kTmemCols);
}

// --------------------------------------------------- folded small-K scan
// Dp <= 128 main scan (est key, no dump): the survivor test runs on the
// tensor cores (fold_col above).  One accumulator per tile (N = the group's
// width rounded to 16, <= 256; two TMEM slots of 256 columns): the code x
// query contraction (-ip, .kind::f8f6f4) and, into the same accumulator, the
// K = 16 tf32 contraction of the row / column factors (-E), so D = -T and a
// pair is flagged iff D < 0.  Epilogue warps take 16-column chunks of the
// tile dynamically (per TMEM lane quarter), OR the 16 accumulators of a chunk
// and leave at once unless a sign bit is set somewhere in the warp; flagged
// pairs get their exact ip from the code and query rows (global, e4m3) and the
// scan's exact key.  A stages carry the tile's codes (TMA) and its X rows (16
// tf32 per vector, written by 4 producer warps from the tile's row
// constants); the row constants live in a per-tile ring.
#ifndef FX_UW
#define FX_UW 128
#endif
#ifndef FX_EPIW
#define FX_EPIW 12
#endif
#ifndef FX_GATE
#define FX_GATE 0
#endif
#ifndef FX_NS0
#define FX_NS0 32
#endif
#ifndef FX_NSMAX
#define FX_NSMAX 256
#endif
constexpr int kFxUW = FX_UW;                // unit width: a tile's group is split into <= 256 / kFxUW column parts
constexpr int kFxTS = kTmemCols / kFxUW;    // TMEM slots (units in flight), kFxUW columns each
#ifndef FX_SA
#define FX_SA 4
#endif
#ifndef FX_RT
#define FX_RT (FX_SA + 512 / FX_UW)
#endif
#ifndef FX_RI
#define FX_RI 6
#endif
constexpr int kFxSA = FX_SA;                // A stages (codes 16 KB + X 8 KB)
constexpr int kFxRT = FX_RT;                // row-constant ring (tiles)
constexpr int kFxRI = FX_RI;                // item records
constexpr int kFxEpiW = FX_EPIW;            // epilogue warps (kFxEpiW / 4 per TMEM lane quarter)
constexpr int kFxXW = 4;                    // X producer warps (one vector row per lane)
constexpr int kFxMmaW = 2 + kFxXW;          // warps 0 sched + B, 1 A loader, 2..5 X producers, 6 MMA
constexpr int kFxEpi0 = kFxMmaW + 1;
constexpr int kFxDefer = 32768;  // deferred (row, chunk) records per CTA (1 MB)
constexpr int kFxNT = (kFxEpi0 + kFxEpiW) * 32;  // 608 threads
constexpr int kFxCh = kFxUW / kEC;               // 8 chunks per unit and lane quarter (at most)
constexpr uint32_t kFxBStage = kSkNG * kKC;      // 32 KB query operand
constexpr uint32_t kFxBXStage = kSkNG * 64;      // 16 KB column factors (16 tf32 per column)
constexpr uint32_t kFxXStage = kTM * 64;         // 8 KB row factors
constexpr uint32_t kFxAStage = kAStage + kFxXStage;  // 24 KB
constexpr uint32_t kFxOffBX = 2 * kFxBStage;
constexpr uint32_t kFxOffA = kFxOffBX + 2 * kFxBXStage;  // multiple of 1024
constexpr uint32_t kFxOffR = kFxOffA + kFxSA * kFxAStage;
constexpr uint32_t kFxSmem = kFxOffR + kFxRT * sizeof(SkRows) + 1024;
static_assert(kFxSmem <= 227 * 1024, "fold scan shared memory");
static_assert(kFxOffA % 1024 == 0 && kFxAStage % 1024 == 0, "A stages 1024-aligned (128-byte swizzle)");
static_assert(kFxTS * kFxUW <= kTmemCols && kFxUW <= 8 * kEC, "fold scan TMEM (<= 8 chunks per unit: rb0 / rb1)");
static_assert(kFxEpiW % 4 == 0 && kFxEpiW / 4 <= kFxTS + 1, "fold scan: accf parity argument (epilogue warps per quarter)");

// units of a group of nc columns: nu parts of wu (multiple of 16, <= kFxUW) columns
__device__ __forceinline__ void fx_units(int nc, int& nu, int& wu) {
    nu = (nc + kFxUW - 1) / kFxUW;
    wu = nu == 1 ? ((nc + 15) & ~15) : (((nc + nu - 1) / nu + 15) & ~15);
}

// exact ip of code row x query row (both e4m3 bytes in the grouped scan's K
// order, codes 0xB8 = -1 / 0, queries 0..15): the flagged pairs' key input
__device__ __forceinline__ float ipn_rows(const uint8_t* __restrict__ crow, const uint8_t* __restrict__ qrow, int Dp) {
    __half2 s0 = __float2half2_rn(0.f), s1 = s0;
    for (int k = 0; k < Dp; k += 16) {
        const uint4 c = __ldg(reinterpret_cast<const uint4*>(crow + k));
        const uint4 q = __ldg(reinterpret_cast<const uint4*>(qrow + k));
        const uint32_t cw[4] = {c.x, c.y, c.z, c.w}, qw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t m = qw[i] & sgnrep(cw[i]);  // q where the code bit is set
            __half2_raw lo = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(m & 0xFFFFu), __NV_E4M3);
            __half2_raw hi = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(m >> 16), __NV_E4M3);
            s0 = __hadd2(s0, *reinterpret_cast<__half2*>(&lo));  // integers <= 15 Dp < 2048: exact
            s1 = __hadd2(s1, *reinterpret_cast<__half2*>(&hi));
        }
    }
    const float2 a = __half22float2(s0), b = __half22float2(s1);
    return -((a.x + a.y) + (b.x + b.y));  // -ip (the f8 accumulator's value), exact
}

// Exact keys of one vector row's flagged pairs within a 16-column chunk (one thread): the ip from the
// e4m3 rows, the scan's estimator, one counter atomic per pair.  Called from the tail phase on the
// deferred records (and in place when the CTA's record region is full).
__device__ __forceinline__ void fx_row_keys(const ScanArgs& a, float2 fac, float pcf, uint32_t row, int64_t crowi,
                                            int gcol0, uint32_t rowbits) {
    const uint8_t* crow = a.codes8 + (size_t)crowi * a.Dp;
    for (uint32_t m = rowbits; m; m &= m - 1) {
        const int gcol = gcol0 + __ffs(m) - 1;
        const ColC cq = colp_get(a.gcolp, gcol);
        const float ipn = ipn_rows(crow, a.qbar8 + (size_t)gcol * a.Dp, a.Dp);
        const float key = est_of<true>(__float_as_uint(ipn), cq, fac, pcf);
        const int pos = atomicAdd(&a.cnt[cq.q], 1);
        if (pos < a.cap) a.buf[(size_t)cq.q * a.cap + pos] = make_key(key, row);
    }
}

// Fast pass over N 16-column chunks of a unit (one TMEM wait): the sign bits of the accumulators.
// Returns the warp-uniform mask of chunks holding a flagged pair; their per-row bits (16 per
// chunk, columns >= ncols and invalid rows cleared) are OR-ed into rb.  N is a template parameter
// so that the registers of the read are a static array (predicated loads into one 4-chunk array
// spilled 176 bytes and doubled the scan time).
template <int N>
__device__ __forceinline__ uint32_t fx_pass(uint32_t taddr, bool vok, int ncols, uint64_t& rb) {
    uint32_t d2[N][kEC];
#pragma unroll
    for (int hh = 0; hh < N; ++hh) tc::tmem_ld16_nw(taddr + (uint32_t)(hh * kEC), d2[hh]);
    tc::tmem_ld_wait();
    uint32_t flag4 = 0u;
#pragma unroll
    for (int hh = 0; hh < N; ++hh) {
        uint32_t any = d2[hh][0];
#pragma unroll
        for (int c = 1; c < kEC; ++c) any |= d2[hh][c];
        flag4 |= (vok && (any >> 31)) ? (1u << hh) : 0u;
    }
    flag4 = __reduce_or_sync(0xFFFFFFFFu, flag4);
    if (flag4) {  // rare
#pragma unroll
        for (int hh = 0; hh < N; ++hh) {
            if ((flag4 >> hh) & 1u) {
                uint32_t rowbits = 0u;
#pragma unroll
                for (int c = kEC - 1; c >= 0; --c) rowbits = (rowbits << 1) | (d2[hh][c] >> 31);
                const int rem = ncols - hh * kEC;
                if (rem < kEC) rowbits &= (1u << rem) - 1u;
                if (!vok) rowbits = 0u;
                rb |= (uint64_t)rowbits << (16 * hh);
            }
        }
    }
    return flag4;
}

template <int NK>
__global__ __launch_bounds__(kFxNT, 1) void scan_fold_kernel(const __grid_constant__ CUtensorMap tmapB,
                                                             const __grid_constant__ CUtensorMap tmapA, ScanArgs a,
                                                             const float* __restrict__ gext,
                                                             const int4* __restrict__ items, int* __restrict__ sched) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
#ifdef RABITQ_DIAG
    volatile long long* crumb = a.trace ? (volatile long long*)a.trace + (size_t)blockIdx.x * 32 : nullptr;
#define FX_CRUMB(slot, val) do { if (crumb) crumb[slot] = (long long)(val); } while (0)
    // timeline of CTA 0 (one lane per event): event ev of tile / unit idx < 1024
#define FX_TL(ev, idx)                                                                   \
    do {                                                                                  \
        if (a.fold_tl && blockIdx.x == 0 && (uint32_t)(idx) < 1024u)                      \
            a.fold_tl[(ev) * 1024 + (int)(idx)] = clock64();                              \
    } while (0)
#else
#define FX_CRUMB(slot, val) do { } while (0)
#define FX_TL(ev, idx) do { } while (0)
#endif
    const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;  // [2] B | [2] BX | [kFxSA] (codes | X) | [kFxRT] row constants
    SkRows* urows = reinterpret_cast<SkRows*>(smem + kFxOffR);
    __shared__ int4 rec[kFxRI];
    __shared__ uint32_t next_chunk[4];
    __shared__ uint32_t defer_n;  // flagged (row, chunk) records deferred to the tail phase
    __shared__ uint32_t mma_issued;  // tiles whose MMAs the MMA warp has issued (epilogue wait gate)
    __shared__ __align__(8) uint64_t ifull[kFxRI], iempty[kFxRI], bfull[2], bfree[2], afull[kFxSA], xfull[kFxSA],
        aempty[kFxSA], accf[2 * kFxTS], acce[kFxTS], rowf[kFxRT];
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == kFxMmaW) tc::tmem_alloc(&tmem_base_s, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s < kFxRI; ++s) {
            tc::mbar_init(&ifull[s], 1);
            tc::mbar_init(&iempty[s], 2 + kFxXW + kFxEpiW);  // A loader, X producers, MMA warp, epilogue warps
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&bfull[b], 1);
            tc::mbar_init(&bfree[b], 1);
        }
        for (int s = 0; s < kFxSA; ++s) {
            tc::mbar_init(&afull[s], 1);
            tc::mbar_init(&xfull[s], kFxXW);
            tc::mbar_init(&aempty[s], 1);
        }
        for (int k = 0; k < kFxTS; ++k) {
            tc::mbar_init(&accf[k], 1);
            tc::mbar_init(&accf[kFxTS + k], 1);
            tc::mbar_init(&acce[k], 4);  // one warp per TMEM lane quarter
        }
        for (int t = 0; t < kFxRT; ++t) tc::mbar_init(&rowf[t], 1);
        for (int q = 0; q < 4; ++q) next_chunk[q] = 0u;
        defer_n = 0u;
        mma_issued = 0u;
        tc::prefetch_tmap(&tmapB);
        tc::prefetch_tmap(&tmapA);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base_s;
    const int64_t nitems = a.list_items[a.nlist];

    if (warp == 0) {
        // ============ scheduler: item records, query operand (B) and column factors (BX) ============
        if (lane == 0) {
            for (uint32_t i = 0;; ++i) {
                const int s = (int)(i % kFxRI);
                if (i >= (uint32_t)kFxRI) tc::mbar_wait(&iempty[s], ((i / kFxRI) - 1) & 1);
                const int64_t id = atomicAdd(sched, 1);
                if (id >= nitems) {
                    rec[s] = make_int4(0, 0, 0, 0);
                    tc::mbar_arrive(&ifull[s]);
                    break;
                }
                const int4 r = __ldg(items + id);
                rec[s] = r;
                FX_CRUMB(0, i);
                tc::mbar_arrive(&ifull[s]);
                const int nc = r.w & 511;
                const int b = (int)(i & 1u);
                if (i >= 2) tc::mbar_wait(&bfree[b], ((i >> 1) - 1) & 1);
                const int nb = (nc + kBoxRows - 1) / kBoxRows;
                const uint32_t bxb = a.fold_diag == 12 ? 0u : (uint32_t)(nb * kBoxRows) * 64u;
                tc::mbar_arrive_expect_tx(&bfull[b], (uint32_t)(nb * kBoxRows * kKC) + bxb);
                for (int bx = 0; bx < nb; ++bx)
                    tc::tma_load_2d(smem + b * kFxBStage + bx * kBoxRows * kKC, &tmapB, &bfull[b], 0,
                                    r.z + bx * kBoxRows);
                if (bxb) tc::bulk_load(smem + kFxOffBX + b * kFxBXStage, gext + (int64_t)r.z * 16, bxb, &bfull[b]);
            }
        }
    } else if (warp == 1) {
        // ============ code operand (A) by TMA + the tile's row constants ============
        if (lane == 0) {
            uint32_t tcnt = 0;
            for (uint32_t i = 0;; ++i) {
                const int s = (int)(i % kFxRI);
                tc::mbar_wait(&ifull[s], (i / kFxRI) & 1);
                const int4 r = rec[s];
                tc::mbar_arrive(&iempty[s]);
                if (r.w == 0) break;
                const int nt = (r.w >> 9) & 15, t0 = (int)((uint32_t)r.w >> 13);
                for (int t = 0; t < nt; ++t, ++tcnt) {
                    const int st = (int)(tcnt % kFxSA);
                    if (tcnt >= (uint32_t)kFxSA) tc::mbar_wait(&aempty[st], ((tcnt / kFxSA) - 1) & 1);
                    FX_CRUMB(1, tcnt);
                    FX_TL(0, tcnt);
                    tc::mbar_arrive_expect_tx(&afull[st], (uint32_t)kAStage);
                    tc::tma_load_2d(smem + kFxOffA + st * kFxAStage, &tmapA, &afull[st], 0, r.x + (t0 + t) * kTM);
                    // row constants of tile tcnt: slot tcnt % 8 was last used by tile tcnt - 8,
                    // whose accumulator slot (released only after its epilogue) precedes tile
                    // tcnt - 2's MMA, which precedes this tile's A stage reuse (tcnt - 4)
                    const int rt = (int)(tcnt % kFxRT);
                    const int v0 = (t0 + t) * kTM;
                    const int nv = r.y - v0 < kTM ? r.y - v0 : kTM;
                    const uint32_t ncp = (uint32_t)((nv + 31) & ~31);
                    const int64_t s0 = (int64_t)r.x + v0;
                    SkRows& R = urows[rt];
                    tc::mbar_arrive_expect_tx(&rowf[rt], ncp * 14u);
                    tc::bulk_load(R.fac, a.fac + s0, ncp * 8u, &rowf[rt]);
                    tc::bulk_load(R.pcnt, a.pcnt + s0, ncp * 2u, &rowf[rt]);
                    tc::bulk_load(R.rows, a.rows + s0, ncp * 4u, &rowf[rt]);
                }
            }
        }
    } else if (warp < kFxMmaW) {
        // ============ X producers: 16 tf32 row factors per vector of each tile ============
        uint32_t tcnt = 0;
        const int rr = (warp - 2) * 32 + lane;
        for (uint32_t i = 0;; ++i) {
            const int s = (int)(i % kFxRI);
            tc::mbar_wait(&ifull[s], (i / kFxRI) & 1);
            const int4 r = rec[s];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&iempty[s]);
            if (r.w == 0) break;
            const int nt = (r.w >> 9) & 15, t0 = (int)((uint32_t)r.w >> 13);
            for (int t = 0; t < nt; ++t, ++tcnt) {
                const int st = (int)(tcnt % kFxSA), rt = (int)(tcnt % kFxRT);
                if (tcnt >= (uint32_t)kFxSA) tc::mbar_wait(&aempty[st], ((tcnt / kFxSA) - 1) & 1);
                tc::mbar_wait(&rowf[rt], (tcnt / kFxRT) & 1);
                const SkRows& R = urows[rt];
                if (lane == 0) FX_CRUMB(2 + (warp - 2), tcnt);
                if (lane == 0 && warp == 2) FX_TL(1, tcnt);
                uint8_t* xs = smem + kFxOffA + st * kFxAStage + kAStage;
                const int nv = r.y - (t0 + t) * kTM;
                float pc = 0.f, ah = 0.f, al = 0.f, bh = 0.f, bl = 0.f;
                if (rr < nv) {
                    const float2 fc = R.fac[rr];
                    pc = (float)R.pcnt[rr];
                    const float beta = __frcp_rn(fc.y), alpha = __fmul_rn(fc.x, beta);
                    if (fc.y > 0.f && isfinite(beta) && isfinite(alpha)) {
                        ah = tc::tf32_rna(alpha);
                        al = tc::tf32_rna(__fsub_rn(alpha, ah));
                        bh = tc::tf32_rna(beta);
                        bl = tc::tf32_rna(__fsub_rn(beta, bh));
                    } else {
                        ah = -kFoldBig;  // f = 0 (n_o = 0): always flagged (with the negated y3 > 0)
                    }
                }
                float4* o = reinterpret_cast<float4*>(xs + (rr >> 3) * 512 + (rr & 7) * 16);
                if (a.fold_diag != 11) {
                o[0] = make_float4(pc, pc, 1.f, 1.f);
                o[8] = make_float4(ah, ah, al, bh);
                o[16] = make_float4(bh, bl, 0.f, 0.f);
                o[24] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
                tc::fence_proxy_async();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&xfull[st]);
                if (lane == 0 && warp == 2) FX_TL(2, tcnt);
            }
        }
    } else if (warp == kFxMmaW) {
        // ============ MMA issuer: per unit D = -ip - E into slot ucnt % 4 ============
        uint32_t tcnt = 0, ucnt = 0;
        const uint32_t accf_s = tc::smem_u32(accf), acce_s = tc::smem_u32(acce);
        for (uint32_t i = 0;; ++i) {
            const int s = (int)(i % kFxRI);
            tc::mbar_wait(&ifull[s], (i / kFxRI) & 1);
            const int4 r = rec[s];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&iempty[s]);
            if (r.w == 0) break;
            const int nc = r.w & 511, nt = (r.w >> 9) & 15;
            // units: the group's columns in nu <= 2 halves of wu (multiple of 16) columns
            int nu, wu;
            fx_units(nc, nu, wu);
            const int wl = ((nc - (nu - 1) * wu) + 15) & ~15;  // last unit's MMA width
            const uint32_t id8 = tc::idesc_f8(kTM, wu), id32 = tc::idesc_tf32_f32(kTM, wu);
            const uint32_t id8l = tc::idesc_f8(kTM, wl), id32l = tc::idesc_tf32_f32(kTM, wl);
            const int b = (int)(i & 1u);
            tc::mbar_wait(&bfull[b], (i >> 1) & 1);
            __syncwarp();
            tc::fence_after_sync();
            const uint64_t bdesc = tc::smem_desc_sw128(tc::smem_u32(smem + b * kFxBStage));
            const uint64_t bxdesc = tc::smem_desc(tc::smem_u32(smem + kFxOffBX + b * kFxBXStage), 128, 512);
#pragma unroll 1
            for (int t = 0; t < nt; ++t) {
                const int as = (int)(tcnt % kFxSA);
                tc::mbar_wait(&afull[as], (tcnt / kFxSA) & 1);
                tc::mbar_wait(&xfull[as], (tcnt / kFxSA) & 1);
                if (lane == 0) FX_TL(3, tcnt);
                const uint32_t abase = tc::smem_u32(smem + kFxOffA + as * kFxAStage);
                const uint64_t adesc = tc::smem_desc_sw128(abase), xdesc = tc::smem_desc(abase + kAStage, 128, 512);
#pragma unroll 1
                for (int u = 0; u < nu; ++u, ++ucnt) {
                    const uint32_t k = ucnt % kFxTS;
                    if (ucnt >= (uint32_t)kFxTS) tc::mbar_wait_s(acce_s + 8u * k, ((ucnt / kFxTS) - 1) & 1);
                    __syncwarp();  // the waits loop per thread: reconverge before elect.sync / tcgen05
                    if (lane == 0) FX_TL(4, ucnt);
                    tc::fence_after_sync();
                    const uint32_t dt = tmem + k * (uint32_t)kFxUW;
                    const bool last = u == nu - 1;
                    // B rows [u wu, +wu): wu x 128 B (SW128: 16-byte descriptor units); BX: wu / 8 x 512 B
                    tc::mma_fold_acc_w<NK>(dt, adesc, bdesc + (uint64_t)(u * wu * 8), last ? id8l : id8, xdesc,
                                           bxdesc + (uint64_t)(u * wu * 4), last ? id32l : id32,
#if FX_GATE
                                           accf_s + 8u * k);
#else
                                           accf_s + 8u * (ucnt % (2u * kFxTS)));
#endif
#if FX_GATE
                    if (lane == 0) atomicExch(&mma_issued, ucnt + 1u);
#endif
                    if (lane == 0) FX_TL(5, ucnt);
                }
                tc::commit_warp(&aempty[as]);                // the tile's codes and X rows are free
                if (t == nt - 1) tc::commit_warp(&bfree[b]);  // the item's B and BX are free
                ++tcnt;
            }
        }
    } else {
        // ============ epilogue: a unit's <= 128 columns x the warp's lane quarter ============
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        const uint32_t rowf_s = tc::smem_u32(rowf), accf_s = tc::smem_u32(accf), acce_s = tc::smem_u32(acce);
        uint32_t i = 0, u0 = 0, tc0 = 0;  // item cursor, its first unit and first tile
        int4 R = make_int4(0, 0, 0, 0);
        int nu = 1, wu = 16, nut = -1;
        for (;;) {
            uint32_t uc = 0;
            if (lane == 0) uc = atomicAdd(&next_chunk[quarter], 1u);
            uc = __shfl_sync(0xFFFFFFFFu, uc, 0);
            bool done = false;
            for (;;) {
                if (nut < 0) {
                    tc::mbar_wait(&ifull[i % kFxRI], (i / kFxRI) & 1);
                    R = rec[i % kFxRI];
                    if (R.w == 0) {
                        done = true;
                        break;
                    }
                    const int nc_ = R.w & 511;
                    fx_units(nc_, nu, wu);
                    nut = ((R.w >> 9) & 15) * nu;
                }
                if (uc < u0 + (uint32_t)nut) break;
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&iempty[i % kFxRI]);
                u0 += (uint32_t)nut;
                tc0 += (uint32_t)((R.w >> 9) & 15);
                ++i;
                nut = -1;
            }
            if (done) break;
            const int nc = R.w & 511, t0 = (int)((uint32_t)R.w >> 13);
            const int x = (int)(uc - u0);
            // x / nu for nu in 1..4 without an integer division (x < 8 * 4)
            const int t = nu == 1 ? x : nu == 2 ? x >> 1 : nu == 4 ? x >> 2 : (x * 43) >> 7, u = x - t * nu;
            const int64_t v = (int64_t)(t0 + t) * kTM + r;
            const bool vok = v < R.y;
            const uint32_t tcnt = tc0 + (uint32_t)t;
            const uint32_t k = uc % kFxTS;
            const int cend = min(nc, (u + 1) * wu) - u * wu;  // valid columns of the unit
            if (lane == 0) FX_CRUMB(10 + (warp - kFxEpi0), ((long long)uc << 32) | (uint32_t)cend);
            if (lane == 0 && quarter == 0) FX_TL(6, uc);
#if FX_GATE
            // Once the MMA warp has issued unit uc, the slot's previous fill has completed
            // (issue waited for its release), so the accf parity wait is unambiguous however
            // far ahead of the MMA this warp took its unit; the tile's rowf phase is complete
            // by then as well (its X rows were consumed).
            if (*(volatile uint32_t*)&mma_issued <= uc) {
                uint32_t ns = FX_NS0;
                while (*(volatile uint32_t*)&mma_issued <= uc) {
                    __nanosleep(ns);
                    if (ns < FX_NSMAX) ns <<= 1;
                }
            }
            tc::mbar_wait_s(accf_s + 8u * k, (uc / kFxTS) & 1);
#else
            // No gate, no polling: unit uc's commit arrives on accf[uc % (2 TS)], two barriers per
            // TMEM slot used alternately, so the parity wait can only confuse "uc complete" with
            // "uc - 2 TS still in flight" -- and unit uc - 2 TS is finished when a warp takes uc:
            // the quarter's warps take units in order and hold one each; were uc - 2 TS unfinished,
            // its slot would not have been released, the MMA warp would be blocked before unit
            // uc - TS, and units uc - 2 TS and uc - TS .. uc - 1 (TS + 1 of them) would all be held
            // by the quarter's other kFxEpiW / 4 - 1 < TS + 1 warps.
            tc::mbar_wait_s(accf_s + 8u * (uc % (2u * kFxTS)), (uc / (2u * kFxTS)) & 1);
#endif
            __syncwarp();  // reconverge before tcgen05.ld.sync.aligned
            if (lane == 0 && quarter == 0) FX_TL(7, uc);
            tc::fence_after_sync();
            const uint32_t tb = lane_base + k * (uint32_t)kFxUW;
            // Fast pass: the sign bits of the unit's accumulators.  Flagged chunks leave their
            // per-row bits (16 per chunk) in rb0 / rb1; the slot is released before the slow
            // path runs, which needs only those bits and the row's constants (ncu: with the slow
            // path inside, a flagged chunk -- about one quarter-unit in ten at CFG4 -- held its
            // accumulator slot for the latency of its global loads and atomics, and the MMA
            // warp, 4 slots ahead at most, waited on it)
            uint64_t rb0 = 0ull, rb1 = 0ull;  // chunks 0-3 and 4-7 of the unit
            uint32_t flagged = 0u;            // warp-uniform: chunk j has a flagged pair
            for (int c2 = 0; c2 < cend; c2 += 4 * kEC) {
                // <= 64 columns per wait, only the unit's valid 16-column chunks (the epilogue
                // warps set the kernel's pace: every instruction per unit counts)
                const int ncols = cend - c2;
                uint64_t rb = 0ull;
                uint32_t flag4;
                if (ncols > 3 * kEC) flag4 = fx_pass<4>(tb + (uint32_t)c2, vok, ncols, rb);
                else if (ncols > 2 * kEC) flag4 = fx_pass<3>(tb + (uint32_t)c2, vok, ncols, rb);
                else if (ncols > kEC) flag4 = fx_pass<2>(tb + (uint32_t)c2, vok, ncols, rb);
                else flag4 = fx_pass<1>(tb + (uint32_t)c2, vok, ncols, rb);
                if (flag4) {
                    if (c2 == 0) rb0 = rb;
                    else rb1 = rb;
                    flagged |= flag4 << (c2 >> 4);
                }
            }
#ifdef RABITQ_DIAG
            if (a.fold_diag >= 8) {  // pure delay instead of the slow path (race hunting)
                if (flagged) __nanosleep(a.fold_diag == 9 ? 20000 : 2000);
                flagged = 0u;
            }
            if (a.fold_diag == 1) flagged = 0u;
            if (lane == 0 && quarter == 0 && flagged) FX_TL(12, uc);
#endif
            float2 fac = make_float2(0.f, 0.f);
            float pcf = 0.f;
            uint32_t row = 0u;
            if (flagged) {
                const int rt = (int)(tcnt % kFxRT);
                tc::mbar_wait_s(rowf_s + 8u * rt, (tcnt / kFxRT) & 1);
                const SkRows& RS = urows[rt];
                if (vok) {
                    fac = RS.fac[r];
                    pcf = (float)RS.pcnt[r];
                    row = RS.rows[r];
                }
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_s(acce_s + 8u * k);  // the slot (and its row constants) may be refilled
            if (lane == 0) FX_TL(8 + quarter, uc);
            // ---- flagged pairs: deferred.  Computing the exact keys here (column constants -> counter
            // atomic -> store: three dependent global round trips) kept the warp away from its next unit
            // for ~3 us, about one quarter-unit in six at CFG4, 1 ms of the 5.2 ms scan (RABITQ_DIAG run
            // without the slow path).  Each flagged (row, chunk) becomes a 32-byte record in the CTA's
            // global region (shared-memory counter, plain stores, nothing waited for); every thread of
            // the CTA computes the keys after the last item.
            for (uint32_t f = flagged; f; f &= f - 1) {
                const int j = __ffs(f) - 1;
                const uint32_t rowbits = (uint32_t)((j < 4 ? rb0 : rb1) >> (16 * (j & 3))) & 0xFFFFu;
                const int gcol0 = (int)((int64_t)R.z + u * wu + j * kEC);  // grouped row of the chunk's column 0
                const uint32_t has = __ballot_sync(0xFFFFFFFFu, rowbits != 0u);
                uint32_t base = 0u;
                if (lane == 0) base = atomicAdd(&defer_n, (uint32_t)__popc(has));
                base = __shfl_sync(0xFFFFFFFFu, base, 0);
                if (rowbits) {
                    const uint32_t pos = base + (uint32_t)__popc(has & ((1u << lane) - 1u));
                    const int64_t crowi = (int64_t)R.x + v;
                    if (pos < (uint32_t)a.fold_defer_cap) {
                        uint4* d = a.fold_defer + ((size_t)blockIdx.x * (size_t)a.fold_defer_cap + pos) * 2;
                        d[0] = make_uint4(__float_as_uint(fac.x), __float_as_uint(fac.y), __float_as_uint(pcf), row);
                        d[1] = make_uint4((uint32_t)crowi, (uint32_t)((uint64_t)crowi >> 32), (uint32_t)gcol0, rowbits);
                    } else {
                        fx_row_keys(a, fac, pcf, row, crowi, gcol0, rowbits);  // region full: in place
                    }
                }
            }
        }
    }
    if (lane == 0) FX_CRUMB(24, warp);
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) FX_CRUMB(25, 1);
    if (warp == kFxMmaW) tc::tmem_dealloc(tmem, kTmemCols);
    {  // tail phase: the deferred records (written before the barrier above by this CTA's epilogue warps)
        const uint32_t nd = min(defer_n, (uint32_t)a.fold_defer_cap);
        const uint4* d = a.fold_defer + (size_t)blockIdx.x * (size_t)a.fold_defer_cap * 2;
        for (uint32_t i = (uint32_t)tid; i < nd; i += (uint32_t)kFxNT) {
            const uint4 w0 = d[2 * i], w1 = d[2 * i + 1];
            fx_row_keys(a, make_float2(__uint_as_float(w0.x), __uint_as_float(w0.y)), __uint_as_float(w0.z), w0.w,
                        (int64_t)(((uint64_t)w1.y << 32) | (uint64_t)w1.x), (int)w1.z, w1.w);
        }
    }
#undef FX_CRUMB
#undef FX_TL
}

}  // namespace

void expand_codes(rabitq_index* idx, cudaStream_t st) {
    const size_t bytes = (size_t)(idx->nslots + kTM) * 32 * idx->W;
    RQ_CUDA(cudaMalloc(&idx->codes8, bytes));
    idx->codes8_f8 = idx->W <= 4;  // Dp <= 128: e4m3 operands (.kind::f8f6f4)
    expand_codes_kernel<<<4096, 256, 0, st>>>(idx->codes, idx->nslots, idx->W, reinterpret_cast<uint4*>(idx->codes8),
                                              idx->codes8_f8);
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

// upper bound on the work items of a grouping with `rows` grouped rows, no
// list holding more than max_group of them (items of list j = ceil(T_j / 8)
// ceil(G_j / 256) <= ceil(T_j / 8) (1 + G_j / 256), T_j = tiles of the list)
int64_t item_bound(const rabitq_index* idx, int64_t rows, int64_t max_group) {
    const int64_t t8max = ((idx->max_list + kTM - 1) / kTM + kTilesPerItem - 1) / kTilesPerItem;
    const int64_t b1 = idx->tiles8_sum * ((max_group + kSkNG - 1) / kSkNG);
    const int64_t b2 = idx->tiles8_sum + t8max * ((rows + kSkNG - 1) / kSkNG);
    return std::max<int64_t>(1, std::min(b1, b2));
}

void prepare_groups(const rabitq_index* idx, const int32_t* probes, int64_t n, const int32_t* sub, Groups& g,
                    cudaStream_t st, int& launches, int rows, bool ta) {
    const int nlist = idx->nlist;
    g.Dp = ((idx->D + 31) / 32) * 32;
    g.n = n;
    g.rows = rows;
    g.ta = ta && idx->codes8 != nullptr;
    // each list's rows start at a multiple of kBoxRows (pad rows: gpair = -1)
    g.nrows = n * rows + (int64_t)kBoxRows * nlist + kTN;
    g.gcount.alloc((size_t)nlist + 1, st);
    g.gstart.alloc((size_t)nlist + 1, st);
    g.itemc.alloc((size_t)nlist + 1, st);
    g.list_items.alloc((size_t)nlist + 1, st);
    g.gfill.alloc((size_t)nlist, st);
    g.gpos.alloc((size_t)n, st);
    g.gpair.alloc((size_t)g.nrows, st);
    g.qbar8.alloc((size_t)g.nrows * g.Dp, st);
    RQ_CUDA(cudaMemsetAsync(g.gcount.p, 0, ((size_t)nlist + 1) * sizeof(int64_t), st));
    RQ_CUDA(cudaMemsetAsync(g.gfill.p, 0, (size_t)nlist * sizeof(int32_t), st));
    RQ_CUDA(cudaMemsetAsync(g.gpair.p, 0xFF, (size_t)g.nrows * sizeof(int32_t), st));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 2048));
    group_count_kernel<<<grid, 256, 0, st>>>(probes, sub, n, g.gcount.p, rows);
    RQ_CHECK_LAUNCH();
    pad_rows_kernel<<<(nlist + 256) / 256, 256, 0, st>>>(nlist, g.gcount.p, g.itemc.p);
    RQ_CHECK_LAUNCH();
    size_t tb = 0;
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, g.itemc.p, g.gstart.p, nlist + 1, st));
    WBuf<uint8_t> tmp;
    tmp.alloc(tb, st);
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, g.itemc.p, g.gstart.p, nlist + 1, st));
    group_fill_kernel<<<grid, 256, 0, st>>>(probes, sub, n, g.gstart.p, g.gfill.p, g.gpos.p, g.gpair.p, rows);
    RQ_CHECK_LAUNCH();
    list_items_kernel<<<(nlist + 256) / 256, 256, 0, st>>>(nlist, idx->list_off, g.gcount.p, group_cols(g.Dp, g.ta),
                                                           g.itemc.p);
    RQ_CHECK_LAUNCH();
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, g.itemc.p, g.list_items.p, nlist + 1, st));
    launches += 8;
}

void group_items(const rabitq_index* idx, const int64_t* list_off, const Groups& g, WBuf<int64_t>& itemc,
                 WBuf<int64_t>& items, cudaStream_t st, int& launches) {
    const int nlist = idx->nlist;
    itemc.alloc((size_t)nlist + 1, st);
    items.alloc((size_t)nlist + 1, st);
    list_items_kernel<<<(nlist + 256) / 256, 256, 0, st>>>(nlist, list_off, g.gcount.p,
                                                           group_cols(g.Dp, g.ta), itemc.p);
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
    prepare_groups(idx, probes, n, list.p, sub, st, launches, full.rows, full.ta);
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
    ScanArgs a = a_in;  // a.nrows = grouped rows allocated (all pairs, or the re-scan's sub list)
    WBuf<ColPair> gcolp;
    gcolp.alloc((size_t)(a.nrows + 1) / 2 + kTN, st);
    // folded survivor test (scan_fold_kernel): the main est-key scan of the small-K path
    const bool small_k = a.codes8 != nullptr && a.small && a.f8 && a.Dp <= kKC && !a.full;
    const bool fold = small_k && a.fold && !lb && !dump && !retry && !dense;
    WBuf<float> gext;
    if (fold) gext.alloc(((size_t)a.nrows + 8) * 16, st);
    colc_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((a.nrows + 255) / 256, 2048)), 256, 0, st>>>(
        a.gpair, a.nrows, a.nprobe, a.D, a.qscal, a.tau, retry ? a.tau64 : nullptr, a.eps0,
        dense ? a.dense_base : nullptr, dense ? a.dense_off : nullptr, a.probes, a.list_amax, gcolp.p, gext.p, a.Dp);
    RQ_CHECK_LAUNCH();
    a.gcolp = gcolp.p;
    int dev = 0, sms = 148;
    RQ_CUDA(cudaGetDevice(&dev));
    RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // B = grouped int8 query rows [nrows x Dp]; TMA box 128 bytes x 16 rows, 128-byte swizzle
    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {(cuuint64_t)a.Dp, (cuuint64_t)a.nrows};
    const cuuint64_t gstride[1] = {(cuuint64_t)a.Dp};
    const cuuint32_t box[2] = {(cuuint32_t)kKC, (cuuint32_t)kBoxRows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = get_encode()(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(a.qbar8), gdim, gstride,
                               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RQ_REQUIRE(cr == CUDA_SUCCESS, RABITQ_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
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
    if (ta && a.small && a.f8 && a.Dp <= kKC && !a.full && (!dump || !(retry || dense))) {
        // small-K scan (Dp <= 128): item table, dynamic scheduler
        RQ_REQUIRE(group_cols(a.Dp, true) == kSkNG && a.items_bound > 0, RABITQ_ERR_INTERNAL,
                   "small-K scan: group width / item bound");
        WBuf<int4> items;
        items.alloc((size_t)a.items_bound, st);
        WBuf<int> sched;
        sched.alloc(1, st);
        RQ_CUDA(cudaMemsetAsync(sched.p, 0, sizeof(int), st));
        item_table_kernel<<<(unsigned)std::max(1, std::min(a.nlist, 8192) / 8), 256, 0, st>>>(
            a.nlist, a.list_off, a.slot_off, a.gstart, a.gcount, a.list_items, items.p);
        RQ_CHECK_LAUNCH();
        if (fold) {
            long long* crumbs_h = nullptr;
            const char* crumbs_path = rq_diag_env("RABITQ_FOLD_CRUMBS");
            if (crumbs_path) {
                RQ_CUDA(cudaHostAlloc(&crumbs_h, (size_t)sms * 32 * sizeof(long long), cudaHostAllocMapped));
                std::memset(crumbs_h, 0xFF, (size_t)sms * 32 * sizeof(long long));
                long long* dptr = nullptr;
                RQ_CUDA(cudaHostGetDevicePointer(&dptr, crumbs_h, 0));
                a.trace = dptr;
            }
            long long* tl_h = nullptr;
            const char* tl_path = rq_diag_env("RABITQ_FOLD_TIMELINE");
            if (tl_path) {
                RQ_CUDA(cudaHostAlloc(&tl_h, (size_t)16 * 1024 * sizeof(long long), cudaHostAllocMapped));
                std::memset(tl_h, 0, (size_t)16 * 1024 * sizeof(long long));
                long long* dptr = nullptr;
                RQ_CUDA(cudaHostGetDevicePointer(&dptr, tl_h, 0));
                a.fold_tl = dptr;
            }
            // deferred flagged records: kFxDefer x 32 B per CTA (a full region falls back to in-place keys)
            WBuf<uint4> defer;
            a.fold_defer_cap = a_in.fold_defer_cap > 0 ? a_in.fold_defer_cap : kFxDefer;
            defer.alloc((size_t)sms * (size_t)a.fold_defer_cap * 2, st);
            a.fold_defer = defer.p;
#define RQ_FOLD(NK)                                                                                          \
    do {                                                                                                       \
        RQ_CUDA(cudaFuncSetAttribute(scan_fold_kernel<NK>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                     (int)kFxSmem));                                                           \
        scan_fold_kernel<NK><<<sms, kFxNT, kFxSmem, st>>>(tmap, tmapA, a, gext.p, items.p, sched.p);          \
    } while (0)
            switch (a.Dp / 32) {
                case 1: RQ_FOLD(1); break;
                case 2: RQ_FOLD(2); break;
                case 3: RQ_FOLD(3); break;
                default: RQ_FOLD(4); break;
            }
#undef RQ_FOLD
            if (tl_h) {
                const cudaError_t e = cudaStreamSynchronize(st);
                if (FILE* f = fopen(tl_path, "wb")) {
                    fwrite(tl_h, sizeof(long long), (size_t)16 * 1024, f);
                    fclose(f);
                }
                RQ_CUDA(e);
            }
            if (crumbs_h) {
                const cudaError_t e = cudaStreamSynchronize(st);
                if (FILE* f = fopen(crumbs_path, "wb")) {
                    fwrite(crumbs_h, sizeof(long long), (size_t)sms * 32, f);
                    fclose(f);
                }
                RQ_CUDA(e);
            }
            RQ_CHECK_LAUNCH();
            return;
        }
#define RQ_SMALL(LB, MODE, DP)                                                                                 \
    do {                                                                                                        \
        RQ_CUDA(cudaFuncSetAttribute(scan_small_kernel<LB, MODE, DP>,                                           \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSkSmem));               \
        scan_small_kernel<LB, MODE, DP><<<sms, kSkNT, kSkSmem, st>>>(tmap, tmapA, a, items.p, sched.p);         \
    } while (0)
        const int mode = dense ? 2 : retry ? 1 : 0;
        if (lb) {
            if (mode == 0 && dump) RQ_SMALL(true, 0, true);
            else if (mode == 0) RQ_SMALL(true, 0, false);
            else if (mode == 1) RQ_SMALL(true, 1, false);
            else RQ_SMALL(true, 2, false);
        } else {
            if (mode == 0 && dump) RQ_SMALL(false, 0, true);
            else if (mode == 0) RQ_SMALL(false, 0, false);
            else if (mode == 1) RQ_SMALL(false, 1, false);
            else RQ_SMALL(false, 2, false);
        }
#undef RQ_SMALL
        RQ_CHECK_LAUNCH();
        return;
    }
    const SmemPlan plan = smem_plan(a.Dp, ta);
    RQ_REQUIRE(plan.slots >= 2 && plan.total <= (uint32_t)kSmemLimit, RABITQ_ERR_INTERNAL,
               "grouped scan: TMEM / shared-memory plan does not fit");
    const size_t smem = plan.total;
    const int grid = sms;
#define RQ_IMMA6(LB, DP, RT, DN, TA, FU, F8)                                                                   \
    do {                                                                                                        \
        RQ_CUDA(cudaFuncSetAttribute(scan_imma_kernel<LB, DP, RT, DN, TA, FU, F8>,                              \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));                  \
        scan_imma_kernel<LB, DP, RT, DN, TA, FU, F8><<<grid, n_threads(TA), smem, st>>>(tmap, tmapA, a);        \
    } while (0)
#define RQ_IMMA5(LB, DP, RT, DN, TA)                          \
    do {                                                      \
        if (a.full) RQ_IMMA6(LB, DP, RT, DN, TA, true, false);  \
        else if (a.f8) RQ_IMMA6(LB, DP, RT, DN, TA, false, true); \
        else RQ_IMMA6(LB, DP, RT, DN, TA, false, false);        \
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
