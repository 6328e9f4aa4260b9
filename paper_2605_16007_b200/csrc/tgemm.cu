// tgemm.cu -- fp32-accurate GEMM on the 5th-generation tensor cores (3xTF32).
//
// C = A B^T over fp32 rows, A [m x K] and B [n x K] both K-contiguous, with
// every operand split as x = hi + lo (hi = x rounded to tf32, lo = tf32 of the
// exact remainder) and C = lo_A hi_B + hi_A lo_B + hi_A hi_B accumulated in
// fp32 in TMEM by tcgen05.mma kind::tf32 (the dropped lo_A lo_B term is below
// 2^-22 relative).  Used for the three dense products of the search path:
//   S1 rotation      Q' = Q P            A = Q rows, B = rows of P^T
//   S2 probe         ||c'||^2 - 2 q'.c'   A = Q' rows, B = c' rows
//   S9 dense re-rank ||q||^2 + ||x||^2 - 2 q.x for the vectors of a query's
//                    nearest list (93 % of CFG2's top-M candidates lie there):
//                    A = the list's fp32 rows (gathered by id), B = the queries
//                    whose nearest list it is, so each list row is read once
//                    per query group instead of once per (query, candidate).
//
// One persistent CTA per SM: 4 producer warps (cp.async of raw fp32 row
// chunks into a staging ring, then hi/lo split into the canonical K-major
// no-swizzle layout), 1 MMA warp (3 passes x 2 UMMA K-steps per 16-float
// chunk), 4 epilogue warps (tcgen05.ld, fused epilogue, double-buffered
// accumulators).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "tc.cuh"
#include "tgemm.cuh"

namespace rabitq {
namespace {

constexpr int kBM = 128;            // A rows per tile (UMMA M, TMEM lanes)
constexpr int kBN = 256;            // max B rows per tile (UMMA N)
constexpr int kBK = 16;             // floats of K per stage (64 bytes per row)
constexpr int kRaw = 4;             // raw fp32 staging stages (prefetch distance kRaw - 1)
constexpr int kSpl = 2;             // split (hi/lo) stages
constexpr int kRawA = kBM * kBK * 4;          // 8 KB
constexpr int kRawB = kBN * kBK * 4;          // 16 KB
constexpr int kSplA = 2 * kRawA;              // hi + lo: 16 KB
constexpr int kSplB = 2 * kRawB;              // 32 KB
constexpr int kSBO = 4 * 128;                 // 8-row core-matrix groups: 4 K-adjacent core matrices of 128 B
constexpr int kProdWarps = 8, kMmaWarp = 8, kEpiWarp0 = 9, kEpiWarps = 4;
constexpr int kNT = (kEpiWarp0 + kEpiWarps) * 32;  // 416
constexpr uint32_t kTmemCols = 2 * kBN;

constexpr int kStg = 32 * 33;  // per epilogue warp: 32 x 32 output block, padded rows (row-major transpose)
constexpr size_t kSmem = 1024 + (size_t)kRaw * (kRawA + kRawB) + (size_t)kSpl * (kSplA + kSplB) + 4 * kBM * 4 +
                         (size_t)kEpiWarps * kStg * 4;

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)                       // c_format: F32
           | (2u << 7) | (2u << 10)        // a/b format: TF32
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// split a float4 of raw values into hi (tf32) and lo (tf32 of the remainder)
__device__ __forceinline__ void split4(const float4 v, float4& hi, float4& lo) {
    hi.x = tf32_rna(v.x);
    hi.y = tf32_rna(v.y);
    hi.z = tf32_rna(v.z);
    hi.w = tf32_rna(v.w);
    lo.x = tf32_rna(__fsub_rn(v.x, hi.x));
    lo.y = tf32_rna(__fsub_rn(v.y, hi.y));
    lo.z = tf32_rna(__fsub_rn(v.z, hi.z));
    lo.w = tf32_rna(__fsub_rn(v.w, hi.w));
}

struct TileInfo {
    int64_t a0, b0, c0;
    int m, n, ldc;
};

__device__ __forceinline__ TileInfo get_tile(const TgParams& p, int t) {
    TileInfo ti;
    if (p.tiles) {
        const TgTile& d = p.tiles[t];
        ti.a0 = d.a0;
        ti.b0 = d.b0;
        ti.c0 = d.c0;
        ti.m = d.m;
        ti.n = d.n;
        ti.ldc = d.ldc;
    } else {
        const int tn = (int)((p.N + kBN - 1) / kBN);
        const int tm = t / tn, tj = t % tn;
        ti.a0 = (int64_t)tm * kBM;
        ti.b0 = (int64_t)tj * kBN;
        const int64_t rm = p.M - ti.a0, rn = p.N - ti.b0;
        ti.m = (int)(rm < kBM ? rm : kBM);
        ti.n = (int)(rn < kBN ? rn : kBN);
        ti.ldc = (int)p.ldc;
        ti.c0 = ti.a0 * p.ldc + ti.b0;
    }
    return ti;
}

__device__ __forceinline__ int ntiles_of(const TgParams& p) {
    return p.tiles ? p.ntiles : (int)(((p.M + kBM - 1) / kBM) * ((p.N + kBN - 1) / kBN));
}

// kTma: A and B rows are plain (no index maps): one 2D TMA per operand and
// stage; otherwise 16-byte cp.async per row chunk (gathered rows)
template <int kEpi, bool kTma>
__global__ __launch_bounds__(kNT, 1) void tgemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                       const __grid_constant__ CUtensorMap tmB, const TgParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* smem = smem_raw + pad;
    uint8_t* rawA = smem;                                     // [kRaw][128 rows][16 floats] row-major
    uint8_t* rawB = rawA + kRaw * kRawA;                      // [kRaw][256 rows][16 floats]
    uint8_t* splA = rawB + kRaw * kRawB;                      // [kSpl][hi, lo][canonical 128 x 16]
    uint8_t* splB = splA + kSpl * kSplA;                      // [kSpl][hi, lo][canonical 256 x 16]
    float* anorm = reinterpret_cast<float*>(splB + kSpl * kSplB);  // [2 buffers][2 halves][128] A row norm parts
    float* stage = anorm + 4 * kBM;                                 // [kEpiWarps][32][33] store transpose
    __shared__ __align__(8) uint64_t full_bar[kSpl], empty_bar[kSpl], accf_bar[2], acce_bar[2], normf_bar[2],
        raw_bar[kRaw];
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == kMmaWarp) tc::tmem_alloc(&tmem_base_s, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s < kSpl; ++s) {
            tc::mbar_init(&full_bar[s], 1);
            tc::mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&accf_bar[b], 1);
            tc::mbar_init(&acce_bar[b], kEpiWarps);
            tc::mbar_init(&normf_bar[b], 1);
        }
        for (int e = 0; e < kRaw; ++e) tc::mbar_init(&raw_bar[e], 1);
        if (kTma) {
            tc::prefetch_tmap(&tmA);
            tc::prefetch_tmap(&tmB);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base_s;
    const int nt = ntiles_of(p);
    const int nk = (p.K + kBK - 1) / kBK;

    if (warp < kProdWarps) {
        // ================= producers: thread t converts B row t and half (t >> 7) of A row t & 127
        const int r = tid & (kBM - 1), half = tid >> 7;
        auto issue = [&](const TileInfo& ti, int kb, int e) {
            const int k0 = kb * kBK;
            if constexpr (kTma) {
                if (tid == 0) {
                    tc::mbar_arrive_expect_tx(&raw_bar[e], (uint32_t)(kRawA + kRawB));
                    tc::tma_load_2d(rawA + e * kRawA, &tmA, &raw_bar[e], k0, (int)ti.a0);
                    tc::tma_load_2d(rawB + e * kRawB, &tmB, &raw_bar[e], k0, (int)ti.b0);
                }
                return;
            }
            const int kv = min(kBK, p.K - k0);  // multiple of 4 (K % 4 == 0)
            {
                float* dst = reinterpret_cast<float*>(rawA + e * kRawA) + r * kBK;
                const bool ok = r < ti.m;
                const int64_t row = ok ? (p.a_idx ? (int64_t)p.a_idx[ti.a0 + r] : ti.a0 + r) : 0;
                const float* src = p.A + row * p.lda + k0;
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    const int c = 2 * half + cc;
                    const bool v = ok && 4 * c < kv;
                    tc::cp_async16_zfill(dst + 4 * c, v ? src + 4 * c : p.A, v ? 16u : 0u);
                }
            }
            {
                const int rb = tid;
                float* dst = reinterpret_cast<float*>(rawB + e * kRawB) + rb * kBK;
                const bool ok = rb < ti.n;
                const int64_t row = ok ? (p.b_idx ? (int64_t)p.b_idx[ti.b0 + rb] : ti.b0 + rb) : 0;
                const float* src = p.B + row * p.ldb + k0;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const bool v = ok && 4 * c < kv;
                    tc::cp_async16_zfill(dst + 4 * c, v ? src + 4 * c : p.B, v ? 16u : 0u);
                }
            }
            tc::cp_async_commit();
        };
        // stage sequence: (tile t, chunk kb) for t = blockIdx.x, blockIdx.x + grid, ...
        int it_t = blockIdx.x, it_k = 0;  // next stage to issue
        TileInfo it_ti{};
        if (it_t < nt) it_ti = get_tile(p, it_t);
        int issued = 0;
        auto issue_next = [&]() {
            if (it_t < nt) issue(it_ti, it_k, issued % kRaw);
            else if (!kTma) tc::cp_async_commit();
            ++issued;
            if (it_t < nt && ++it_k == nk) {
                it_k = 0;
                it_t += gridDim.x;
                if (it_t < nt) it_ti = get_tile(p, it_t);
            }
        };
        for (int i = 0; i < kRaw - 1; ++i) issue_next();
        uint32_t gs = 0;
        int tcount = 0;
        for (int t = blockIdx.x; t < nt; t += gridDim.x, ++tcount) {
            float nrm = 0.0f;  // squared norm of A row r (fp32, sequential over K)
            for (int kb = 0; kb < nk; ++kb, ++gs) {
                issue_next();
                const int e = (int)(gs % kRaw), s = (int)(gs % kSpl);
                if constexpr (kTma) tc::mbar_wait(&raw_bar[e], (gs / kRaw) & 1);
                else tc::cp_async_wait<kRaw - 1>();
                const uint32_t u = gs / kSpl;
                if (u > 0) tc::mbar_wait_backoff(&empty_bar[s], (u - 1) & 1);
                // A row r: 4 float4 -> hi / lo in core-matrix layout (r/8)*SBO + kc*128 + (r%8)*16
                {
                    const float4* src = reinterpret_cast<const float4*>(rawA + e * kRawA) + r * 4;
                    uint8_t* hi = splA + s * kSplA;
                    uint8_t* lo = hi + kRawA;
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        const int c = 2 * half + cc;
                        const float4 v = src[c];
                        nrm = __fmaf_rn(v.x, v.x, nrm);
                        nrm = __fmaf_rn(v.y, v.y, nrm);
                        nrm = __fmaf_rn(v.z, v.z, nrm);
                        nrm = __fmaf_rn(v.w, v.w, nrm);
                        float4 h, l;
                        split4(v, h, l);
                        const int off = (r >> 3) * kSBO + c * 128 + (r & 7) * 16;
                        *reinterpret_cast<float4*>(hi + off) = h;
                        *reinterpret_cast<float4*>(lo + off) = l;
                    }
                }
                {
                    const int rb = tid;
                    const float4* src = reinterpret_cast<const float4*>(rawB + e * kRawB) + rb * 4;
                    uint8_t* hi = splB + s * kSplB;
                    uint8_t* lo = hi + kRawB;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        float4 h, l;
                        split4(src[c], h, l);
                        const int off = (rb >> 3) * kSBO + c * 128 + (rb & 7) * 16;
                        *reinterpret_cast<float4*>(hi + off) = h;
                        *reinterpret_cast<float4*>(lo + off) = l;
                    }
                }
                // last chunk: publish the row norms of this tile for the epilogue
                // (buffer = tile parity; its previous readers arrived on acce before
                // the MMAs of this tile could start)
                if (kb == nk - 1) anorm[((tcount & 1) * 2 + half) * kBM + r] = nrm;
                tc::fence_proxy_async();
                tc::named_barrier(1, kProdWarps * 32);
                if (tid == 0) {
                    tc::mbar_arrive(&full_bar[s]);
                    if (kb == nk - 1) tc::mbar_arrive(&normf_bar[tcount & 1]);
                }
            }
        }
        if (!kTma) tc::cp_async_wait<0>();
    } else if (warp == kMmaWarp) {
        // ================= MMA issuer
        uint32_t gs = 0;
        int tcount = 0;
        const uint32_t aS = tc::smem_u32(splA), bS = tc::smem_u32(splB);
        for (int t = blockIdx.x; t < nt; t += gridDim.x, ++tcount) {
            const TileInfo ti = get_tile(p, t);
            const int n16 = max(16, (ti.n + 15) & ~15);
            const uint32_t idesc = idesc_tf32(kBM, n16);
            const int b = tcount & 1;
            const uint32_t ub = (uint32_t)tcount >> 1;
            if (ub > 0) tc::mbar_wait_backoff(&acce_bar[b], (ub - 1) & 1);
            tc::fence_after_sync();
            const uint32_t dacc = tmem + (uint32_t)(b * kBN);
            for (int kb = 0; kb < nk; ++kb, ++gs) {
                const int s = (int)(gs % kSpl);
                const uint32_t u = gs / kSpl;
                tc::mbar_wait(&full_bar[s], u & 1);
                tc::fence_after_sync();
                const uint32_t ahi = aS + s * kSplA, alo = ahi + kRawA;
                const uint32_t bhi = bS + s * kSplB, blo = bhi + kRawB;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint32_t ko = ks * 256;  // 2 K-adjacent core matrices (8 tf32) per UMMA
                    const uint32_t acc0 = (kb > 0 || ks > 0) ? 1u : 0u;
                    // small terms first
                    mma_tf32(dacc, tc::smem_desc(alo + ko, 128, kSBO), tc::smem_desc(bhi + ko, 128, kSBO), idesc, acc0);
                    mma_tf32(dacc, tc::smem_desc(ahi + ko, 128, kSBO), tc::smem_desc(blo + ko, 128, kSBO), idesc, 1u);
                    mma_tf32(dacc, tc::smem_desc(ahi + ko, 128, kSBO), tc::smem_desc(bhi + ko, 128, kSBO), idesc, 1u);
                }
                tc::commit_warp(&empty_bar[s]);
                if (kb == nk - 1) tc::commit_warp(&accf_bar[b]);
            }
        }
    } else {
        // ================= epilogue: warp w reads TMEM lanes 32 (w % 4) .. (A rows)
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        int tcount = 0;
        for (int t = blockIdx.x; t < nt; t += gridDim.x, ++tcount) {
            const TileInfo ti = get_tile(p, t);
            const int b = tcount & 1;
            const uint32_t ub = (uint32_t)tcount >> 1;
            tc::mbar_wait(&accf_bar[b], ub & 1);
            tc::fence_after_sync();
            const bool rok = r < ti.m;
            tc::mbar_wait(&normf_bar[b], ub & 1);
            float an = 0.0f;
            if constexpr (kEpi == TG_EPI_DIST) an = __fadd_rn(anorm[(b * 2) * kBM + r], anorm[(b * 2 + 1) * kBM + r]);
            if constexpr (kEpi != TG_EPI_DIST && kEpi != TG_EPI_ARGMIN) {
                // row-major C: 32 x 32 blocks transposed through shared memory so
                // that each store instruction writes 32 consecutive columns of a row
                float* stg = stage + (warp - kEpiWarp0) * kStg;
                for (int c0 = 0; c0 < ti.n; c0 += 32) {
                    uint32_t acc[32];
                    tc::tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * kBN + c0), acc);
#pragma unroll
                    for (int i = 0; i < 32; ++i) stg[lane * 33 + i] = __uint_as_float(acc[i]);
                    __syncwarp();
                    const int col = c0 + lane;
                    const bool cok = col < ti.n;
                    float bn = 0.0f;
                    if constexpr (kEpi == TG_EPI_PROBE) bn = cok ? p.b_norm[ti.b0 + col] : 0.0f;
                    const int rmax = min(32, ti.m - quarter * 32);
                    for (int rr = 0; rr < rmax; ++rr) {
                        const float v = stg[rr * 33 + lane];
                        if (cok) {
                            float* dst = p.C + ti.c0 + (int64_t)(quarter * 32 + rr) * ti.ldc + col;
                            if constexpr (kEpi == TG_EPI_PROBE) *dst = __fmaf_rn(-2.0f, v, bn);
                            else *dst = v;
                        }
                    }
                    __syncwarp();
                }
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&acce_bar[b]);
                continue;
            }
            if constexpr (kEpi == TG_EPI_ARGMIN) {
                // nearest B row of this A row within the tile: (orderable key << 32 | id)
                unsigned long long best = ~0ull;
                for (int c0 = 0; c0 < ti.n; c0 += 16) {
                    uint32_t acc[16];
                    tc::tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * kBN + c0), acc);
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int col = c0 + i;
                        if (col < ti.n) {
                            const float d = __fmaf_rn(-2.0f, __uint_as_float(acc[i]), __ldg(p.b_norm + ti.b0 + col));
                            const unsigned long long key =
                                ((unsigned long long)f2o(d) << 32) | (unsigned long long)(ti.b0 + col);
                            best = key < best ? key : best;
                        }
                    }
                }
                if (rok) atomicMin(p.amin + ti.a0 + r, best);
                tc::fence_before_sync();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&acce_bar[b]);
                continue;
            }
            for (int c0 = 0; c0 < ti.n; c0 += 16) {
                uint32_t acc[16];
                tc::tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * kBN + c0), acc);
                if (!rok) continue;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int col = c0 + i;
                    if (col >= ti.n) break;
                    const float v = __uint_as_float(acc[i]);
                    if constexpr (kEpi == TG_EPI_STORE) {
                        p.C[ti.c0 + (int64_t)r * ti.ldc + col] = v;
                    } else if constexpr (kEpi == TG_EPI_PROBE) {
                        p.C[ti.c0 + (int64_t)r * ti.ldc + col] = __fmaf_rn(-2.0f, v, p.b_norm[ti.b0 + col]);
                    } else {
                        // dense re-rank: column-major tile so that lanes (rows) store contiguously
                        const int64_t bi = p.b_idx ? (int64_t)p.b_idx[ti.b0 + col] : ti.b0 + col;
                        const float d = __fmaf_rn(-2.0f, v, __fadd_rn(an, p.b_norm[bi]));
                        p.C[ti.c0 + (int64_t)col * ti.ldc + r] = fmaxf(d, 0.0f);
                    }
                }
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&acce_bar[b]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == kMmaWarp) tc::tmem_dealloc(tmem, kTmemCols);
}

// ------------------------------------------------------------------------
// Dense re-rank block (1xTF32, TMA-fed): d~ = n_o^2 + ||q - c||^2 - 2 (x - c).(q - c)
// for every vector x of a list (A rows = slot-ordered residuals, 128-row tiles)
// and every query q sharing that nearest list (B rows, sorted residuals).
// Operands go straight from global memory into the UMMA layout by 2D TMA with
// 128-byte swizzle (32 floats of K per stage); tf32 reads the top 19 bits of
// each fp32, so |d~ - d| <= 2^-8 (n_o^2 + ||q - c||^2) (the re-rank's filter
// bound, search.cu).  Warp 0: TMA, warp 1: MMA, warps 2-5: epilogue.
constexpr int kDK = 32;                       // floats of K per stage (128 bytes)
constexpr int kDStages = 2;  // 96 KB: leaves an SM room for quantizer blocks alongside (side-stream overlap)
constexpr int kDA = kBM * kDK * 4;            // 16 KB
constexpr int kDBoxRows = 64;                 // B box rows (n <= 256: up to 4 boxes)
constexpr int kDB = kBN * kDK * 4;            // 32 KB (max)
constexpr int kDNT = 6 * 32;
constexpr size_t kDSmem = 1024 + (size_t)kDStages * (kDA + kDB);

__global__ __launch_bounds__(kDNT, 1) void tgemm_dist1_kernel(const __grid_constant__ CUtensorMap tmA,
                                                              const __grid_constant__ CUtensorMap tmB,
                                                              const TgParams p, const float* __restrict__ a_norm) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const uint32_t pad = (1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u;
    uint8_t* sA = smem_raw + pad;                 // [stages][128 rows][128 B] SW128
    uint8_t* sB = sA + kDStages * kDA;            // [stages][256 rows][128 B] SW128
    __shared__ __align__(8) uint64_t full_bar[kDStages], empty_bar[kDStages], accf_bar[2], acce_bar[2];
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 1) tc::tmem_alloc(&tmem_base_s, kTmemCols);
    if (tid == 0) {
        for (int s = 0; s < kDStages; ++s) {
            tc::mbar_init(&full_bar[s], 1);
            tc::mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&accf_bar[b], 1);
            tc::mbar_init(&acce_bar[b], 4);
        }
        tc::prefetch_tmap(&tmA);
        tc::prefetch_tmap(&tmB);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base_s;
    const int nt = p.ntiles;
    const int nk = (p.K + kDK - 1) / kDK;
    if (warp == 0) {
        if (lane == 0) {
            uint32_t gs = 0;
            for (int t = blockIdx.x; t < nt; t += gridDim.x) {
                const TgTile d = p.tiles[t];
                const int nbox = (d.n + kDBoxRows - 1) / kDBoxRows;
                for (int kb = 0; kb < nk; ++kb, ++gs) {
                    const int s = (int)(gs % kDStages);
                    const uint32_t u = gs / kDStages;
                    if (u > 0) tc::mbar_wait_backoff(&empty_bar[s], (u - 1) & 1);
                    tc::mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(kDA + nbox * kDBoxRows * kDK * 4));
                    tc::tma_load_2d(sA + s * kDA, &tmA, &full_bar[s], kb * kDK, (int)d.a0);
                    for (int bx = 0; bx < nbox; ++bx)
                        tc::tma_load_2d(sB + s * kDB + bx * kDBoxRows * kDK * 4, &tmB, &full_bar[s], kb * kDK,
                                        (int)(d.b0 + bx * kDBoxRows));
                }
            }
        }
    } else if (warp == 1) {
        uint32_t gs = 0;
        int tcount = 0;
        const uint64_t a0 = tc::smem_desc_sw128(tc::smem_u32(sA)), b0 = tc::smem_desc_sw128(tc::smem_u32(sB));
        for (int t = blockIdx.x; t < nt; t += gridDim.x, ++tcount) {
            const TgTile d = p.tiles[t];
            const int n16 = max(16, (d.n + 15) & ~15);
            const uint32_t idesc = idesc_tf32(kBM, n16);
            const int b = tcount & 1;
            const uint32_t ub = (uint32_t)tcount >> 1;
            if (ub > 0) tc::mbar_wait_backoff(&acce_bar[b], (ub - 1) & 1);
            tc::fence_after_sync();
            const uint32_t dacc = tmem + (uint32_t)(b * kBN);
            for (int kb = 0; kb < nk; ++kb, ++gs) {
                const int s = (int)(gs % kDStages);
                tc::mbar_wait(&full_bar[s], (gs / kDStages) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int ks = 0; ks < kDK / 8; ++ks)  // K = 8 tf32 (32 bytes) per UMMA
                    mma_tf32(dacc, a0 + (uint64_t)((s * kDA + ks * 32) >> 4), b0 + (uint64_t)((s * kDB + ks * 32) >> 4),
                             idesc, (kb > 0 || ks > 0) ? 1u : 0u);
                tc::commit_warp(&empty_bar[s]);
                if (kb == nk - 1) tc::commit_warp(&accf_bar[b]);
            }
        }
    } else {
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        int tcount = 0;
        for (int t = blockIdx.x; t < nt; t += gridDim.x, ++tcount) {
            const TgTile d = p.tiles[t];
            const int b = tcount & 1;
            const uint32_t ub = (uint32_t)tcount >> 1;
            const bool rok = r < d.m;
            const float an = rok ? a_norm[d.a0 + r] : 0.0f;
            tc::mbar_wait(&accf_bar[b], ub & 1);
            tc::fence_after_sync();
            for (int c0 = 0; c0 < d.n; c0 += 16) {
                uint32_t acc[16];
                tc::tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(b * kBN + c0), acc);
                if (!rok) continue;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const int col = c0 + i;
                    if (col >= d.n) break;
                    const float v = __uint_as_float(acc[i]);
                    const float dd = __fmaf_rn(-2.0f, v, __fmaf_rn(an, an, p.b_norm[d.b0 + col]));
                    p.C[d.c0 + (int64_t)col * d.ldc + r] = dd;
                }
            }
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&acce_bar[b]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace

static PFN_cuTensorMapEncodeTiled_v12000 tg_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        RQ_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        RQ_REQUIRE(f && q == cudaDriverEntryPointSuccess, RABITQ_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }
    return fn;
}

// fp32 [rows x K] row-major, stride ld floats; box = box_k floats x box_rows rows,
// zero fill out of bounds
static void make_tmap(CUtensorMap* m, const float* base, int64_t rows, int K, int64_t ld, int box_rows, int box_k = kBK,
                      CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE) {
    const cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    const cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
    const cuuint32_t box[2] = {(cuuint32_t)box_k, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult cr = tg_encode()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box,
                                    estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    RQ_REQUIRE(cr == CUDA_SUCCESS, RABITQ_ERR_CUDA, "tgemm: cuTensorMapEncodeTiled failed");
}

void tgemm_dist1(const TgParams& p, const float* a_norm, cudaStream_t st) {
    RQ_REQUIRE(p.tiles && p.a_idx == nullptr && p.b_idx == nullptr && p.K % 4 == 0, RABITQ_ERR_INTERNAL,
               "tgemm_dist1: plain tiled operands");
    if (p.ntiles <= 0) return;
    int dev = 0, sms = 148;
    RQ_CUDA(cudaGetDevice(&dev));
    RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CUtensorMap tmA, tmB;
    make_tmap(&tmA, p.A, p.M, p.K, p.lda, kBM, kDK, CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap(&tmB, p.B, p.N, p.K, p.ldb, kDBoxRows, kDK, CU_TENSOR_MAP_SWIZZLE_128B);
    RQ_CUDA(cudaFuncSetAttribute(tgemm_dist1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDSmem));
    tgemm_dist1_kernel<<<std::min(p.ntiles, sms), kDNT, kDSmem, st>>>(tmA, tmB, p, a_norm);
    RQ_CHECK_LAUNCH();
}

void tgemm(const TgParams& p, int epi, cudaStream_t st) {
    RQ_REQUIRE(p.K % 4 == 0 && p.lda % 4 == 0 && p.ldb % 4 == 0, RABITQ_ERR_INTERNAL, "tgemm: K and strides % 4");
    const int nt = p.tiles ? p.ntiles : (int)(((p.M + kBM - 1) / kBM) * ((p.N + kBN - 1) / kBN));
    if (nt <= 0) return;
    int dev = 0, sms = 148;
    RQ_CUDA(cudaGetDevice(&dev));
    RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int grid = std::min(nt, sms);
    // plain A and B rows: TMA (tile mode needs p.M / p.N = the row extents of A / B)
    const bool tma = p.a_idx == nullptr && p.b_idx == nullptr;
    CUtensorMap tmA, tmB;
    std::memset(&tmA, 0, sizeof(tmA));
    std::memset(&tmB, 0, sizeof(tmB));
    if (tma) {
        make_tmap(&tmA, p.A, p.M, p.K, p.lda, kBM);
        make_tmap(&tmB, p.B, p.N, p.K, p.ldb, kBN);
    }
#define RQ_TG(E, T)                                                                                                    \
    do {                                                                                                               \
        RQ_CUDA(cudaFuncSetAttribute(tgemm_kernel<E, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));  \
        tgemm_kernel<E, T><<<grid, kNT, kSmem, st>>>(tmA, tmB, p);                                                    \
    } while (0)
    if (epi == TG_EPI_STORE) {
        if (tma) RQ_TG(TG_EPI_STORE, true);
        else RQ_TG(TG_EPI_STORE, false);
    } else if (epi == TG_EPI_PROBE) {
        if (tma) RQ_TG(TG_EPI_PROBE, true);
        else RQ_TG(TG_EPI_PROBE, false);
    } else if (epi == TG_EPI_ARGMIN) {
        RQ_REQUIRE(p.tiles == nullptr && p.amin != nullptr, RABITQ_ERR_INTERNAL, "tgemm argmin: plain mode");
        if (tma) RQ_TG(TG_EPI_ARGMIN, true);
        else RQ_TG(TG_EPI_ARGMIN, false);
    } else {
        if (tma) RQ_TG(TG_EPI_DIST, true);
        else RQ_TG(TG_EPI_DIST, false);
    }
#undef RQ_TG
    RQ_CHECK_LAUNCH();
}

}  // namespace rabitq
