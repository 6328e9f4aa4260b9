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
// Work item = (list, 128-vector tile, 128-query group); persistent CTAs
// stride over the items.  Per item the K loop runs in 128-byte chunks through
// two shared-memory stages: 256 threads expand codes (A) and cp.async the
// query rows (B) into the canonical K-major no-swizzle layout while the
// previous chunk's 4 UMMAs run; tcgen05.commit -> mbarrier frees a stage.
// 3 CTAs per SM (64 KB of stages each) overlap one CTA's epilogue with
// another's MMAs.
//
// This ignores query boundaries for scheduling and re-opens the
// list grouping the paper rejected for its NPU pipeline: on B200 it
// turns the bandwidth-bound scan into tensor-core work.
#include <cub/cub.cuh>

#include <algorithm>

#include "search.cuh"
#include "tc.cuh"

namespace rabitq {
namespace {

constexpr int kTM = 128;     // vectors per tile (UMMA M)
constexpr int kTN = 128;     // queries per group (UMMA N)
constexpr int kKC = 128;     // bytes of K per stage
constexpr int kNT = 256;     // threads per CTA
constexpr int kStageA = kTM * kKC;  // 16 KB
constexpr int kStageB = kTN * kKC;  // 16 KB
constexpr int kSBO = (kKC / 16) * 128;  // byte distance between 8-row core-matrix groups
constexpr int kCTAsPerSM = 3;

struct ColC {
    PairC c;        // 16 B
    float tau;      // threshold of the column's query
    float epsnq;    // eps0 * n_q (lower-bound key)
    int q;          // query (-1: empty column)
    int pair;       // (query, probe) pair index
};

// 16 code bits -> 16 bytes of 0/1 (x * 0x00204081 spreads 4 bits to 4 bytes)
__device__ __forceinline__ uint4 expand16(uint32_t b) {
    uint4 r;
    r.x = ((b & 0xFu) * 0x00204081u) & 0x01010101u;
    r.y = (((b >> 4) & 0xFu) * 0x00204081u) & 0x01010101u;
    r.z = (((b >> 8) & 0xFu) * 0x00204081u) & 0x01010101u;
    r.w = (((b >> 12) & 0xFu) * 0x00204081u) & 0x01010101u;
    return r;
}

template <bool kLB, bool kDump>
__global__ __launch_bounds__(kNT, kCTAsPerSM) void scan_imma_kernel(ScanArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* stA = smem;                       // [2][kStageA]
    uint8_t* stB = smem + 2 * kStageA;         // [2][kStageB]
    ColC* colc = reinterpret_cast<ColC*>(smem + 2 * kStageA + 2 * kStageB);  // [kTN]
    __shared__ __align__(8) uint64_t mbar[2];
    __shared__ uint32_t tmem_base_s;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) tc::tmem_alloc(&tmem_base_s, kTN);
    if (tid == 0) {
        tc::mbar_init(&mbar[0], 1);
        tc::mbar_init(&mbar[1], 1);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base_s;
    uint32_t phase[2] = {0u, 0u};
    bool pending[2] = {false, false};

    const int64_t total = a.list_items[a.nlist];
    const int nchunks = (a.Dp + kKC - 1) / kKC;
    for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
        // ---- locate (list, tile, group) ----
        int64_t lo = 0, hi = a.nlist;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (a.list_items[mid] <= item) lo = mid;
            else hi = mid;
        }
        const int j = (int)lo;
        const int64_t L = a.list_off[j + 1] - a.list_off[j];
        const int64_t G = a.gstart[j + 1] - a.gstart[j];
        const int64_t ng = (G + kTN - 1) / kTN;
        const int64_t local = item - a.list_items[j];
        const int64_t tv = local / ng, g = local % ng;
        const int64_t slot0 = a.slot_off[j] + tv * kTM;
        const int64_t grow0 = a.gstart[j] + g * kTN;
        const int64_t rem = G - g * kTN;
        const int ncols = (int)(rem < kTN ? rem : kTN);
        const int ncols16 = (ncols + 15) & ~15;  // UMMA N (M = 128 needs N % 16 == 0): no MMA work on empty columns
        const uint32_t idesc = tc::idesc_i8(kTM, ncols16);

        // ---- per-column constants (one query per column) ----
        if (tid < kTN) {
            ColC cc;
            if (tid < ncols) {
                const int p = a.gpair[grow0 + tid];
                const int q = p / a.nprobe;
                cc.c = pair_consts(a.qscal[p], a.D);
                cc.tau = a.tau[q];
                cc.epsnq = __fmul_rn(a.eps0, sqrtf(cc.c.nq2));
                cc.q = q;
                cc.pair = p;
            } else {
                cc.c = PairC{0.f, 0.f, 0.f, 0.f};
                cc.tau = -INFINITY;
                cc.epsnq = 0.f;
                cc.q = -1;
                cc.pair = -1;
            }
            colc[tid] = cc;
        }

        // ---- K loop: produce stage, issue 4 UMMAs, commit ----
        for (int c = 0; c < nchunks; ++c) {
            const int s = c & 1;
            if (pending[s]) {
                tc::mbar_wait(&mbar[s], phase[s]);
                phase[s] ^= 1u;
                pending[s] = false;
            }
            uint8_t* A = stA + s * kStageA;
            uint8_t* B = stB + s * kStageB;
            const int kbytes = min(kKC, a.Dp - c * kKC);  // multiple of 32
            // A: thread -> (row r, 2 code words) -> 4 core-matrix rows of 16 bytes
            {
                const int r = tid & (kTM - 1), wp = tid >> 7;
                const int64_t slot = slot0 + r;
                const uint32_t* cbase = a.codes + ((size_t)(slot >> 5) * a.W) * 32 + (slot & 31);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int wl = wp * 2 + h;          // word within the chunk
                    if (wl * 32 >= kbytes) break;
                    const int w = c * (kKC / 32) + wl;  // < W since kbytes covers it
                    const uint32_t x = __ldg(cbase + (size_t)w * 32);
                    uint8_t* dst = A + (r >> 3) * kSBO + (r & 7) * 16 + (wl * 2) * 128;
                    *reinterpret_cast<uint4*>(dst) = expand16(x & 0xFFFFu);
                    *reinterpret_cast<uint4*>(dst + 128) = expand16(x >> 16);
                }
            }
            // B: the group's query rows (ncols rounded up to 16) x kbytes, 16-byte units by cp.async
            {
                const int units = ncols16 * (kbytes / 16);
                const int per_row = kbytes / 16;
                for (int u = tid; u < units; u += kNT) {
                    const int rr = u / per_row, k16 = u % per_row;
                    const uint8_t* src = a.qbar8 + (size_t)(grow0 + rr) * a.Dp + c * kKC + k16 * 16;
                    uint8_t* dst = B + (rr >> 3) * kSBO + (rr & 7) * 16 + k16 * 128;
                    tc::cp_async16(dst, src);
                }
            }
            tc::cp_async_wait_all();
            tc::fence_proxy_async();
            __syncthreads();
            if (tid == 0) {
                tc::fence_after_sync();
                const uint32_t aaddr = tc::smem_u32(A), baddr = tc::smem_u32(B);
                for (int ks = 0; ks < kbytes / 32; ++ks) {
                    const uint64_t ad = tc::smem_desc(aaddr + ks * 256, 128, kSBO);
                    const uint64_t bd = tc::smem_desc(baddr + ks * 256, 128, kSBO);
                    tc::mma_i8(tmem, ad, bd, idesc, (c > 0 || ks > 0) ? 1u : 0u);
                }
                tc::commit(&mbar[s]);
            }
            pending[s] = true;
        }
        // all UMMAs of this item done <=> the last commit arrived
        {
            const int s = (nchunks - 1) & 1;
            tc::mbar_wait(&mbar[s], phase[s]);
            phase[s] ^= 1u;
            pending[s] = false;
        }
        tc::fence_after_sync();

        // ---- epilogue: S from TMEM -> estimator -> threshold -> append ----
        {
            const int r = (warp & 3) * 32 + lane;  // TMEM lane = tile row = vector
            const int64_t v = tv * kTM + r;
            const bool vok = v < L;
            const int64_t slot = slot0 + r;
            const float2 fac = vok ? a.fac[slot] : make_float2(0.f, 0.f);
            const int pc = vok ? (int)a.pcnt[slot] : 0;
            const float g1 = (kLB && vok) ? a.g1[slot] : 0.f;
            const int colbase = (warp >> 2) * 64;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int col0 = colbase + h * 32;
                if (col0 >= ncols) break;  // warp-uniform
                uint32_t acc[32];
                tc::tmem_ld32(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)col0, acc);
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int cidx = col0 + i;
                    if (cidx >= ncols) break;  // warp-uniform
                    const ColC& cc = colc[cidx];
                    const int ip = (int)acc[i];
                    const float est = rabitq_est(ip, pc, fac, cc.c);
                    const float key = rank_key<kLB>(est, cc.epsnq, g1);
                    if constexpr (kDump) {
                        if (vok) {
                            const int64_t di = (a.item_off[cc.pair] + (v >> 5)) * 32 + (v & 31);
                            if (di < a.dump_cap) {
                                a.dump_ip[di] = ip;
                                a.dump_est[di] = est;
                            }
                        }
                    }
                    const bool surv = vok && key <= cc.tau;
                    const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, surv);
                    if (ballot) {
                        int base = 0;
                        if (lane == 0) base = atomicAdd(&a.cnt[cc.q], __popc(ballot));
                        base = __shfl_sync(0xFFFFFFFFu, base, 0);
                        if (surv) {
                            const int pos = base + __popc(ballot & ((1u << lane) - 1u));
                            if (pos < a.cap) a.buf[(size_t)cc.q * a.cap + pos] = make_key(key, a.rows[slot]);
                        }
                    }
                }
            }
        }
        tc::fence_before_sync();
        __syncthreads();  // TMEM accumulator and colc are free for the next item
    }
    // drain: a stage may still have an outstanding commit
    for (int s = 0; s < 2; ++s)
        if (pending[s]) tc::mbar_wait(&mbar[s], phase[s]);
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, kTN);
}

// ------------------------------------------------------------ list grouping
__global__ void group_count_kernel(const int32_t* __restrict__ probes, int64_t npairs, int64_t* __restrict__ gcount) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs; p += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)&gcount[probes[p]], 1ull);
}

__global__ void group_fill_kernel(const int32_t* __restrict__ probes, int64_t npairs,
                                  const int64_t* __restrict__ gstart, int32_t* __restrict__ gfill,
                                  int32_t* __restrict__ gpos, int32_t* __restrict__ gpair) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs; p += (int64_t)gridDim.x * blockDim.x) {
        const int j = probes[p];
        const int64_t pos = gstart[j] + atomicAdd(&gfill[j], 1);
        gpos[p] = (int32_t)pos;
        gpair[pos] = (int32_t)p;
    }
}

__global__ void list_items_kernel(int nlist, const int64_t* __restrict__ list_off, const int64_t* __restrict__ gcount,
                                  int64_t* __restrict__ items) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= nlist; j += gridDim.x * blockDim.x) {
        if (j == nlist) {
            items[j] = 0;
            continue;
        }
        const int64_t L = list_off[j + 1] - list_off[j];
        const int64_t G = gcount[j];
        items[j] = ((L + kTM - 1) / kTM) * ((G + kTN - 1) / kTN);
    }
}

}  // namespace

bool imma_wanted(const rabitq_index* idx, int64_t npairs, int scan_path) {
    if (scan_path == RABITQ_SCAN_POPC) return false;
    if (scan_path == RABITQ_SCAN_IMMA) return true;
    // AUTO: the tensor-core path pays once lists are shared by enough queries
    return npairs >= (int64_t)8 * idx->nlist;
}

void prepare_groups(const rabitq_index* idx, const int32_t* probes, int64_t npairs, Groups& g, cudaStream_t st,
                    int& launches) {
    const int nlist = idx->nlist;
    g.Dp = ((idx->D + 31) / 32) * 32;
    g.gcount.alloc((size_t)nlist + 1, st);
    g.gstart.alloc((size_t)nlist + 1, st);
    g.itemc.alloc((size_t)nlist + 1, st);
    g.list_items.alloc((size_t)nlist + 1, st);
    g.gfill.alloc((size_t)nlist, st);
    g.gpos.alloc((size_t)npairs, st);
    g.gpair.alloc((size_t)npairs + kTN, st);
    g.qbar8.alloc(((size_t)npairs + kTN) * g.Dp, st);
    RQ_CUDA(cudaMemsetAsync(g.gcount.p, 0, ((size_t)nlist + 1) * sizeof(int64_t), st));
    RQ_CUDA(cudaMemsetAsync(g.gfill.p, 0, (size_t)nlist * sizeof(int32_t), st));
    RQ_CUDA(cudaMemsetAsync(g.gpair.p + npairs, 0, kTN * sizeof(int32_t), st));
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((npairs + 255) / 256, 2048));
    group_count_kernel<<<grid, 256, 0, st>>>(probes, npairs, g.gcount.p);
    RQ_CHECK_LAUNCH();
    size_t tb = 0;
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, g.gcount.p, g.gstart.p, nlist + 1, st));
    size_t tb2 = 0;
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, g.itemc.p, g.list_items.p, nlist + 1, st));
    WBuf<uint8_t> tmp;
    tmp.alloc(std::max(tb, tb2), st);
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, g.gcount.p, g.gstart.p, nlist + 1, st));
    group_fill_kernel<<<grid, 256, 0, st>>>(probes, npairs, g.gstart.p, g.gfill.p, g.gpos.p, g.gpair.p);
    RQ_CHECK_LAUNCH();
    list_items_kernel<<<(nlist + 256) / 256, 256, 0, st>>>(nlist, idx->list_off, g.gcount.p, g.itemc.p);
    RQ_CHECK_LAUNCH();
    RQ_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb2, g.itemc.p, g.list_items.p, nlist + 1, st));
    launches += 7;
}

void scan_imma(const ScanArgs& a, bool lb, bool dump, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = 2 * (size_t)kStageA + 2 * (size_t)kStageB + kTN * sizeof(ColC);
    const int grid = sms * kCTAsPerSM;
#define RQ_IMMA(LB, DP)                                                                              \
    do {                                                                                             \
        RQ_CUDA(cudaFuncSetAttribute(scan_imma_kernel<LB, DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)smem));                                                    \
        scan_imma_kernel<LB, DP><<<grid, kNT, smem, st>>>(a);                                        \
    } while (0)
    if (dump) {
        if (lb) RQ_IMMA(true, true);
        else RQ_IMMA(false, true);
    } else {
        if (lb) RQ_IMMA(true, false);
        else RQ_IMMA(false, false);
    }
#undef RQ_IMMA
    RQ_CHECK_LAUNCH();
}

}  // namespace rabitq
