// common.cuh -- internal device/host primitives of librabitq (sm_100a).
//
// Product code.  Shares nothing with oracle/ (the test oracle).
// Paper: arxiv 2605.16007, cited as P:Lnnn; NS = BASELINE.json
// north_star; R#n = DESIGN.md readings.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "rabitq.h"

namespace rabitq {

// ----------------------------------------------------------------- errors --
struct Error : std::runtime_error {
    rabitq_status status;
    Error(rabitq_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define RQ_CUDA(call)                                                                         \
    do {                                                                                      \
        cudaError_t e_ = (call);                                                              \
        if (e_ != cudaSuccess) {                                                              \
            rabitq_status s_ = (e_ == cudaErrorMemoryAllocation) ? RABITQ_ERR_OUT_OF_MEMORY   \
                                                                 : RABITQ_ERR_CUDA;           \
            throw ::rabitq::Error(s_, std::string(#call) + ": " + cudaGetErrorString(e_) +    \
                                          " (" + __FILE__ + ":" + std::to_string(__LINE__) +  \
                                          ")");                                               \
        }                                                                                     \
    } while (0)

#define RQ_CHECK_LAUNCH() RQ_CUDA(cudaGetLastError())

#define RQ_REQUIRE(cond, status, msg)                      \
    do {                                                   \
        if (!(cond)) throw ::rabitq::Error((status), (msg)); \
    } while (0)

constexpr uint32_t kQuantTag = 0x51554E54u;             // 'QUNT' (R#12)
constexpr uint64_t kQuantSeedXor = 0x5241424954515155ull; // R#12
constexpr int kBlockVec = 32;                            // vectors per interleaved code block
constexpr uint32_t kPadRow = 0xFFFFFFFFu;

// ------------------------------------------------------------- Philox4x32 --
// Philox4x32-10 (Salmon et al., SC'11), the counter-based generator NS(2)
// names.  Written for the device (__umulhi) and the host (64-bit products).
struct U4 {
    uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ U4 philox4x32_10(uint32_t k0, uint32_t k1, U4 c) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        // one 32x32 -> 64-bit multiply each (IMAD.WIDE.U32 on the device)
        const uint64_t p0 = 0xD2511F53ull * c.x, p1 = 0xCD9E8D57ull * c.z;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// The same generator with the key schedule k_r = (k0 + r W0, k1 + r W1)
// precomputed on the host: passed as a kernel parameter, the round keys are
// constant-bank operands of the XORs (no per-call key bumps).
struct PhiloxSched {
    uint32_t k0[10], k1[10];
};
inline PhiloxSched philox_sched(uint32_t k0, uint32_t k1) {
    PhiloxSched s;
    for (int r = 0; r < 10; ++r) {
        s.k0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
        s.k1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
    }
    return s;
}
__device__ __forceinline__ U4 philox4x32_10(const PhiloxSched& s, U4 c) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = 0xD2511F53ull * c.x, p1 = 0xCD9E8D57ull * c.z;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c = U4{hi1 ^ c.y ^ s.k0[r], lo1, hi0 ^ c.w ^ s.k1[r], lo0};
    }
    return c;
}

// Diagnostic environment switches exist only in a -DRABITQ_DIAG build: the
// product library's paths and results never depend on the environment.
inline const char* rq_diag_env(const char* name) {
#ifdef RABITQ_DIAG
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

// --------------------------------------------------- order-preserving keys --
__host__ __device__ __forceinline__ uint32_t f2o(float f) {
#ifdef __CUDA_ARCH__
    uint32_t b = __float_as_uint(f);
#else
    uint32_t b;
    memcpy(&b, &f, 4);
#endif
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ float o2f(uint32_t o) {
    uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
#ifdef __CUDA_ARCH__
    return __uint_as_float(b);
#else
    float f;
    memcpy(&f, &b, 4);
    return f;
#endif
}
__host__ __device__ __forceinline__ uint64_t make_key(float v, uint32_t row) {
    return ((uint64_t)f2o(v) << 32) | row;
}

// ------------------------------------------------------------- estimator --
// Per-(query, list) constants of the estimator (NS(4), R#1):
//   <xbar, qbar> sqrt(D) = 2 Delta ip + 2 v_l pc - (Delta S_q + D v_l)
//   est = n_o^2 + ||r_q||^2 - (2 n_o / (rho_o sqrt(D))) <xbar, qbar> sqrt(D)
// Every kernel that evaluates est goes through pair_consts + rabitq_est, with
// explicit round-to-nearest intrinsics (no contraction choices left to the
// compiler), so the pruning threshold and the scan compare bit-identical
// values.
struct PairC {
    float a;    // 2 Delta
    float b;    // 2 v_l
    float K;    // Delta S_q + D v_l
    float nq2;  // ||r_q||^2
};

// qs = {v_l, Delta, ||r_q||^2, S_q}
__device__ __forceinline__ PairC pair_consts(float4 qs, int D) {
    PairC c;
    c.a = __fmul_rn(2.0f, qs.y);
    c.b = __fmul_rn(2.0f, qs.x);
    c.K = __fmaf_rn(qs.y, qs.w, __fmul_rn((float)D, qs.x));
    c.nq2 = qs.z;
    return c;
}

// fac = {A = n_o^2, f1 = 2 n_o / (rho_o sqrt(D))}
__device__ __forceinline__ float rabitq_est(int ip, int pc, float2 fac, const PairC& c) {
    const float t = __fmaf_rn(c.a, __int2float_rn(ip), __fmaf_rn(c.b, __int2float_rn(pc), -c.K));
    return __fmaf_rn(-fac.y, t, __fadd_rn(fac.x, c.nq2));
}

// ranking key: est, or the lower bound est - eps0 n_q g1 (R#15)
template <bool kLB>
__device__ __forceinline__ float rank_key(float est, float epsnq, float g1) {
    if constexpr (kLB) return __fsub_rn(est, __fmul_rn(epsnq, g1));
    else return est;
}

// ------------------------------------------------------- warp primitives --
// Blackwell packed FP32 (FADD2 / FFMA2 / FMUL2): two IEEE round-to-nearest
// operations per instruction, each lane of the pair rounded exactly as the
// scalar op would be
#define RQ_F2_OP(name, op)                                                                                 \
    __device__ __forceinline__ float2 name(float2 a, float2 b) {                                           \
        float2 d;                                                                                          \
        asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t" op    \
            " rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"                                                    \
            : "=f"(d.x), "=f"(d.y)                                                                         \
            : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));                                                     \
        return d;                                                                                          \
    }
RQ_F2_OP(fadd2, "add.rn.f32x2")
RQ_F2_OP(fsub2, "sub.rn.f32x2")
RQ_F2_OP(fmul2, "mul.rn.f32x2")
RQ_F2_OP(fadd2_rm, "add.rm.f32x2")  // round toward -inf
#undef RQ_F2_OP
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// ----------------------------------------------- block radix select (k-th) --
// k-th smallest (1-based) of n keys produced by get(i), by most-significant-
// digit radix select with 8-bit digits (one histogram pass per digit,
// early exit once the digit prefix is unique).  All NT threads must call.
// Scratch: hist[256] + 4 words in shared memory.
// The digits above the highest bit in which min and max differ are common to
// all keys: one min/max pass skips them (and their single-bin histograms).
template <int NT, typename KeyT, typename Get>
__device__ KeyT block_select_kth(Get get, int n, int k, uint32_t* hist, uint32_t* sc) {
    constexpr int kBits = sizeof(KeyT) * 8;
    static_assert(NT % 32 == 0 && NT / 32 <= 64, "block size");
    KeyT prefix = 0, mask = 0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int shift0 = kBits - 8;
    {
        KeyT mn = ~(KeyT)0, mx = 0;
        for (int i = tid; i < n; i += NT) {
            const KeyT key = get(i);
            mn = key < mn ? key : mn;
            mx = key > mx ? key : mx;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const KeyT a = __shfl_xor_sync(0xFFFFFFFFu, mn, o), b = __shfl_xor_sync(0xFFFFFFFFu, mx, o);
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
        }
        KeyT* wr = reinterpret_cast<KeyT*>(hist);  // [2][NT / 32] (hist is free here)
        __syncthreads();
        if (lane == 0) {
            wr[warp] = mn;
            wr[NT / 32 + warp] = mx;
        }
        __syncthreads();
        for (int w = 0; w < NT / 32; ++w) {
            const KeyT a = wr[w], b = wr[NT / 32 + w];
            mn = a < mn ? a : mn;
            mx = b > mx ? b : mx;
        }
        __syncthreads();
        const KeyT diff = mn ^ mx;
        if (diff == 0) return mn;  // every key equal (n >= 1)
        int hb;
        if constexpr (sizeof(KeyT) == 8) hb = 63 - __clzll((long long)diff);
        else hb = 31 - __clz((int)diff);
        shift0 = (hb / 8) * 8;
        if (shift0 + 8 < kBits) {
            mask = ~(KeyT)0 << (shift0 + 8);
            prefix = mn & mask;
        }
    }
    for (int shift = shift0; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += NT) hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += NT) {
            const KeyT key = get(i);
            if ((key & mask) == prefix) atomicAdd(&hist[(uint32_t)(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            // lane l owns bins [8l, 8l+8)
            uint32_t loc[8];
            uint32_t s = 0;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                loc[b] = hist[tid * 8 + b];
                s += loc[b];
            }
            uint32_t incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (tid >= o) incl += t;
            }
            const uint32_t excl = incl - s;
            if (excl < (uint32_t)k && (uint32_t)k <= incl) {
                uint32_t run = excl;
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    if (run < (uint32_t)k && (uint32_t)k <= run + loc[b]) {
                        sc[0] = tid * 8 + b;
                        sc[1] = k - run;
                        sc[2] = loc[b];
                    }
                    run += loc[b];
                }
            }
        }
        __syncthreads();
        const uint32_t digit = sc[0];
        k = (int)sc[1];
        const uint32_t cnt = sc[2];
        prefix |= (KeyT)digit << shift;
        mask |= (KeyT)255u << shift;
        __syncthreads();
        if (cnt == 1 && shift > 0) {
            // the prefix identifies exactly one key: fetch it
            for (int i = tid; i < n; i += NT) {
                const KeyT key = get(i);
                if ((key & mask) == prefix) {
                    if constexpr (sizeof(KeyT) == 8) {
                        sc[0] = (uint32_t)key;
                        sc[1] = (uint32_t)(key >> 32);
                    } else {
                        sc[0] = (uint32_t)key;
                    }
                }
            }
            __syncthreads();
            KeyT r;
            if constexpr (sizeof(KeyT) == 8) r = ((KeyT)sc[1] << 32) | sc[0];
            else r = (KeyT)sc[0];
            __syncthreads();
            return r;
        }
    }
    return prefix;
}

// In-place ascending bitonic sort of n (power of two) keys in shared memory.
template <int NT, typename KeyT>
__device__ void block_bitonic_sort(KeyT* a, int n) {
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            __syncthreads();
            for (int t = threadIdx.x; t < (n >> 1); t += NT) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                KeyT x = a[lo], y = a[hi];
                if ((x > y) == up) {
                    a[lo] = y;
                    a[hi] = x;
                }
            }
        }
    }
    __syncthreads();
}

__host__ __device__ __forceinline__ int next_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// ---------------------------------------------------------- SGEMM (gemm.cu)
// C[M x N] = A[M x K] * B, B = [K x N] (kBT = false) or [N x K] (kBT = true),
// all row-major fp32.  epi 0: C = acc; epi 1: C = cn[col] - 2 acc (the
// decomposed squared distance minus the row norm).
void sgemm(int M, int N, int K, const float* A, int lda, const float* B, int ldb, bool b_trans,
           float* C, int ldc, int epi, const float* cn, cudaStream_t st);

// -------------------------------------------------------------- haar.cpp
// Haar-random orthogonal P [D x D] (row-major fp32), R#5.
void haar_rotation_host(int D, uint64_t seed, float* P);

}  // namespace rabitq
