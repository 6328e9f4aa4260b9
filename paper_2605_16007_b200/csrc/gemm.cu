// gemm.cu -- fp32 SIMT GEMM used for the query rotation (S1) and the
// decomposed query-to-centroid distance ||c||^2 - 2 q.c (S2) and
// the build-side k-means assignment.  128x128x8 CTA tile, 256 threads, 8x8
// register micro-tile split in two 4-wide halves (conflict-free LDS.128),
// shared-memory double buffering.
//
// fp32 on purpose: probing decides which lists are scanned; tf32 tensor
// cores would reorder near-tied centroids.
#include "common.cuh"

namespace rabitq {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, NT = 256;

template <bool kBT, int kEpi>
__global__ __launch_bounds__(NT) void sgemm_kernel(int M, int N, int K, const float* __restrict__ A,
                                                   int lda, const float* __restrict__ B, int ldb,
                                                   float* __restrict__ C, int ldc,
                                                   const float* __restrict__ cn) {
    __shared__ __align__(16) float As[2][BK][BM];
    __shared__ __align__(16) float Bs[2][BK][BN];
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;

    // global->smem load mapping: A tile 128 x 8: row = tid >> 1, k = (tid & 1) * 4 .. +3
    const int a_r = tid >> 1, a_k = (tid & 1) * 4;
    // B tile: NN: k = tid >> 5, n = (tid & 31) * 4 .. +3;  NT: like A
    float ra[4], rb[4];

    auto load_tiles = [&](int k0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int gm = m0 + a_r, gk = k0 + a_k + i;
            ra[i] = (gm < M && gk < K) ? __ldg(A + (size_t)gm * lda + gk) : 0.0f;
        }
        if constexpr (kBT) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gn = n0 + a_r, gk = k0 + a_k + i;
                rb[i] = (gn < N && gk < K) ? __ldg(B + (size_t)gn * ldb + gk) : 0.0f;
            }
        } else {
            const int bk = tid >> 5, bn = (tid & 31) * 4;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int gn = n0 + bn + i, gk = k0 + bk;
                rb[i] = (gn < N && gk < K) ? __ldg(B + (size_t)gk * ldb + gn) : 0.0f;
            }
        }
    };
    auto store_tiles = [&](int buf) {
#pragma unroll
        for (int i = 0; i < 4; ++i) As[buf][a_k + i][a_r] = ra[i];
        if constexpr (kBT) {
#pragma unroll
            for (int i = 0; i < 4; ++i) Bs[buf][a_k + i][a_r] = rb[i];
        } else {
            const int bk = tid >> 5, bn = (tid & 31) * 4;
            *reinterpret_cast<float4*>(&Bs[buf][bk][bn]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
        }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

    load_tiles(0);
    store_tiles(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += BK) {
        const bool more = (k0 + BK) < K;
        if (more) load_tiles(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[8], b[8];
            const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
            const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
            const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
            a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
            a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
            b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
            b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (more) {
            store_tiles(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int gm = m0 + ((i < 4) ? (ty * 4 + i) : (64 + ty * 4 + i - 4));
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int gn = n0 + ((j < 4) ? (tx * 4 + j) : (64 + tx * 4 + j - 4));
            if (gn >= N) continue;
            float v = acc[i][j];
            if constexpr (kEpi == 1) v = __ldg(cn + gn) - 2.0f * v;
            C[(size_t)gm * ldc + gn] = v;
        }
    }
}

}  // namespace

void sgemm(int M, int N, int K, const float* A, int lda, const float* B, int ldb, bool b_trans, float* C,
           int ldc, int epi, const float* cn, cudaStream_t st) {
    if (M <= 0 || N <= 0) return;
    // grid.y is limited to 65535 row tiles: taller products run as row slabs
    constexpr int kSlab = 65535 * BM;
    if (M > kSlab) {
        for (int r0 = 0; r0 < M; r0 += kSlab)
            sgemm(std::min(kSlab, M - r0), N, K, A + (size_t)r0 * lda, lda, B, ldb, b_trans, C + (size_t)r0 * ldc,
                  ldc, epi, cn, st);
        return;
    }
    dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM);
    if (b_trans) {
        if (epi == 1) sgemm_kernel<true, 1><<<grid, NT, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, cn);
        else sgemm_kernel<true, 0><<<grid, NT, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, cn);
    } else {
        if (epi == 1) sgemm_kernel<false, 1><<<grid, NT, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, cn);
        else sgemm_kernel<false, 0><<<grid, NT, 0, st>>>(M, N, K, A, lda, B, ldb, C, ldc, cn);
    }
    RQ_CHECK_LAUNCH();
}

}  // namespace rabitq
