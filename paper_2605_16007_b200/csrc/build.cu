// build.cu -- index construction on the GPU (untimed; P:L156-159, P:L301-307,
// P:L197-209).  Everything runs in the rotated space (x' = P^T x): rotation
// preserves L2 distances, so k-means on x' gives c' = P^T c
// directly and the residual r_o = x' - c' needs no second rotation.
//
//   1. P: host Haar generation (haar.cpp) or caller-provided.
//   2. training rows: stratified seeded sample of min(n, 256 nlist) rows.
//   3. k-means (Lloyd, fp32): GEMM distance ||c'||^2 - 2 t'.c' + argmin,
//      atomic centroid sums, empty clusters re-seeded from the farthest
//      training points (R#6).
//   4. assign + encode every vector in chunks: rotate (GEMM), nearest
//      centroid, sign bits of r_o (R#7), n_o = ||r_o||, rho_o = ||r_o||_1 /
//      (sqrt(D) n_o) (R#9).
//   5. stable radix sort by list (ids ascending within a list) and scatter
//      into the 32-slot word-interleaved layout (index.cuh).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "index.cuh"
#include "search.cuh"
#include "tgemm.cuh"

namespace rabitq {
namespace {

__global__ void gather_rows_kernel(const float* __restrict__ X, int D, const int64_t* __restrict__ rows,
                                   int64_t m, float* __restrict__ out) {
    const int64_t total = m * D;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / D, d = e % D;
        out[e] = X[(size_t)rows[i] * D + d];
    }
}

// slot-ordered copy of the fp32 vectors, centred on their list's centroid in
// the original space (x - c_j; pad slots zero): a list's rows are contiguous
// for TMA, and the dense re-rank's GEMM form ||q-c||^2 + ||x-c||^2 - 2 (q-c).(x-c)
// works on residuals instead of raw vectors (no cancellation of large norms)
__global__ void slot_rows_kernel(const float* __restrict__ X, int D, const uint32_t* __restrict__ rows,
                                 const int64_t* __restrict__ slot_off, const float* __restrict__ Corig, int nlist,
                                 float* __restrict__ Xs) {
    const int per = D / 4;
    for (int j = blockIdx.x; j < nlist; j += gridDim.x) {
        const int64_t s0 = slot_off[j], s1 = slot_off[j + 1];
        const float4* c = reinterpret_cast<const float4*>(Corig + (size_t)j * D);
        for (int64_t e = threadIdx.x; e < (s1 - s0) * per; e += blockDim.x) {
            const int64_t s = s0 + e / per;
            const int k = (int)(e % per);
            const uint32_t r = rows[s];
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (r != kPadRow) {
                const float4 x = reinterpret_cast<const float4*>(X + (size_t)r * D)[k];
                const float4 cc = c[k];
                v = make_float4(__fsub_rn(x.x, cc.x), __fsub_rn(x.y, cc.y), __fsub_rn(x.z, cc.z), __fsub_rn(x.w, cc.w));
            }
            reinterpret_cast<float4*>(Xs + (size_t)s * D)[k] = v;
        }
    }
}

// max n_o^2 per list (the grouped scan's fast-test rounding margin)
__global__ void list_amax_kernel(const float2* __restrict__ fac, const int64_t* __restrict__ slot_off,
                                 const int64_t* __restrict__ list_off, int nlist, float* __restrict__ amax) {
    __shared__ float red[8];
    for (int j = blockIdx.x; j < nlist; j += gridDim.x) {
        const int64_t s0 = slot_off[j], L = list_off[j + 1] - list_off[j];
        float m = 0.0f;
        for (int64_t v = threadIdx.x; v < L; v += blockDim.x) m = fmaxf(m, fac[s0 + v].x);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
        __syncthreads();
        if (threadIdx.x == 0) {
            float r = 0.0f;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmaxf(r, red[w]);
            amax[j] = r;
        }
        __syncthreads();
    }
}

// Pt = P^T (the rotation's B operand for the tensor-core GEMM: rows of P^T are K-contiguous)
__global__ void transpose_kernel(const float* __restrict__ P, int D, float* __restrict__ Pt) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)D * D; e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e / D), j = (int)(e % D);
        Pt[(int64_t)j * D + i] = P[e];
    }
}

__global__ void finite_kernel(const float* __restrict__ X, int64_t count, int* flag) {
    bool bad = false;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count;
         e += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(X[e]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void row_norm2_kernel(const float* __restrict__ C, int rows, int D, float* __restrict__ out) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= rows) return;
    float s = 0.0f;
    for (int i = lane; i < D; i += 32) {
        const float v = C[(size_t)warp * D + i];
        s = fmaf(v, v, s);
    }
    s = warp_sumf(s);
    if (lane == 0) out[warp] = s;
}

// nearest centroid per row of a [m x nlist] distance block, ties -> lowest id
__global__ void argmin_kernel(const float* __restrict__ dist, int64_t m, int nlist, int32_t* __restrict__ assign,
                              float* __restrict__ best, int32_t* __restrict__ prev,
                              unsigned long long* __restrict__ changed) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= m) return;
    const float* d = dist + (size_t)row * nlist;
    float bv = INFINITY;
    int bi = 0x7FFFFFFF;
    for (int j = lane; j < nlist; j += 32) {
        const float v = d[j];
        if (v < bv) { bv = v; bi = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xFFFFFFFFu, bv, o);
        const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
        if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) {
        if (bi == 0x7FFFFFFF) bi = 0;  // all-NaN row cannot happen (inputs checked finite)
        assign[row] = bi;
        if (best) best[row] = bv;
        if (prev) {
            if (prev[row] != bi) atomicAdd(changed, 1ull);
            prev[row] = bi;
        }
    }
}

// the same outputs from the tensor-core GEMM's fused argmin (tgemm TG_EPI_ARGMIN):
// key = orderable(||c||^2 - 2 x.c) << 32 | centroid
__global__ void argmin_keys_kernel(const unsigned long long* __restrict__ keys, int64_t m,
                                   int32_t* __restrict__ assign, float* __restrict__ best,
                                   int32_t* __restrict__ prev, unsigned long long* __restrict__ changed) {
    for (int64_t row = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; row < m; row += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long k = keys[row];
        const int bi = (int)(uint32_t)k;
        assign[row] = bi;
        if (best) best[row] = o2f((uint32_t)(k >> 32));
        if (prev) {
            if (prev[row] != bi) atomicAdd(changed, 1ull);
            prev[row] = bi;
        }
    }
}

__global__ void kmeans_accum_kernel(const float* __restrict__ T, int64_t m, int D, const int32_t* __restrict__ a,
                                    float* __restrict__ sums, int* __restrict__ counts) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= m) return;
    const int j = a[row];
    for (int i = lane; i < D; i += 32) atomicAdd(&sums[(size_t)j * D + i], T[(size_t)row * D + i]);
    if (lane == 0) atomicAdd(&counts[j], 1);
}

__global__ void kmeans_divide_kernel(float* __restrict__ C, const float* __restrict__ sums,
                                     const int* __restrict__ counts, int nlist, int D) {
    const int64_t total = (int64_t)nlist * D;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / D);
        if (counts[j] > 0) C[e] = sums[e] / (float)counts[j];
    }
}

// warp per vector: r_o = x' - c'_a, bits = [r >= 0] (R#7), n_o, rho (R#9)
__global__ void encode_kernel(const float* __restrict__ Xr, int64_t m, int D, int W, const float* __restrict__ Cr,
                              const int32_t* __restrict__ assign, uint32_t* __restrict__ codes,
                              float* __restrict__ n_o, float* __restrict__ rho) {
    const int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (v >= m) return;
    const float* x = Xr + (size_t)v * D;
    const float* c = Cr + (size_t)assign[v] * D;
    double s2 = 0.0, s1 = 0.0;
    for (int w = 0; w < W; ++w) {
        const int i = w * 32 + lane;
        float r = 0.0f;
        bool bit = false;
        if (i < D) {
            r = __fsub_rn(x[i], c[i]);
            bit = (r >= 0.0f);
            s2 += (double)r * (double)r;
            s1 += fabs((double)r);
        }
        const uint32_t word = __ballot_sync(0xFFFFFFFFu, bit);
        if (lane == 0) codes[(size_t)v * W + w] = word;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s2 += __shfl_xor_sync(0xFFFFFFFFu, s2, o);
        s1 += __shfl_xor_sync(0xFFFFFFFFu, s1, o);
    }
    if (lane == 0) {
        const double no = sqrt(s2);
        n_o[v] = (float)no;
        rho[v] = (no > 0.0) ? (float)(s1 / (sqrt((double)D) * no)) : 1.0f;
    }
}

// sorted position p -> slot; writes codes (interleaved), factors, rows
__global__ void scatter_kernel(int64_t n, int D, int W, const int32_t* __restrict__ skeys,
                               const uint32_t* __restrict__ srows, const int64_t* __restrict__ list_off,
                               const int64_t* __restrict__ slot_off, const uint32_t* __restrict__ codes_id,
                               const float* __restrict__ no_id, const float* __restrict__ rho_id,
                               uint32_t* __restrict__ codes, float2* __restrict__ fac, float* __restrict__ g1,
                               float* __restrict__ n_o, float* __restrict__ rho, uint32_t* __restrict__ rows,
                               uint32_t* __restrict__ slot_of_row, uint16_t* __restrict__ pcnt) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int j = skeys[p];
        const uint32_t row = srows[p];
        const int64_t slot = slot_off[j] + (p - list_off[j]);
        const int64_t blk = slot >> 5;
        const int lane = (int)(slot & 31);
        int pc = 0;
        for (int w = 0; w < W; ++w) {
            const uint32_t cw = codes_id[(size_t)row * W + w];
            codes[((size_t)blk * W + w) * 32 + lane] = cw;
            pc += __popc(cw);
        }
        pcnt[slot] = (uint16_t)pc;
        const float no = no_id[row], rh = rho_id[row];
        const double dno = no, drh = rh;
        fac[slot] = make_float2((float)(dno * dno), (float)(2.0 * dno / (drh * sqrt((double)D))));
        const double om = fmax(0.0, 1.0 - drh * drh);
        g1[slot] = (D > 1) ? (float)(2.0 * dno * sqrt(om) / (drh * sqrt((double)D - 1.0))) : 0.0f;
        n_o[slot] = no;
        rho[slot] = rh;
        rows[slot] = row;
        slot_of_row[row] = (uint32_t)slot;
    }
}

__global__ void hist_kernel(const int32_t* __restrict__ a, int64_t n, int64_t* __restrict__ h) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)&h[a[i]], 1ull);
}

__global__ void iota_kernel(uint32_t* v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

inline int grid_for(int64_t work, int per_block = 256) {
    int64_t g = (work + per_block - 1) / per_block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

// device buffer RAII for build temporaries
template <typename T>
struct DBuf {
    T* p = nullptr;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        if (count) RQ_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
    }
    ~DBuf() { release(); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
};

// stratified seeded sample: one row from each of m equal strata of [0, n)
std::vector<int64_t> stratified(int64_t n, int64_t m, uint64_t seed, uint32_t tag) {
    std::vector<int64_t> r(m);
    if (m >= n) {
        for (int64_t i = 0; i < m; ++i) r[i] = i;
        return r;
    }
    for (int64_t i = 0; i < m; ++i) {
        U4 w = philox4x32_10((uint32_t)seed, (uint32_t)(seed >> 32), U4{(uint32_t)i, (uint32_t)(i >> 32), tag, 0u});
        const int64_t lo = (n * i) / m, hi = (n * (i + 1)) / m;  // hi > lo since m < n
        const uint64_t u = ((uint64_t)w.x << 32) | w.y;
        r[i] = lo + (int64_t)(u % (uint64_t)(hi - lo));
    }
    return r;
}

}  // namespace

void free_index_memory(rabitq_index* idx) {
    cudaFree(idx->P);
    cudaFree(idx->Pt);
    idx->Pt = nullptr;
    cudaFree(idx->Cr);
    cudaFree(idx->cnorm);
    cudaFree(idx->list_off);
    cudaFree(idx->slot_off);
    cudaFree(idx->codes);
    cudaFree(idx->fac);
    cudaFree(idx->pcnt);
    idx->pcnt = nullptr;
    cudaFree(idx->g1);
    cudaFree(idx->n_o);
    cudaFree(idx->rho);
    cudaFree(idx->rows);
    cudaFree(idx->slot_of_row);
    cudaFree(idx->X_owned);
    cudaFree(idx->Xs);
    idx->Xs = nullptr;
    cudaFree(idx->codes8);
    idx->codes8 = nullptr;
    if (idx->side) cudaStreamDestroy(idx->side);
    idx->side = nullptr;
    cudaFree(idx->Corig);
    idx->Corig = nullptr;
    cudaFree(idx->list_amax);
    idx->list_amax = nullptr;
    idx->P = idx->Cr = idx->cnorm = nullptr;
    idx->list_off = idx->slot_off = nullptr;
    idx->codes = nullptr;
    idx->fac = nullptr;
    idx->g1 = idx->n_o = idx->rho = nullptr;
    idx->rows = nullptr;
    idx->slot_of_row = nullptr;
    idx->X_owned = nullptr;
    idx->X = nullptr;
}

void build_index(rabitq_index* idx, const float* X, int64_t n, int D, int nlist, uint64_t seed,
                 const rabitq_build_opts& o) {
    cudaStream_t st = idx->stream;
    const int W = (D + 31) / 32;
    idx->D = D;
    idx->W = W;
    idx->nlist = nlist;
    idx->n = n;
    idx->seed = seed;
    idx->id_offset = o.id_offset;

    cudaPointerAttributes pa{};
    RQ_CUDA(cudaPointerGetAttributes(&pa, X));
    const bool x_dev = (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
    if (x_dev) RQ_REQUIRE(pa.device == idx->device, RABITQ_ERR_INVALID_ARGUMENT, "X is on another device");

    // ---- vectors kept for the exact re-rank ----
    const float* Xd;
    if (o.borrow_vectors) {
        RQ_REQUIRE(x_dev, RABITQ_ERR_INVALID_ARGUMENT, "borrow_vectors requires a device pointer X");
        idx->borrowed = true;
        Xd = X;
    } else {
        RQ_CUDA(cudaMalloc(&idx->X_owned, (size_t)n * D * sizeof(float)));
        RQ_CUDA(cudaMemcpyAsync(idx->X_owned, X, (size_t)n * D * sizeof(float), cudaMemcpyDefault, st));
        Xd = idx->X_owned;
    }
    idx->X = Xd;
    {
        DBuf<int> flag(1);
        RQ_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
        finite_kernel<<<grid_for((int64_t)n * D), 256, 0, st>>>(Xd, (int64_t)n * D, flag.p);
        RQ_CHECK_LAUNCH();
        int h = 0;
        RQ_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        RQ_CUDA(cudaStreamSynchronize(st));
        RQ_REQUIRE(h == 0, RABITQ_ERR_INVALID_DATA, "X contains non-finite values");
    }

    // ---- rotation P ----
    RQ_CUDA(cudaMalloc(&idx->P, (size_t)D * D * sizeof(float)));
    if (o.rotation) {
        RQ_CUDA(cudaMemcpyAsync(idx->P, o.rotation, (size_t)D * D * sizeof(float), cudaMemcpyDefault, st));
    } else {
        std::vector<float> hP((size_t)D * D);
        haar_rotation_host(D, seed, hP.data());
        RQ_CUDA(cudaMemcpyAsync(idx->P, hP.data(), hP.size() * sizeof(float), cudaMemcpyHostToDevice, st));
        RQ_CUDA(cudaStreamSynchronize(st));
    }
    RQ_CUDA(cudaMalloc(&idx->Pt, (size_t)D * D * sizeof(float)));
    transpose_kernel<<<grid_for((int64_t)D * D), 256, 0, st>>>(idx->P, D, idx->Pt);
    RQ_CHECK_LAUNCH();
    RQ_CUDA(cudaMalloc(&idx->Cr, (size_t)nlist * D * sizeof(float)));
    RQ_CUDA(cudaMalloc(&idx->cnorm, (size_t)nlist * sizeof(float)));

    // distance block budget: rows per chunk so that [rows x nlist] fp32 <= ~1 GiB
    const int64_t chunk_rows = std::max<int64_t>(
        1024, std::min<int64_t>(std::min<int64_t>(n, 1 << 20), ((int64_t)1 << 28) / std::max(nlist, 1)));
    // distance GEMM + argmin: 3xTF32 tensor cores with the argmin fused into the
    // epilogue (no distance matrix; NEXT-3) when D % 4 == 0, else fp32 SIMT
    const bool tc_dist = D % 4 == 0 && !rq_diag_env("RABITQ_SIMT_GEMM");
    DBuf<float> dist(tc_dist ? 0 : (size_t)chunk_rows * nlist);
    DBuf<unsigned long long> akeys(tc_dist ? (size_t)chunk_rows : 0);
    auto nearest = [&](const float* A, int64_t m, int32_t* a_out, float* best, int32_t* prev,
                       unsigned long long* changed) {
        if (tc_dist) {
            RQ_CUDA(cudaMemsetAsync(akeys.p, 0xFF, (size_t)m * sizeof(unsigned long long), st));
            TgParams g{};
            g.A = A;
            g.lda = D;
            g.B = idx->Cr;
            g.ldb = D;
            g.K = D;
            g.M = m;
            g.N = nlist;
            g.b_norm = idx->cnorm;
            g.amin = akeys.p;
            tgemm(g, TG_EPI_ARGMIN, st);
            argmin_keys_kernel<<<grid_for(m), 256, 0, st>>>(akeys.p, m, a_out, best, prev, changed);
            RQ_CHECK_LAUNCH();
        } else {
            sgemm((int)m, nlist, D, A, D, idx->Cr, D, true, dist.p, nlist, 1, idx->cnorm, st);
            argmin_kernel<<<(int)((m * 32 + 255) / 256), 256, 0, st>>>(dist.p, m, nlist, a_out, best, prev, changed);
            RQ_CHECK_LAUNCH();
        }
    };

    // ---- k-means in the rotated space ----
    if (o.centroids_rot) {
        RQ_CUDA(cudaMemcpyAsync(idx->Cr, o.centroids_rot, (size_t)nlist * D * sizeof(float), cudaMemcpyDefault, st));
    } else {
        const int64_t ts = o.train_size > 0 ? std::min<int64_t>(o.train_size, n)
                                            : std::min<int64_t>(n, (int64_t)256 * nlist);
        RQ_REQUIRE(ts >= nlist, RABITQ_ERR_INVALID_ARGUMENT, "train_size < nlist");
        std::vector<int64_t> trows = stratified(n, ts, seed, 0x5452u /* 'TR' */);
        DBuf<int64_t> d_trows(ts);
        RQ_CUDA(cudaMemcpyAsync(d_trows.p, trows.data(), ts * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        DBuf<float> T((size_t)ts * D), Tr((size_t)ts * D);
        gather_rows_kernel<<<grid_for(ts * D), 256, 0, st>>>(Xd, D, d_trows.p, ts, T.p);
        RQ_CHECK_LAUNCH();
        sgemm((int)ts, D, D, T.p, D, idx->P, D, false, Tr.p, D, 0, nullptr, st);
        T.release();
        if (o.init_centroids) {
            DBuf<float> C0((size_t)nlist * D);
            RQ_CUDA(cudaMemcpyAsync(C0.p, o.init_centroids, (size_t)nlist * D * sizeof(float), cudaMemcpyDefault, st));
            sgemm(nlist, D, D, C0.p, D, idx->P, D, false, idx->Cr, D, 0, nullptr, st);
            RQ_CUDA(cudaStreamSynchronize(st));
        } else {
            std::vector<int64_t> crow = stratified(ts, nlist, seed, 0x4352u /* 'CR' */);
            DBuf<int64_t> d_crow(nlist);
            RQ_CUDA(cudaMemcpyAsync(d_crow.p, crow.data(), nlist * sizeof(int64_t), cudaMemcpyHostToDevice, st));
            gather_rows_kernel<<<grid_for((int64_t)nlist * D), 256, 0, st>>>(Tr.p, D, d_crow.p, nlist, idx->Cr);
            RQ_CHECK_LAUNCH();
            RQ_CUDA(cudaStreamSynchronize(st));
        }
        DBuf<int32_t> ta(ts), tprev(ts);
        DBuf<float> tbest(ts), tnorm(ts), sums((size_t)nlist * D);
        DBuf<int> counts(nlist);
        DBuf<unsigned long long> changed(1);
        RQ_CUDA(cudaMemsetAsync(tprev.p, 0xFF, ts * sizeof(int32_t), st));
        row_norm2_kernel<<<(int)((ts * 32 + 255) / 256), 256, 0, st>>>(Tr.p, (int)ts, D, tnorm.p);
        RQ_CHECK_LAUNCH();
        const int iters = o.kmeans_iters > 0 ? o.kmeans_iters : 25;
        std::vector<int> hcounts(nlist);
        std::vector<float> hbest, htn;
        for (int it = 0; it < iters; ++it) {
            row_norm2_kernel<<<(nlist * 32 + 255) / 256, 256, 0, st>>>(idx->Cr, nlist, D, idx->cnorm);
            RQ_CUDA(cudaMemsetAsync(changed.p, 0, sizeof(unsigned long long), st));
            for (int64_t r0 = 0; r0 < ts; r0 += chunk_rows) {
                const int64_t m = std::min(chunk_rows, ts - r0);
                nearest(Tr.p + (size_t)r0 * D, m, ta.p + r0, tbest.p + r0, tprev.p + r0, changed.p);
            }
            unsigned long long hchanged = 0;
            RQ_CUDA(cudaMemcpyAsync(&hchanged, changed.p, sizeof(hchanged), cudaMemcpyDeviceToHost, st));
            RQ_CUDA(cudaStreamSynchronize(st));
            if (hchanged == 0) break;  // converged: no assignment changed
            RQ_CUDA(cudaMemsetAsync(sums.p, 0, (size_t)nlist * D * sizeof(float), st));
            RQ_CUDA(cudaMemsetAsync(counts.p, 0, nlist * sizeof(int), st));
            kmeans_accum_kernel<<<(int)((ts * 32 + 255) / 256), 256, 0, st>>>(Tr.p, ts, D, ta.p, sums.p, counts.p);
            RQ_CHECK_LAUNCH();
            kmeans_divide_kernel<<<grid_for((int64_t)nlist * D), 256, 0, st>>>(idx->Cr, sums.p, counts.p, nlist, D);
            RQ_CHECK_LAUNCH();
            RQ_CUDA(cudaMemcpyAsync(hcounts.data(), counts.p, nlist * sizeof(int), cudaMemcpyDeviceToHost, st));
            RQ_CUDA(cudaStreamSynchronize(st));
            std::vector<int> empty;
            for (int j = 0; j < nlist; ++j)
                if (hcounts[j] == 0) empty.push_back(j);
            if (!empty.empty()) {
                // re-seed each empty cluster with a distinct farthest training point (R#6)
                hbest.resize(ts);
                htn.resize(ts);
                RQ_CUDA(cudaMemcpyAsync(hbest.data(), tbest.p, ts * sizeof(float), cudaMemcpyDeviceToHost, st));
                RQ_CUDA(cudaMemcpyAsync(htn.data(), tnorm.p, ts * sizeof(float), cudaMemcpyDeviceToHost, st));
                RQ_CUDA(cudaStreamSynchronize(st));
                std::vector<int64_t> order(ts);
                for (int64_t t = 0; t < ts; ++t) order[t] = t;
                const size_t ne = std::min<size_t>(empty.size(), (size_t)ts);
                std::partial_sort(order.begin(), order.begin() + ne, order.end(), [&](int64_t a, int64_t b) {
                    const float da = hbest[a] + htn[a], db = hbest[b] + htn[b];
                    return da > db || (da == db && a < b);
                });
                for (size_t e = 0; e < ne; ++e)
                    RQ_CUDA(cudaMemcpyAsync(idx->Cr + (size_t)empty[e] * D, Tr.p + (size_t)order[e] * D,
                                            D * sizeof(float), cudaMemcpyDeviceToDevice, st));
            }
        }
    }
    row_norm2_kernel<<<(nlist * 32 + 255) / 256, 256, 0, st>>>(idx->Cr, nlist, D, idx->cnorm);
    RQ_CHECK_LAUNCH();

    // ---- assign + encode all vectors ----
    DBuf<int32_t> assign(n);
    DBuf<uint32_t> codes_id((size_t)n * W);
    DBuf<float> no_id(n), rho_id(n);
    {
        DBuf<float> xr((size_t)chunk_rows * D);
        for (int64_t r0 = 0; r0 < n; r0 += chunk_rows) {
            const int64_t m = std::min(chunk_rows, n - r0);
            sgemm((int)m, D, D, Xd + (size_t)r0 * D, D, idx->P, D, false, xr.p, D, 0, nullptr, st);
            nearest(xr.p, m, assign.p + r0, nullptr, nullptr, nullptr);
            encode_kernel<<<(int)((m * 32 + 255) / 256), 256, 0, st>>>(xr.p, m, D, W, idx->Cr, assign.p + r0,
                                                                         codes_id.p + (size_t)r0 * W, no_id.p + r0,
                                                                         rho_id.p + r0);
            RQ_CHECK_LAUNCH();
        }
    }
    dist.release();
    akeys.release();

    // ---- lists: sizes, offsets, 32-aligned slots ----
    DBuf<int64_t> hist(nlist);
    RQ_CUDA(cudaMemsetAsync(hist.p, 0, nlist * sizeof(int64_t), st));
    hist_kernel<<<grid_for(n), 256, 0, st>>>(assign.p, n, hist.p);
    RQ_CHECK_LAUNCH();
    std::vector<int64_t> sizes(nlist);
    RQ_CUDA(cudaMemcpyAsync(sizes.data(), hist.p, nlist * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    RQ_CUDA(cudaStreamSynchronize(st));
    idx->h_list_off.assign(nlist + 1, 0);
    idx->h_slot_off.assign(nlist + 1, 0);
    idx->max_list = 0;
    idx->tiles8_sum = 0;
    for (int j = 0; j < nlist; ++j) {
        idx->h_list_off[j + 1] = idx->h_list_off[j] + sizes[j];
        idx->h_slot_off[j + 1] = idx->h_slot_off[j] + ((sizes[j] + 31) / 32) * 32;
        idx->max_list = std::max(idx->max_list, sizes[j]);
        idx->tiles8_sum += ((sizes[j] + 127) / 128 + 7) / 8;
    }
    idx->nslots = idx->h_slot_off[nlist];
    // one spare 128-slot tile so bulk tile loads past the last list stay in bounds
    const int64_t alloc_slots = idx->nslots + 128;
    RQ_CUDA(cudaMalloc(&idx->list_off, (nlist + 1) * sizeof(int64_t)));
    RQ_CUDA(cudaMalloc(&idx->slot_off, (nlist + 1) * sizeof(int64_t)));
    RQ_CUDA(cudaMemcpyAsync(idx->list_off, idx->h_list_off.data(), (nlist + 1) * sizeof(int64_t),
                            cudaMemcpyHostToDevice, st));
    RQ_CUDA(cudaMemcpyAsync(idx->slot_off, idx->h_slot_off.data(), (nlist + 1) * sizeof(int64_t),
                            cudaMemcpyHostToDevice, st));
    RQ_CUDA(cudaMalloc(&idx->codes, (size_t)alloc_slots * W * sizeof(uint32_t)));
    RQ_CUDA(cudaMalloc(&idx->fac, (size_t)alloc_slots * sizeof(float2)));
    RQ_CUDA(cudaMalloc(&idx->pcnt, (size_t)alloc_slots * sizeof(uint16_t)));
    RQ_CUDA(cudaMemsetAsync(idx->pcnt, 0, (size_t)alloc_slots * sizeof(uint16_t), st));
    RQ_CUDA(cudaMalloc(&idx->g1, (size_t)alloc_slots * sizeof(float)));
    RQ_CUDA(cudaMalloc(&idx->n_o, (size_t)alloc_slots * sizeof(float)));
    RQ_CUDA(cudaMalloc(&idx->rho, (size_t)alloc_slots * sizeof(float)));
    RQ_CUDA(cudaMalloc(&idx->rows, (size_t)alloc_slots * sizeof(uint32_t)));
    RQ_CUDA(cudaMalloc(&idx->slot_of_row, (size_t)n * sizeof(uint32_t)));
    RQ_CUDA(cudaMemsetAsync(idx->codes, 0, (size_t)alloc_slots * W * sizeof(uint32_t), st));
    RQ_CUDA(cudaMemsetAsync(idx->fac, 0, (size_t)alloc_slots * sizeof(float2), st));
    RQ_CUDA(cudaMemsetAsync(idx->g1, 0, (size_t)alloc_slots * sizeof(float), st));
    RQ_CUDA(cudaMemsetAsync(idx->n_o, 0, (size_t)alloc_slots * sizeof(float), st));
    RQ_CUDA(cudaMemsetAsync(idx->rho, 0, (size_t)alloc_slots * sizeof(float), st));
    RQ_CUDA(cudaMemsetAsync(idx->rows, 0xFF, (size_t)alloc_slots * sizeof(uint32_t), st));

    // ---- stable sort by list (ids ascending within a list) ----
    {
        DBuf<int32_t> skeys(n);
        DBuf<uint32_t> vals(n), svals(n);
        iota_kernel<<<grid_for(n), 256, 0, st>>>(vals.p, n);
        RQ_CHECK_LAUNCH();
        int end_bit = 1;
        while ((1 << end_bit) < nlist) ++end_bit;
        size_t tmp_bytes = 0;
        RQ_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, assign.p, skeys.p, vals.p, svals.p, (int)n, 0,
                                                end_bit, st));
        DBuf<uint8_t> tmp(tmp_bytes);
        RQ_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, assign.p, skeys.p, vals.p, svals.p, (int)n, 0,
                                                end_bit, st));
        scatter_kernel<<<grid_for(n), 256, 0, st>>>(n, D, W, skeys.p, svals.p, idx->list_off, idx->slot_off,
                                                    codes_id.p, no_id.p, rho_id.p, idx->codes, idx->fac, idx->g1,
                                                    idx->n_o, idx->rho, idx->rows, idx->slot_of_row, idx->pcnt);
        RQ_CHECK_LAUNCH();
        RQ_CUDA(cudaStreamSynchronize(st));
    }

    RQ_CUDA(cudaMalloc(&idx->list_amax, (size_t)nlist * sizeof(float)));
    list_amax_kernel<<<std::min(nlist, 4096), 256, 0, st>>>(idx->fac, idx->slot_off, idx->list_off, nlist,
                                                           idx->list_amax);
    RQ_CHECK_LAUNCH();

    // ---- expanded codes: the grouped scan's A operand by TMA (when they fit comfortably) ----
    {
        const char* env = rq_diag_env("RABITQ_CODES8");  // "0": not built (the scan expands codes in the kernel)
        size_t freeb = 0, totalb = 0;
        RQ_CUDA(cudaMemGetInfo(&freeb, &totalb));
        const size_t bytes = (size_t)(idx->nslots + 128) * 32 * W;
        if (!(env && env[0] == '0') && W <= 32 && bytes <= (size_t)(0.25 * (double)freeb)) {
            expand_codes(idx, st);
            RQ_CUDA(cudaStreamSynchronize(st));
        }
    }

    // ---- slot-ordered vectors for the dense re-rank (when they fit comfortably) ----
    {
        const char* env = rq_diag_env("RABITQ_SLOT_VECTORS");  // "0": never build the copy
        size_t freeb = 0, totalb = 0;
        RQ_CUDA(cudaMemGetInfo(&freeb, &totalb));
        const size_t bytes = (size_t)(idx->nslots + 128) * D * sizeof(float);
        if (D % 4 == 0 && !(env && env[0] == '0') && bytes <= (size_t)(0.4 * (double)freeb)) {
            // original-space centroids c = P c' (row form: C = C' P^T)
            RQ_CUDA(cudaMalloc(&idx->Corig, (size_t)nlist * D * sizeof(float)));
            sgemm(nlist, D, D, idx->Cr, D, idx->Pt, D, false, idx->Corig, D, 0, nullptr, st);
            RQ_CUDA(cudaMalloc(&idx->Xs, bytes));
            RQ_CUDA(cudaMemsetAsync(idx->Xs + (size_t)idx->nslots * D, 0, (size_t)128 * D * sizeof(float), st));
            slot_rows_kernel<<<std::min(nlist, 4096), 256, 0, st>>>(idx->X, D, idx->rows, idx->slot_off, idx->Corig,
                                                                    nlist, idx->Xs);
            RQ_CHECK_LAUNCH();
            RQ_CUDA(cudaStreamSynchronize(st));
        }
    }
}

}  // namespace rabitq
