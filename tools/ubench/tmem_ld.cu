// TMEM read throughput microbenchmark (tcgen05.ld 32x32b): bytes per cycle per
// SM for 4..24 reading warps, loads of 16 / 64 columns per wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld tools/ubench/tmem_ld.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
#define LD16(r, addr)                                                                                      \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) \
                 : "r"(addr))

template <int PER_WAIT>
__global__ void kern(int iters, unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t base_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = base_s + ((uint32_t)((warp & 3) * 32) << 16);
    uint32_t x = 0;
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[PER_WAIT][16];
#pragma unroll
        for (int p = 0; p < PER_WAIT; ++p) LD16(r[p], tm + (uint32_t)((((it * PER_WAIT + p) * 16) + (warp >> 2) * 64) & 511));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int p = 0; p < PER_WAIT; ++p)
#pragma unroll
            for (int i = 0; i < 16; ++i) x ^= r[p][i];
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
    if (x == 0x12345678u) sink[threadIdx.x] = x;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base_s));
}

int main() {
    unsigned long long* cyc; uint32_t* sink;
    cudaMalloc(&cyc, 8); cudaMalloc(&sink, 4096);
    const int iters = 4096;
    for (int pw : {1, 2, 4}) {
        for (int nw : {4, 8, 12, 16, 24, 32}) {
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            auto launch = [&]() {
                if (pw == 1) kern<1><<<148, nw * 32>>>(iters, cyc, sink);
                if (pw == 2) kern<2><<<148, nw * 32>>>(iters, cyc, sink);
                if (pw == 4) kern<4><<<148, nw * 32>>>(iters, cyc, sink);
            };
            launch();
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double bytes = (double)nw * 32 * 16 * 4 * pw * iters;
            printf("per_wait=%d warps=%2d cycles=%llu  B/cyc/SM=%.1f  (event %.3f ms, %.2f TB/s chip) err=%s\n", pw, nw, c,
                   bytes / c, ms, bytes * 148 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
