// tc.cuh -- thin inline-PTX wrappers for the sm_100a features the grouped
// scan uses: tcgen05 (UMMA int8, TMEM alloc/ld, commit), mbarriers,
// cp.async and the async-proxy fence.  Field layouts follow the PTX ISA
// descriptions of the shared-memory matrix descriptor and the instruction
// descriptor for .kind::i8.
#pragma once
#include <stdint.h>

namespace rabitq {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)  // suspend-time hint (ns): sleep in hardware until the phase completes
        : "memory");
}

// the same on a precomputed shared-space address (no generic -> shared
// conversion per call in hot loops)
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}" ::"r"(bar),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// The same for waits that are rarely on the critical path (a producer ahead of
// its consumer): exponential __nanosleep back-off between polls keeps the
// waiting warp from taking issue slots from the warps doing the work.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) {
    uint32_t ns = 32;
    while (!mbar_test(bar, parity)) {
        __nanosleep(ns);
        if (ns < 512) ns <<= 1;
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void named_barrier(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- TMA
// 2D tiled bulk tensor load global -> shared, completion counted in bytes on `bar`
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(smem_dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
// 1D bulk copy global -> shared (size multiple of 16 bytes), completion in bytes on `bar`
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(smem_dst)),
                 "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// ---------------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// 16-byte async copy (L2 only); src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
// 4-byte async copy; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Shared-memory matrix descriptor, canonical K-major layout without swizzle:
// 8 rows x 16 bytes core matrices; LBO = byte distance between core matrices
// adjacent along K, SBO = between core matrices adjacent along M/N.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
    // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
    return d;
}

// K-major operand written by TMA with 128-byte swizzle: rows of 128 bytes,
// 8-row swizzle atoms 1024 bytes apart (SBO); LBO unused (1 by convention).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}

// Instruction descriptor, .kind::i8: D = s32, A = u8 or s8, B = u8, both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed = false, bool b_signed = false) {
    return (2u << 4)                       // c_format: S32
           | ((a_signed ? 1u : 0u) << 7)   // a format: 0 unsigned / 1 signed 8-bit
           | ((b_signed ? 1u : 0u) << 10)  // b format: 0 unsigned / 1 signed 8-bit
           | (0u << 15) | (0u << 16)       // a/b major: K
           | ((uint32_t)(N >> 3) << 17)    // N / 8
           | ((uint32_t)(M >> 4) << 24);   // M / 16
}

// Instruction descriptor, .kind::f8f6f4 with A = B = e4m3 and an f32 accumulator
// (dtype 1 at bits 4-5, a/b formats E4M3 = 0), both K-major.
__host__ __device__ constexpr uint32_t idesc_f8(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// idesc of the grouped scan's code x query contraction: e4m3 (kF8) or s8 x u8
template <bool kF8>
__host__ __device__ constexpr uint32_t idesc_scan(int M, int N) {
    return kF8 ? idesc_f8(M, N) : idesc_i8(M, N, /*a_signed=*/true);
}

// D[tmem] (+)= A[smem] . B[smem]^T, one elected thread issues.
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]^T (A: 128 lanes = rows, K bytes packed 4 per
// 32-bit column), one elected thread issues.
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// The same from a whole warp (all lanes call it with warp-uniform operands):
// one lane is elected inside the asm, so the operands can stay in uniform
// registers and no per-instruction election loop is generated.
__device__ __forceinline__ void mma_i8_ts_warp(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// nk (1..4) UMMAs of consecutive 32-byte K steps (A: +8 TMEM columns, B
// descriptor: +2 (32 bytes)) and the commit of `bar`, from a whole warp with one
// election: the address increments stay inside the asm, so the operands cross
// to uniform registers once per chunk instead of once per UMMA.  kF8: the
// operands are e4m3 bytes (.kind::f8f6f4, f32 accumulator) instead of 8-bit
// integers (.kind::i8, s32 accumulator).
#define RQ_KIND_I8 "kind::i8"
#define RQ_KIND_F8 "kind::f8f6f4"
#define RQ_MMA_TS_HEAD(K)                                 \
    "{\n\t.reg .pred p, e, t;\n\t"                        \
    ".reg .b32 a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t" \
    "setp.ne.b32 p, %4, 0;\n\t"                          \
    "setp.eq.b32 t, 0, 0;\n\t"                           \
    "add.u32 a1, %1, 8;\n\tadd.u32 a2, %1, 16;\n\tadd.u32 a3, %1, 24;\n\t" \
    "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t" \
    "elect.sync _|e, 0xffffffff;\n\t"                    \
    "@e tcgen05.mma.cta_group::1." K " [%0], [%1], %2, %3, p;\n\t"
#define RQ_MMA_TS_K1(K) "@e tcgen05.mma.cta_group::1." K " [%0], [a1], b1, %3, t;\n\t"
#define RQ_MMA_TS_K2(K) "@e tcgen05.mma.cta_group::1." K " [%0], [a2], b2, %3, t;\n\t"
#define RQ_MMA_TS_K3(K) "@e tcgen05.mma.cta_group::1." K " [%0], [a3], b3, %3, t;\n\t"
#define RQ_MMA_SS_HEAD(K)                                 \
    "{\n\t.reg .pred p, e, t;\n\t"                        \
    ".reg .b64 a1, a2, a3, b1, b2, b3;\n\t"              \
    "setp.ne.b32 p, %4, 0;\n\t"                          \
    "setp.eq.b32 t, 0, 0;\n\t"                           \
    "add.u64 a1, %1, 2;\n\tadd.u64 a2, %1, 4;\n\tadd.u64 a3, %1, 6;\n\t" \
    "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t" \
    "elect.sync _|e, 0xffffffff;\n\t"                    \
    "@e tcgen05.mma.cta_group::1." K " [%0], %1, %2, %3, p;\n\t"
#define RQ_MMA_SS_K1(K) "@e tcgen05.mma.cta_group::1." K " [%0], a1, b1, %3, t;\n\t"
#define RQ_MMA_SS_K2(K) "@e tcgen05.mma.cta_group::1." K " [%0], a2, b2, %3, t;\n\t"
#define RQ_MMA_SS_K3(K) "@e tcgen05.mma.cta_group::1." K " [%0], a3, b3, %3, t;\n\t"
#define RQ_MMA_TAIL "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t}"
#define RQ_MMA_ARGS_TS ::"r"(tmem_d), "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(smem_u32(bar)) : "memory"
#define RQ_MMA_ARGS_SS ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(smem_u32(bar)) : "memory"
#define RQ_MMA_SWITCH(HEAD, K1, K2, K3, ARGS, KIND)                                       \
    switch (nk) {                                                                         \
        case 1: asm volatile(HEAD(KIND) RQ_MMA_TAIL ARGS); break;                         \
        case 2: asm volatile(HEAD(KIND) K1(KIND) RQ_MMA_TAIL ARGS); break;                \
        case 3: asm volatile(HEAD(KIND) K1(KIND) K2(KIND) RQ_MMA_TAIL ARGS); break;       \
        default: asm volatile(HEAD(KIND) K1(KIND) K2(KIND) K3(KIND) RQ_MMA_TAIL ARGS); break; \
    }
template <bool kF8 = false>
__device__ __forceinline__ void mma_i8_ts_chunk(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate, int nk, uint64_t* bar) {
    if constexpr (kF8) {
        RQ_MMA_SWITCH(RQ_MMA_TS_HEAD, RQ_MMA_TS_K1, RQ_MMA_TS_K2, RQ_MMA_TS_K3, RQ_MMA_ARGS_TS, RQ_KIND_F8)
    } else {
        RQ_MMA_SWITCH(RQ_MMA_TS_HEAD, RQ_MMA_TS_K1, RQ_MMA_TS_K2, RQ_MMA_TS_K3, RQ_MMA_ARGS_TS, RQ_KIND_I8)
    }
}

// The same with A in shared memory too (TMA-written, 128-byte swizzle, K-major):
// both descriptors advance by 2 (32 bytes) per K step.
template <bool kF8 = false>
__device__ __forceinline__ void mma_i8_ss_chunk(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate, int nk, uint64_t* bar) {
    if constexpr (kF8) {
        RQ_MMA_SWITCH(RQ_MMA_SS_HEAD, RQ_MMA_SS_K1, RQ_MMA_SS_K2, RQ_MMA_SS_K3, RQ_MMA_ARGS_SS, RQ_KIND_F8)
    } else {
        RQ_MMA_SWITCH(RQ_MMA_SS_HEAD, RQ_MMA_SS_K1, RQ_MMA_SS_K2, RQ_MMA_SS_K3, RQ_MMA_ARGS_SS, RQ_KIND_I8)
    }
}
#undef RQ_MMA_SWITCH
#undef RQ_MMA_ARGS_SS
#undef RQ_MMA_ARGS_TS
#undef RQ_MMA_TAIL
#undef RQ_MMA_SS_K3
#undef RQ_MMA_SS_K2
#undef RQ_MMA_SS_K1
#undef RQ_MMA_SS_HEAD
#undef RQ_MMA_TS_K3
#undef RQ_MMA_TS_K2
#undef RQ_MMA_TS_K1
#undef RQ_MMA_TS_HEAD
#undef RQ_KIND_F8
#undef RQ_KIND_I8

__device__ __forceinline__ void commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// 32 lanes x 8 columns of 32-bit into TMEM (warp w writes lanes 32 (w % 4) ..);
// tmem_st_wait() makes them visible to a following tcgen05 fence + sync.
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint4& lo, const uint4& hi) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(lo.x),
                 "r"(lo.y), "r"(lo.z), "r"(lo.w), "r"(hi.x), "r"(hi.y), "r"(hi.z), "r"(hi.w)
                 : "memory");
}
// 32 lanes x 16 columns of 32-bit into TMEM
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint4& a, const uint4& b, const uint4& c,
                                          const uint4& d) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w), "r"(c.x), "r"(c.y), "r"(c.z),
        "r"(c.w), "r"(d.x), "r"(d.y), "r"(d.z), "r"(d.w)
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// arrive on an mbarrier once every previously issued tcgen05.mma of this thread completed
__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// 32 lanes x 16 columns of 32-bit from TMEM (waits for completion)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 1 column of 32-bit from TMEM (waits for completion)
__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    return r;
}

// 32 lanes x 32 columns of 32-bit from TMEM (warp w reads lanes 32 (w % 4) ..)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// 32 lanes x 16 columns of 32-bit from TMEM without waiting (tmem_ld_wait()
// before the registers are read)
__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// arrive on an mbarrier with an arrival count
__device__ __forceinline__ void mbar_arrive_cnt_s(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

// One unit of the folded scan, from a whole warp with one election:
//   D_ip = A_codes . B_query^T over nk 32-byte K steps (.kind::f8f6f4, e4m3),
//   D_e  = X . BX^T over K = 16 tf32 (two UMMAs of K = 8, canonical K-major
//          layout without swizzle: LBO = 128 B, SBO = 512 B, +256 B per UMMA),
// then one commit of `bar` (both accumulators complete).
__device__ __forceinline__ void mma_fold_unit(uint32_t tmem_ip, uint32_t tmem_e, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc8, int nk, uint64_t xdesc, uint64_t bxdesc,
                                              uint32_t idesc32, uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e, t, p1, p2, p3;\n\t"
        ".reg .b64 a1, a2, a3, b1, b2, b3, x1, y1;\n\t"
        "setp.eq.b32 t, 0, 0;\n\t"
        "setp.gt.s32 p1, %5, 1;\n\tsetp.gt.s32 p2, %5, 2;\n\tsetp.gt.s32 p3, %5, 3;\n\t"
        "add.u64 a1, %2, 2;\n\tadd.u64 a2, %2, 4;\n\tadd.u64 a3, %2, 6;\n\t"
        "add.u64 b1, %3, 2;\n\tadd.u64 b2, %3, 4;\n\tadd.u64 b3, %3, 6;\n\t"
        "add.u64 x1, %6, 16;\n\tadd.u64 y1, %7, 16;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %2, %3, %4, !t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], %6, %7, %8, !t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], x1, y1, %8, t;\n\t"
        "and.pred p1, p1, e;\n\tand.pred p2, p2, e;\n\tand.pred p3, p3, e;\n\t"
        "@p1 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a1, b1, %4, t;\n\t"
        "@p2 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a2, b2, %4, t;\n\t"
        "@p3 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a3, b3, %4, t;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%9];\n\t}" ::"r"(tmem_ip),
        "r"(tmem_e), "l"(adesc), "l"(bdesc), "r"(idesc8), "r"(nk), "l"(xdesc), "l"(bxdesc), "r"(idesc32),
        "r"(smem_u32(bar))
        : "memory");
}

// The same issued by a single thread (no election), NK = 1..4 K steps of the
// ip contraction known at compile time.
template <int NK>
__device__ __forceinline__ void mma_fold_unit1(uint32_t tmem_ip, uint32_t tmem_e, uint64_t adesc, uint64_t bdesc,
                                               uint32_t idesc8, uint64_t xdesc, uint64_t bxdesc, uint32_t idesc32,
                                               uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred t;\n\t"
        ".reg .b64 a1, b1, x1, y1;\n\t"
        "setp.eq.b32 t, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %2, %3, %4, !t;\n\t"
        "add.u64 x1, %5, 16;\n\tadd.u64 y1, %6, 16;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%1], %5, %6, %7, !t;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%1], x1, y1, %7, t;\n\t}" ::"r"(tmem_ip),
        "r"(tmem_e), "l"(adesc), "l"(bdesc), "r"(idesc8), "l"(xdesc), "l"(bxdesc), "r"(idesc32)
        : "memory");
#pragma unroll
    for (int k = 1; k < NK; ++k) {
        asm volatile(
            "{\n\t.reg .pred t;\n\tsetp.eq.b32 t, 0, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, t;\n\t}" ::"r"(tmem_ip),
            "l"(adesc + (uint64_t)(2 * k)), "l"(bdesc + (uint64_t)(2 * k)), "r"(idesc8)
            : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// Warp-wide version (every lane calls it with warp-uniform operands; one lane
// is elected inside each asm).
template <int NK>
__device__ __forceinline__ void mma_fold_unit_w(uint32_t tmem_ip, uint32_t tmem_e, uint64_t adesc, uint64_t bdesc,
                                                uint32_t idesc8, uint64_t xdesc, uint64_t bxdesc, uint32_t idesc32,
                                                uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred t, e;\n\t"
        ".reg .b64 a1, a2, a3, b1, b2, b3, x1, y1;\n\t"
        "setp.eq.b32 t, 0, 0;\n\t"
        "add.u64 x1, %5, 16;\n\tadd.u64 y1, %6, 16;\n\t"
        "add.u64 a1, %2, 2;\n\tadd.u64 a2, %2, 4;\n\tadd.u64 a3, %2, 6;\n\t"
        "add.u64 b1, %3, 2;\n\tadd.u64 b2, %3, 4;\n\tadd.u64 b3, %3, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %2, %3, %4, !t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], %5, %6, %7, !t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%1], x1, y1, %7, t;\n\t"
        ".reg .pred k1, k2, k3;\n\t"
        "setp.gt.and.s32 k1, %9, 1, e;\n\tsetp.gt.and.s32 k2, %9, 2, e;\n\tsetp.gt.and.s32 k3, %9, 3, e;\n\t"
        "@k1 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a1, b1, %4, t;\n\t"
        "@k2 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a2, b2, %4, t;\n\t"
        "@k3 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a3, b3, %4, t;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t}" ::"r"(tmem_ip),
        "r"(tmem_e), "l"(adesc), "l"(bdesc), "r"(idesc8), "l"(xdesc), "l"(bxdesc), "r"(idesc32), "r"(bar), "n"(NK)
        : "memory");
}

// One accumulator: D = A_codes . B_query^T (NK K steps, .kind::f8f6f4) + X . BX^T
// (K = 16 tf32), warp-wide with one elected lane, then one commit of `bar`.
template <int NK>
__device__ __forceinline__ void mma_fold_acc_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc8,
                                               uint64_t xdesc, uint64_t bxdesc, uint32_t idesc32, uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred t, e, k1, k2, k3;\n\t"
        ".reg .b64 a1, a2, a3, b1, b2, b3, x1, y1;\n\t"
        "setp.eq.b32 t, 0, 0;\n\t"
        "add.u64 x1, %4, 16;\n\tadd.u64 y1, %5, 16;\n\t"
        "add.u64 a1, %1, 2;\n\tadd.u64 a2, %1, 4;\n\tadd.u64 a3, %1, 6;\n\t"
        "add.u64 b1, %2, 2;\n\tadd.u64 b2, %2, 4;\n\tadd.u64 b3, %2, 6;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.gt.and.s32 k1, %8, 1, e;\n\tsetp.gt.and.s32 k2, %8, 2, e;\n\tsetp.gt.and.s32 k3, %8, 3, e;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, !t;\n\t"
        "@k1 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a1, b1, %3, t;\n\t"
        "@k2 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a2, b2, %3, t;\n\t"
        "@k3 tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a3, b3, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %4, %5, %6, t;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], x1, y1, %6, t;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%7];\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc8), "l"(xdesc), "l"(bxdesc), "r"(idesc32), "r"(bar), "r"(NK)
        : "memory");
}

__host__ __device__ constexpr uint32_t idesc_tf32_f32(int M, int N) {
    return (1u << 4)                 // c_format: F32
           | (2u << 7) | (2u << 10)  // a/b format: TF32
           | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

}  // namespace tc
}  // namespace rabitq
