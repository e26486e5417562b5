// tc_sm100.cuh -- minimal tcgen05 (5th-gen tensor core) toolkit for sm_100a:
// TMEM allocation, K-major SWIZZLE_128B shared-memory operand images, the
// kind::tf32 MMA, commit-to-mbarrier, TMEM <-> register moves.
//
// Operand image (one K-block = 32 fp32 of K): row m occupies 128 bytes, the
// 16-byte chunk q of row m sits at chunk position q ^ (m & 7), 8-row groups
// are 1024 bytes apart (SBO), so a K-block of an R-row operand is R*128 bytes
// and must start 1024-byte aligned.  One MMA consumes K = 8 (32 bytes): the
// k-th step of a K-block advances the descriptor start address by 32*k bytes
// (the hardware applies the swizzle to the final address bits).
//
// 3xTF32: x = hi + lo with hi = tf32(x), lo = tf32(x - hi); a*b is formed as
// hi*hi + hi*lo + lo*hi (the lo*lo term, ~2^-22 relative, is dropped), which
// keeps the trailing update at ~fp32 accuracy on the TF32 tensor pipe.
#pragma once
#include <cstdint>

namespace bsvd {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// float offset of element (row, k) inside a K-major SW128 image whose K-blocks
// (32 columns of K) are `kb_stride` floats apart
__device__ __forceinline__ int img_off(int row, int k, int kb_stride) {
    return (k >> 5) * kb_stride + row * 32 + ((((k & 31) >> 2) ^ (row & 7)) << 2) + (k & 3);
}

__device__ __forceinline__ float tf32_rn(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ void split3(float x, float &hi, float &lo) {
    hi = tf32_rn(x);
    lo = tf32_rn(x - hi);
}

// Shared-memory matrix descriptor: K-major, SWIZZLE_128B, LBO = 16 B (unused
// for swizzled K-major), SBO = 1024 B, descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

// Instruction descriptor: kind::tf32, D fp32, A/B K-major, M x N.
template <int M, int N, bool NEG_A>
__device__ __forceinline__ constexpr uint32_t idesc_tf32() {
    static_assert(M == 128 && N % 16 == 0 && N >= 16 && N <= 256, "UMMA shape");
    return (1u << 4) | (2u << 7) | (2u << 10) | ((NEG_A ? 1u : 0u) << 13) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         bool accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)accumulate));
}

__device__ __forceinline__ void commit(uint64_t *mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(mbar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mbar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// TMEM allocation by one full warp; the base address lands in *slot.
template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t *slot) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "n"(COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int COLS>
__device__ __forceinline__ void tmem_free(uint32_t base) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS) : "memory");
}

// 32 lanes x 16 columns: thread t of warp w <-> TMEM lane 32*(w%4)+t.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D(tmem) (+)= sum over NKB K-blocks of A(M x 32) * B(N x 32)^T, 3xTF32 from
// hi/lo images: A_hi/A_lo and B_hi/B_lo K-block kb at base + kb * stride.
// Issued by one thread.
template <int M, int N, bool NEG_A>
__device__ __forceinline__ void mma3_kblock(uint32_t d_tmem, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi,
                                            uint32_t b_lo, bool accumulate) {
    constexpr uint32_t id = idesc_tf32<M, N, NEG_A>();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint32_t o = 32u * k;
        mma_tf32(d_tmem, sdesc(a_hi + o), sdesc(b_hi + o), id, accumulate || k > 0);
        mma_tf32(d_tmem, sdesc(a_hi + o), sdesc(b_lo + o), id, true);
        mma_tf32(d_tmem, sdesc(a_lo + o), sdesc(b_hi + o), id, true);
    }
}

}  // namespace tc
}  // namespace bsvd
