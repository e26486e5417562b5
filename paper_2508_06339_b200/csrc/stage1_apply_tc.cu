// stage1_apply_tc.cu -- the stage-1 trailing update on the 5th-generation
// tensor cores (tcgen05, kind::tf32, 3xTF32 split for fp32 accuracy), for
// fp32 compute at ts = 128 (the headline configuration).  Same math as the
// FMA kernels of stage1_apply.cu (the reference's UNMQR / TSMQR,
// kernels.py:364-421, in compact-WY form):
//
//   leaf  : W = V^T X ;             X -= U W
//   TT    : W = X_top + Vb^T X_bot ; X_top -= T^T W ;  X_bot -= U W
//
// One CTA = one 128 x 128 column block of one tile row (leaf) or node pair
// (TT).  X is read once from HBM into (a) the fp32 accumulator columns of
// TMEM (tcgen05.st: exact, so the update X - U W is formed in TMEM with no
// rounding of X) and (b) the hi/lo TF32 B-operand image in shared memory.
// W = V^T X accumulates in TMEM, is read back once, split into hi/lo and
// becomes the B operand of the second product, which the MMA subtracts from
// the X accumulators (A negated in the instruction descriptor).  The
// 128 x 128 A operands (V^T, T^T, U) come pre-split and pre-swizzled from
// k_node_tu and stream through two 32 KB K-block buffers by bulk async copy
// (cp.async.bulk, completion on an mbarrier), one thread issuing copies and
// MMAs, commit-to-mbarrier freeing each buffer.  X is written back from TMEM.
#include "common.cuh"
#include "kernels.cuh"
#include "tc_sm100.cuh"

namespace bsvd {
namespace tcapply {

constexpr int TS = 128;           // tile size (= UMMA M = K of both products)
constexpr int BN = 128;           // columns per CTA (= UMMA N)
constexpr int NT = 256;           // threads: row r = tid % 128, column half tid / 128
constexpr int CHUNK = 2 * TS * 32;            // floats per A K-block (hi + lo)
constexpr int BIMG = BN * TS;                 // floats per B image (hi or lo)
constexpr size_t SMEM = (size_t)(2 * CHUNK + 2 * BIMG) * sizeof(float) + 1024;

template <typename S>
struct View {
    S *base;
    int64_t rs, cs;
    __device__ __forceinline__ S *ptr(int64_t r, int64_t c) const { return base + r * rs + c * cs; }
};

__device__ __forceinline__ void bulk_load(float *dst, const float *src, uint32_t bytes, uint64_t *mbar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(mbar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            tc::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(tc::smem_u32(mbar))
        : "memory");
}

// Load 16 columns [c0, c0+16) of view row r (thread's row) as fp32.
template <typename S>
__device__ __forceinline__ void load_row16(const View<S> &V, int64_t r, int64_t c0, float (&v)[16]) {
    using CV = Conv<S, float>;
    if (V.cs == 1) {                                   // row contiguous (LQ side)
        const S *p = V.ptr(r, c0);
        if constexpr (sizeof(S) == 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 f = __ldcg(reinterpret_cast<const float4 *>(p) + q);
                v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
            }
        } else {                                       // fp16 storage: two 16-byte loads
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint4 u = __ldcg(reinterpret_cast<const uint4 *>(p) + q);
                const __half2 *h2 = reinterpret_cast<const __half2 *>(&u);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __half22float2(h2[e]);
                    v[8 * q + 2 * e] = f.x;
                    v[8 * q + 2 * e + 1] = f.y;
                }
            }
        }
    } else {                                           // column contiguous: coalesced over r
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = CV::ld(*V.ptr(r, c0 + q));
    }
}
template <typename S>
__device__ __forceinline__ void store_row16(const View<S> &V, int64_t r, int64_t c0, const float (&v)[16]) {
    using CV = Conv<S, float>;
    if (V.cs == 1) {
        S *p = V.ptr(r, c0);
        if constexpr (sizeof(S) == 4) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                reinterpret_cast<float4 *>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                uint4 u;
                __half2 *h2 = reinterpret_cast<__half2 *>(&u);
#pragma unroll
                for (int e = 0; e < 4; ++e) h2[e] = __floats2half2_rn(v[8 * q + 2 * e], v[8 * q + 2 * e + 1]);
                reinterpret_cast<uint4 *>(p)[q] = u;
            }
        }
    } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) *V.ptr(r, c0 + q) = CV::st(v[q]);
    }
}

// 16 values of B-operand row block (rows c0..c0+15 of the N x K image, K index k)
__device__ __forceinline__ void put_b16(float *Bhi, float *Blo, int c0, int k, const float (&v)[16]) {
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        float h, l;
        tc::split3(v[q], h, l);
        const int o = tc::img_off(c0 + q, k, BN * 32);
        Bhi[o] = h;
        Blo[o] = l;
    }
}

struct Pipe {
    uint64_t full[2], free_[2], done;
    uint32_t tslot;
};

// Chunk stream: chunk c = K-block (c % 4) of A image (c / 4); buffer c % 2.
__device__ __forceinline__ void issue_chunk(Pipe &p, float *abuf, const float *img_slot, int c) {
    bulk_load(abuf + (c & 1) * CHUNK, img_slot + (c >> 2) * (2 * TS * TS) + (c & 3) * CHUNK,
              CHUNK * sizeof(float), &p.full[c & 1]);
}

// One product: chunks [c_begin, c_begin + 4) against the B image, into d_tmem.
// Thread 0 only.  Keeps the next chunk's copy in flight behind the MMAs.
template <bool NEG>
__device__ __forceinline__ void run_product(Pipe &p, float *abuf, const float *Bhi, const float *Blo,
                                            const float *img_slot, int c_begin, int c_total,
                                            uint32_t d_tmem, bool accumulate) {
    for (int kb = 0; kb < 4; ++kb) {
        const int c = c_begin + kb;
        tc::mbar_wait(&p.full[c & 1], (c >> 1) & 1);
        tc::fence_after();
        const float *a = abuf + (c & 1) * CHUNK;
        tc::mma3_kblock<TS, BN, NEG>(d_tmem, tc::smem_u32(a), tc::smem_u32(a + TS * 32),
                                     tc::smem_u32(Bhi + kb * BN * 32), tc::smem_u32(Blo + kb * BN * 32),
                                     accumulate || kb > 0);
        tc::commit(&p.free_[c & 1]);
        // refill the other buffer (chunk c - 1's) with chunk c + 1
        if (c >= 1 && c + 1 < c_total) {
            tc::mbar_wait(&p.free_[(c - 1) & 1], ((c - 1) >> 1) & 1);
            issue_chunk(p, abuf, img_slot, c + 1);
        }
    }
}

// TMEM columns [col, col + BN) of the thread's row -> hi/lo B image (K index = row)
__device__ __forceinline__ void tmem_to_b(uint32_t tbase, int col, int row, int half, float *Bhi,
                                          float *Blo) {
    const uint32_t lane = (uint32_t)(threadIdx.x & 96) << 16;
    for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 16) {
        float v[16];
        tc::tmem_ld16(tbase + lane + col + c0, v);
        put_b16(Bhi, Blo, c0, row, v);
    }
}

}  // namespace tcapply

using namespace tcapply;

// Leaf level: grid (column blocks, m tile rows, batch).
template <typename S>
__global__ void __launch_bounds__(tcapply::NT, 1) k_apply_leaf_tc(tcapply::View<S> V, int64_t top,
                                                                  int64_t cbase, const float *img,
                                                                  int64_t img_bstride, int64_t a_bstride) {
    extern __shared__ unsigned char smraw[];
    float *sm = (float *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    float *abuf = sm, *Bhi = sm + 2 * CHUNK, *Blo = Bhi + BIMG;
    __shared__ Pipe p;
    const int tid = threadIdx.x, warp = tid >> 5, row = tid & 127, half = tid >> 7;
    const int64_t b = blockIdx.z, l = blockIdx.y;
    V.base += b * a_bstride;
    const float *slot = img + b * img_bstride + l * 6 * (int64_t)TS * TS;
    const int64_t r0 = (top + l) * TS, c0 = cbase + (int64_t)blockIdx.x * BN;
    if (warp == 0) tc::tmem_alloc<256>(&p.tslot);
    if (tid == 32) {
        tc::mbar_init(&p.full[0], 1);
        tc::mbar_init(&p.full[1], 1);
        tc::mbar_init(&p.free_[0], 1);
        tc::mbar_init(&p.free_[1], 1);
        tc::mbar_init(&p.done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tW = p.tslot, tX = p.tslot + BN;
    if (tid == 0) {
        issue_chunk(p, abuf, slot, 0);
        issue_chunk(p, abuf, slot, 1);
    }
    // X -> the hi/lo B image.  Every product accumulates from zero in TMEM
    // and X - U W is formed in fp32 (round to nearest) on the CUDA cores:
    // accumulating onto X inside the MMA pipe biased the update (error
    // ~1e-4 of sigma_max at n = 8192 against 2e-7 for the FMA path).
    const uint32_t lane = (uint32_t)(warp & 3) * 32 << 16;
    for (int cc = half * (BN / 2); cc < (half + 1) * (BN / 2); cc += 16) {
        float v[16];
        load_row16(V, r0 + row, c0 + cc, v);
        put_b16(Bhi, Blo, cc, row, v);
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
        tc::fence_after();
        run_product<false>(p, abuf, Bhi, Blo, slot, 0, 8, tW, false);      // W = V^T X
        tc::commit(&p.done);
    }
    tc::mbar_wait(&p.done, 0);
    tc::fence_after();
    tmem_to_b(tW, 0, row, half, Bhi, Blo);                                   // W -> B image
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
        tc::fence_after();
        run_product<true>(p, abuf, Bhi, Blo, slot, 4, 8, tX, false);        // P = -U W
        tc::commit(&p.done);
    }
    tc::mbar_wait(&p.done, 1);
    tc::fence_after();
    for (int cc = half * (BN / 2); cc < (half + 1) * (BN / 2); cc += 16) {
        float v[16], x[16];
        tc::tmem_ld16(tX + lane + cc, v);
        load_row16(V, r0 + row, c0 + cc, x);                 // L2-resident re-read
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] += x[q];
        store_row16(V, r0 + row, c0 + cc, v);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<256>(p.tslot);
}

// Tree level j: grid (column blocks, node pairs, batch); node (j, p) combines
// tile rows a = (2p) << (j-1) (top) and bb = (2p+1) << (j-1) (bottom).
template <typename S>
__global__ void __launch_bounds__(tcapply::NT, 1) k_apply_tt_tc(tcapply::View<S> V, int64_t top,
                                                                int64_t cbase, const float *img,
                                                                int64_t slot0, int j, int64_t img_bstride,
                                                                int64_t a_bstride) {
    extern __shared__ unsigned char smraw[];
    float *sm = (float *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    float *abuf = sm, *Bhi = sm + 2 * CHUNK, *Blo = Bhi + BIMG;
    __shared__ Pipe p;
    const int tid = threadIdx.x, warp = tid >> 5, row = tid & 127, half = tid >> 7;
    const int64_t b = blockIdx.z, pr = blockIdx.y;
    V.base += b * a_bstride;
    const float *slot = img + b * img_bstride + (slot0 + pr) * 6 * (int64_t)TS * TS;
    const int64_t rt = (top + ((2 * pr) << (j - 1))) * TS, rb = (top + ((2 * pr + 1) << (j - 1))) * TS;
    const int64_t c0 = cbase + (int64_t)blockIdx.x * BN;
    if (warp == 0) tc::tmem_alloc<512>(&p.tslot);
    if (tid == 32) {
        tc::mbar_init(&p.full[0], 1);
        tc::mbar_init(&p.full[1], 1);
        tc::mbar_init(&p.free_[0], 1);
        tc::mbar_init(&p.free_[1], 1);
        tc::mbar_init(&p.done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tW = p.tslot, tXt = p.tslot + BN, tXb = p.tslot + 2 * BN;
    if (tid == 0) {
        issue_chunk(p, abuf, slot, 0);
        issue_chunk(p, abuf, slot, 1);
    }
    const uint32_t lane = (uint32_t)(warp & 3) * 32 << 16;
    for (int cc = half * (BN / 2); cc < (half + 1) * (BN / 2); cc += 16) {
        float v[16];
        load_row16(V, rb + row, c0 + cc, v);                    // X_bot: B image
        put_b16(Bhi, Blo, cc, row, v);
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
        tc::fence_after();
        run_product<false>(p, abuf, Bhi, Blo, slot, 0, 12, tW, false);     // Vb^T X_bot
        tc::commit(&p.done);
    }
    tc::mbar_wait(&p.done, 0);
    tc::fence_after();
    for (int c0w = half * (BN / 2); c0w < (half + 1) * (BN / 2); c0w += 16) {   // W = X_top + Vb^T X_bot
        float v[16], x[16];
        tc::tmem_ld16(tW + lane + c0w, v);
        load_row16(V, rt + row, c0 + c0w, x);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] += x[q];
        put_b16(Bhi, Blo, c0w, row, v);
    }
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
        tc::fence_after();
        run_product<true>(p, abuf, Bhi, Blo, slot, 4, 12, tXt, false);     // -T^T W
        run_product<true>(p, abuf, Bhi, Blo, slot, 8, 12, tXb, false);     // -U W
        tc::commit(&p.done);
    }
    tc::mbar_wait(&p.done, 1);
    tc::fence_after();
    for (int cc = half * (BN / 2); cc < (half + 1) * (BN / 2); cc += 16) {
        float v[16], x[16];
        tc::tmem_ld16(tXt + lane + cc, v);
        load_row16(V, rt + row, c0 + cc, x);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] += x[q];
        store_row16(V, rt + row, c0 + cc, v);
        tc::tmem_ld16(tXb + lane + cc, v);
        load_row16(V, rb + row, c0 + cc, x);
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] += x[q];
        store_row16(V, rb + row, c0 + cc, v);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(p.tslot);
}

// Host: one tree level (0 = leaves) of one sweep side on the tensor cores.
template <typename S>
cudaError_t launch_apply_level_tc(S *a, int64_t n, int64_t batch, int64_t a_bstride, bool lq, int64_t top,
                                  int64_t k, int64_t m, const float *img, int64_t img_bstride, int j,
                                  cudaStream_t st) {
    const int64_t ncols = (n / TS - 1 - k) * TS;
    if (ncols <= 0) return cudaSuccess;
    tcapply::View<S> V{a, lq ? n : 1, lq ? 1 : n};
    const int64_t cbase = (k + 1) * TS;
    const unsigned gx = (unsigned)(ncols / BN);
    cudaError_t e;
    if ((e = ensure_smem(k_apply_leaf_tc<S>, SMEM)) != cudaSuccess) return e;
    if ((e = ensure_smem(k_apply_tt_tc<S>, SMEM)) != cudaSuccess) return e;
    if (j == 0) {
        k_apply_leaf_tc<S><<<dim3(gx, (unsigned)m, (unsigned)batch), NT, SMEM, st>>>(V, top, cbase, img,
                                                                                     img_bstride, a_bstride);
        bsvd_host::count_launch();
        return cudaGetLastError();
    }
    int64_t off = 0, cnt_prev = m;
    for (int q = 1; q < j; ++q) {
        off += cnt_prev;
        cnt_prev = (m + ((int64_t)1 << q) - 1) >> q;
    }
    off += cnt_prev;                                     // tree_offset(m, j)
    const int64_t pairs = cnt_prev / 2;
    if (pairs <= 0) return cudaSuccess;
    k_apply_tt_tc<S><<<dim3(gx, (unsigned)pairs, (unsigned)batch), NT, SMEM, st>>>(V, top, cbase, img, off, j,
                                                                                   img_bstride, a_bstride);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

template cudaError_t launch_apply_level_tc<float>(float *, int64_t, int64_t, int64_t, bool, int64_t, int64_t,
                                                  int64_t, const float *, int64_t, int, cudaStream_t);
template cudaError_t launch_apply_level_tc<__half>(__half *, int64_t, int64_t, int64_t, bool, int64_t,
                                                   int64_t, int64_t, const float *, int64_t, int, cudaStream_t);

}  // namespace bsvd
