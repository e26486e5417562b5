// stage1_flat_tc.cu -- the flat stage 1's two trailing-update products on the
// 5th-generation tensor cores (tcgen05, TMEM accumulators, TMA), 3xTF32,
// ts = 128, FP32 storage:
//
//   G1:  Wp[s] = V[rows_s]^T X[rows_s]          (k_fgemm1's split-K partials)
//   G2:  X[TS:M, :] -= V[TS:M, :] W2            (k_fgemm2)
//
// (the compact-WY update of tsmqr / unmqr, kernels.py:364-421, aggregated over
// the whole panel).  One CTA per 128 x 128 output tile, warp-specialised:
//   warp 9 (one thread)   TMA: 32-wide K-blocks of both operands into a
//                         3-stage (G1) / 2-stage (G2) shared-memory ring, raw
//                         fp32 landing directly as K-major SWIZZLE_128B images;
//                         for G2 also the 128 x 128 X tile of the epilogue;
//   warps 0-7             split every staged value in place into
//                         hi = tf32(x) and lo = tf32(x - hi) (a second image),
//                         then run the epilogue;
//   warp 8 (one thread)   issues hi*hi + hi*lo + lo*hi per K = 8 step into the
//                         TMEM accumulator, returns each stage by tcgen05.commit.
// Accuracy: measured on this part (scripts/tc_acc_probe.cu) the kind::tf32
// accumulation is unbiased; 3xTF32 products carry ~2^-22 relative error.
//
// Orientation: the MMA's M dimension (TMEM lanes) runs along the matrix's
// contiguous axis in G2's epilogue, so its X read-modify-write is coalesced on
// both sweep sides:
//   G2, RQ (rows contiguous): D[r][c] = sum_j Vrm[r][j] W2T[c][j]
//   G2, LQ (cols contiguous): D[c][r] = sum_j W2T[c][j] Vrm[r][j]
//   G1:                       D[j][c] = sum_r Vcm[j][r] X(r, c)
// All operands are K-major in memory except X in G1 on the LQ side, whose raw
// [32 r][128 c] box is transposed by the split warps.
//
// FP16 storage (H): X is exactly representable in tf32 (11 significant bits),
// so its lo part is zero: X's boxes land raw (fp16, unswizzled) in the B_lo
// slot, the split warps widen them into the fp32 B_hi image, and the
// A_hi * B_lo product is skipped (two MMAs per K = 8 step instead of three);
// the X update reads and writes fp16 (round to nearest).
#include <cuda.h>
#include <stdio.h>

#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_sm100.cuh"

namespace bsvd {
namespace ftc {

constexpr int TS = 128, BM = 128, BN = 128, KB = 32;
constexpr int NSW = 8;                       // split / epilogue warps
constexpr int W_MMA = NSW, W_TMA = NSW + 1;

constexpr int IMG = BM * KB;                 // floats per operand image (one K-block, 16 KB)
constexpr int STAGE = 4 * IMG;               // A_hi, A_lo, B_hi, B_lo
// Accumulation epochs: the TMEM accumulator restarts from zero every EPK
// K-blocks and each epoch is added into fp32 registers (round to nearest) by
// the epilogue warps.  Measured: the tensor-core accumulation error of one
// element grows linearly with the accumulated K (a K = 2048 single accumulator
// gave 7e-5 sigma_max at n = 8192), so epochs are kept short; two TMEM
// accumulators alternate so the MMAs of epoch e+1 overlap the drain of e.
constexpr int EPK = 1;
constexpr int TMEM_COLS = 2 * BN;
template <int MODE>
struct Cfg {
    // G1 (MODE 1): eight more warps drain the TMEM epochs, so the split warps
    // only split and the tensor pipe is not held up by the drains
    static constexpr bool SEP = MODE == 1;
    static constexpr int NTH = (NSW + 2 + (SEP ? NSW : 0)) * 32;
    static constexpr int NST = MODE == 1 ? 3 : 2;
    static constexpr size_t XT = MODE == 2 ? (size_t)BM * BN : 0;   // X tile floats
    static constexpr size_t SMEM = ((size_t)NST * STAGE + XT) * sizeof(float) + 1024;
};

struct Maps {
    CUtensorMap Xk;     // matrix, box {32 inner, 128}, SW128 (G1, RQ: B)
    CUtensorMap Xm;     // matrix, box {128 inner, 32}, no swizzle (G1, LQ: raw B)
    CUtensorMap Xt;     // matrix, box {128, 128}, no swizzle (G2 epilogue tile)
    CUtensorMap Vcm;    // [j][n] (inner r), box {32, 128}, SW128 (G1: A)
    CUtensorMap Vrm;    // [r][128] (inner j), box {32, 128}, SW128 (G2)
    CUtensorMap W2T;    // [c][128] (inner j), box {32, 128}, SW128 (G2)
};

struct Args {
    int M, C;               // panel rows, trailing columns
    int row_base, col_base; // global (row, column) of the view's X(0, 0)
    int rps;                // G1 rows per split
    float *Wp;              // G1 output (member 0)
    float *Gp;              // G1's Gram partials [ns][TS][TS] (member 0)
    int64_t ws_bstride;     // floats
    void *X;                // G2 epilogue: matrix base (member 0), storage type
    int64_t n, a_bstride;   // G2 epilogue: leading dim, batch stride
    int no_pf;              // development: no L2 prefetch of G1's X boxes
};

__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
// L2 prefetch of one TMA box (no shared memory, no completion)
__device__ __forceinline__ void tma3_prefetch(const CUtensorMap *map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(m)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(m)) : "memory");
}
__device__ __forceinline__ void split4(float4 v, float4 &h, float4 &l) {
    tc::split3(v.x, h.x, l.x);
    tc::split3(v.y, h.y, l.y);
    tc::split3(v.z, h.z, l.z);
    tc::split3(v.w, h.w, l.w);
}
// in-place split of one image (16 KB): the layout is irrelevant, elementwise
__device__ __forceinline__ void split_image(float *hi, float *lo, int t) {
#pragma unroll
    for (int i = 0; i < IMG / 4 / (NSW * 32); ++i) {
        const int o = (t + i * NSW * 32) * 4;
        float4 h, l;
        split4(*reinterpret_cast<const float4 *>(hi + o), h, l);
        *reinterpret_cast<float4 *>(hi + o) = h;
        *reinterpret_cast<float4 *>(lo + o) = l;
    }
}

template <int MODE, bool LQ, bool H>
__global__ void __launch_bounds__(Cfg<MODE>::NTH, 1) k_tgemm(const __grid_constant__ Maps maps, const Args g) {
    using CF = Cfg<MODE>;
    constexpr bool SEP = CF::SEP;
    constexpr int NST = CF::NST;
    extern __shared__ __align__(1024) unsigned char smraw[];
    float *sm = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
    float *xt = sm + NST * STAGE;   // G2 X tile [128 outer][128 inner]
    __shared__ __align__(8) uint64_t loaded[NST], full[NST], empty[NST], accfull[2], accempty[2], xload;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int b = blockIdx.z;

    int m0 = 0, n0 = 0, k_lo = 0, nkb = TS / KB, sp = 0;
    // G1's extra column tile: G = V^T V (B = A), the Gram matrix of the panel's
    // reflectors from which k_tbuild forms T
    const bool gtile = MODE == 1 && (int)blockIdx.x == g.C / BN;
    if (MODE == 1) {
        n0 = blockIdx.x * BN;
        sp = blockIdx.y;
        k_lo = sp * g.rps;
        const int k_hi = min(g.M, k_lo + g.rps);
        nkb = k_hi > k_lo ? (k_hi - k_lo) / KB : 0;
    } else {
        m0 = LQ ? blockIdx.y * BM : TS + blockIdx.x * BM;
        n0 = LQ ? TS + blockIdx.x * BN : blockIdx.y * BN;
    }

    if (warp == W_MMA) {
        tc::tmem_alloc<TMEM_COLS>(&tslot);
        if (lane == 0) {
            for (int i = 0; i < NST; ++i) {
                tc::mbar_init(&loaded[i], 1);
                tc::mbar_init(&full[i], NSW * 32);
                tc::mbar_init(&empty[i], 1);
            }
            for (int i = 0; i < 2; ++i) {
                tc::mbar_init(&accfull[i], 1);
                tc::mbar_init(&accempty[i], NSW * 32);
            }
            tc::mbar_init(&xload, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tslot;

    if (warp == W_TMA) {
        const bool no_pf = g.no_pf != 0;
        if (lane == 0) {
            if (MODE == 2) {   // the epilogue's X tile, 64 KB, first
                // RQ: inner = rows (m), outer = cols (n); LQ: inner = cols (m), outer = rows (n)
                const int inner = (LQ ? g.col_base : g.row_base) + m0;
                const int outer = (LQ ? g.row_base : g.col_base) + n0;
                expect_tx(&xload, (uint32_t)(BM * BN * (H ? 2 : 4)));
                tma3(xt, &maps.Xt, &xload, inner, outer, b);
            }
            // G1 streams X from HBM: the smem ring (3 stages) covers less than
            // the DRAM latency at the MMA rate, so the X boxes PF K-blocks
            // ahead are prefetched into L2 first
            constexpr int PF = 8;
            auto prefetch_x = [&](int kb) {
                if (MODE != 1 || gtile || kb >= nkb) return;
                const int kk = kb * KB;
                if (!LQ) tma3_prefetch(&maps.Xk, g.row_base + k_lo + kk, g.col_base + n0, b);
                else tma3_prefetch(&maps.Xm, g.col_base + n0, g.row_base + k_lo + kk, b);
            };
            if (MODE == 1 && !no_pf)
                for (int kb = NST; kb < NST + PF; ++kb) prefetch_x(kb);
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % NST;
                if (MODE == 1 && !no_pf && kb >= NST) prefetch_x(kb + PF);
                if (kb >= NST) tc::mbar_wait(&empty[st], (uint32_t)((kb / NST - 1) & 1));
                float *base = sm + st * STAGE;
                const uint32_t bbytes = MODE == 1 && H ? IMG * 2 : IMG * 4;   // fp16 X box: half the bytes
                expect_tx(&loaded[st], (uint32_t)(IMG * 4 + (gtile ? 0 : bbytes)));
                const int kk = kb * KB;
                if (MODE == 1) {
                    tma3(base, &maps.Vcm, &loaded[st], k_lo + kk, 0, b);              // A[j][r]
                    if (gtile) {
                    } else if (!LQ)   // B[c][r]: X(r, c) at inner = row_base + r, outer = col_base + c
                        tma3(base + (H ? 3 : 2) * IMG, &maps.Xk, &loaded[st], g.row_base + k_lo + kk,
                             g.col_base + n0, b);
                    else       // raw [32 r][128 c]: inner = col_base + c, outer = row_base + r
                        tma3(base + 3 * IMG, &maps.Xm, &loaded[st], g.col_base + n0, g.row_base + k_lo + kk, b);
                } else if (!LQ) {
                    tma3(base, &maps.Vrm, &loaded[st], kk, m0, b);                     // A[r][j]
                    tma3(base + 2 * IMG, &maps.W2T, &loaded[st], kk, n0, b);           // B[c][j]
                } else {
                    tma3(base, &maps.W2T, &loaded[st], kk, m0, b);                     // A[c][j]
                    tma3(base + 2 * IMG, &maps.Vrm, &loaded[st], kk, n0, b);           // B[r][j]
                }
            }
        }
    } else if (warp == W_MMA) {
        if (lane == 0 && nkb > 0) {
            constexpr uint32_t id = tc::idesc_tf32<BM, BN, false>();
            for (int kb = 0; kb < nkb; ++kb) {
                const int st = kb % NST, ep = kb / EPK, ab = ep & 1;
                const bool first = kb % EPK == 0;
                if (first && ep >= 2) {   // accumulator ab drained (epoch ep - 2)
                    tc::mbar_wait(&accempty[ab], (uint32_t)((ep / 2 - 1) & 1));
                    tc::fence_after();
                }
                tc::mbar_wait(&full[st], (uint32_t)((kb / NST) & 1));
                tc::fence_after();
                float *base = sm + st * STAGE;
                const uint32_t ah = tc::smem_u32(base), al = tc::smem_u32(base + IMG);
                const uint32_t bh = gtile ? ah : tc::smem_u32(base + 2 * IMG);
                const uint32_t bl = gtile ? al : tc::smem_u32(base + 3 * IMG);
                const uint32_t acc = tmem + (uint32_t)(ab * BN);
                // the small cross terms first, the hi*hi products last: the
                // accumulator only reaches full magnitude for the last K/8 adds
                // (each TMEM accumulation rounds relative to the accumulator)
                const bool b_exact = MODE == 1 && H && !gtile;   // fp16 X: lo == 0
#pragma unroll
                for (int k = 0; k < KB / 8; ++k) {
                    const uint32_t o = 32u * k;
                    if (!b_exact) tc::mma_tf32(acc, tc::sdesc(ah + o), tc::sdesc(bl + o), id, !first || k > 0);
                    tc::mma_tf32(acc, tc::sdesc(al + o), tc::sdesc(bh + o), id, !b_exact || !first || k > 0);
                }
#pragma unroll
                for (int k = 0; k < KB / 8; ++k) {
                    const uint32_t o = 32u * k;
                    tc::mma_tf32(acc, tc::sdesc(ah + o), tc::sdesc(bh + o), id, true);
                }
                tc::commit(&empty[st]);
                if (kb % EPK == EPK - 1 || kb == nkb - 1) tc::commit(&accfull[ab]);
            }
        }
    } else {
        // ---------------- split warps (and, unless SEP, drain + epilogue) ----
        const int t = tid;   // 0 .. 255 for the split warps
        const int q = warp & 3;              // TMEM lane quadrant (hardware: warp % 4)
        const int chalf = SEP ? (warp - NSW - 2) >> 2 : warp >> 2;   // half of the 128 accumulator columns
        const bool splitter = warp < NSW, drainer = SEP ? warp >= NSW + 2 : true;
        const int m = q * 32 + lane;         // accumulator row
        const int nep = (nkb + EPK - 1) / EPK;
        float sum[64];
#pragma unroll
        for (int i = 0; i < 64; ++i) sum[i] = 0.f;
        int drained = 0;
        auto drain = [&](int ep) {           // add epoch ep's accumulator into sum
            const int ab = ep & 1;
            tc::mbar_wait(&accfull[ab], (uint32_t)((ep / 2) & 1));
            tc::fence_after();
#pragma unroll
            for (int c = 0; c < 64; c += 16) {
                float v[16];
                tc::tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * BN + chalf * 64 + c), v);
#pragma unroll
                for (int i = 0; i < 16; ++i) sum[c + i] += v[i];
            }
            tc::fence_before();
            mbar_arrive(&accempty[ab]);
        };
        for (int kb = 0; kb < (splitter ? nkb : 0); ++kb) {
            const int st = kb % NST;
            tc::mbar_wait(&loaded[st], (uint32_t)((kb / NST) & 1));
            float *base = sm + st * STAGE;
            split_image(base, base + IMG, t);                 // A in place
            if (gtile) {
            } else if (MODE == 1 && H) {
                // raw fp16 box in the B_lo slot -> fp32 B_hi image (exact)
                const __half *raw = reinterpret_cast<const __half *>(base + 3 * IMG);
                float4 v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ch = t + i * NSW * 32;
                    if (!LQ) {      // raw [128 c][32 r]: 4 consecutive r of one c
                        const int c = ch >> 3, r4 = (ch & 7) * 4;
                        const uint2 u = *reinterpret_cast<const uint2 *>(raw + c * KB + r4);
                        const float2 x0 = __half22float2(*reinterpret_cast<const __half2 *>(&u.x));
                        const float2 x1 = __half22float2(*reinterpret_cast<const __half2 *>(&u.y));
                        v[i] = make_float4(x0.x, x0.y, x1.x, x1.y);
                    } else {        // raw [32 r][128 c]: lanes over c
                        const int c = ch & (BN - 1), r4 = (ch >> 7) * 4;
                        const __half *rp = raw + r4 * BN + c;
                        v[i] = make_float4(__half2float(rp[0]), __half2float(rp[BN]), __half2float(rp[2 * BN]),
                                           __half2float(rp[3 * BN]));
                    }
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ch = t + i * NSW * 32;
                    const int c = LQ ? (ch & (BN - 1)) : ch >> 3, r4 = LQ ? (ch >> 7) * 4 : (ch & 7) * 4;
                    *reinterpret_cast<float4 *>(base + 2 * IMG + tc::img_off(c, r4, 0)) = v[i];
                }
            } else if (MODE == 1 && LQ) {
                // raw [32 r][128 c] in the B_lo slot -> K-major images [c][r]:
                // thread chunk = (c, 4 consecutive r); lanes run over c, so the
                // raw reads are row-contiguous and the swizzled 16-B chunk
                // writes of 8 consecutive lanes land in 8 distinct bank quads
                float4 v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ch = t + i * NSW * 32, c = ch & (BN - 1), r4 = (ch >> 7) * 4;
                    const float *raw = base + 3 * IMG + r4 * BN + c;
                    v[i] = make_float4(raw[0], raw[BN], raw[2 * BN], raw[3 * BN]);
                }
                asm volatile("bar.sync 1, %0;" ::"n"(NSW * 32) : "memory");   // all raw reads done
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int ch = t + i * NSW * 32, c = ch & (BN - 1), r4 = (ch >> 7) * 4;
                    float4 h, l;
                    split4(v[i], h, l);
                    const int o = tc::img_off(c, r4, 0);
                    *reinterpret_cast<float4 *>(base + 2 * IMG + o) = h;
                    *reinterpret_cast<float4 *>(base + 3 * IMG + o) = l;
                }
            } else {
                split_image(base + 2 * IMG, base + 3 * IMG, t);   // B in place
            }
            tc::fence_async_smem();   // generic-proxy image writes -> the MMA (async proxy)
            mbar_arrive(&full[st]);
            // drain epoch e once the first K-block of epoch e+1 is staged (the
            // MMAs keep running in the other accumulator meanwhile)
            if (!SEP && kb % EPK == 0 && kb >= EPK) drain(drained++);
        }
        if (!drainer) goto done;
        while (drained < nep) drain(drained++);
        // ---------------- epilogue (sum = the accumulated tile row m) ----------
        if (MODE == 2) tc::mbar_wait(&xload, 0);
        const int64_t wo = (int64_t)b * g.ws_bstride;
        using ST = typename std::conditional<H, __half, float>::type;
        ST *X = reinterpret_cast<ST *>(g.X) + (int64_t)b * g.a_bstride;
        const ST *xts = reinterpret_cast<const ST *>(xt);
        // G2 destination: X(lane m, column c) at X[(outer0 + c) * n + inner0 + m]
        const int64_t inner0 = (LQ ? g.col_base : g.row_base) + m0, outer0 = (LQ ? g.row_base : g.col_base) + n0;
        const int c0 = chalf * 64;
        if (MODE == 1) {
            float *dst = gtile ? g.Gp + wo + ((int64_t)sp * TS + m) * TS + c0
                               : g.Wp + wo + ((int64_t)sp * TS + m) * g.C + n0 + c0;
#pragma unroll
            for (int i = 0; i < 64; i += 4)
                *reinterpret_cast<float4 *>(dst + i) = make_float4(sum[i], sum[i + 1], sum[i + 2], sum[i + 3]);
        } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                const float x = H ? __half2float(reinterpret_cast<const __half *>(xts)[(c0 + i) * BM + m])
                                  : reinterpret_cast<const float *>(xts)[(c0 + i) * BM + m];
                const float y = x - sum[i];
                if constexpr (H)
                    X[(outer0 + c0 + i) * g.n + inner0 + m] = __float2half_rn(y);
                else
                    X[(outer0 + c0 + i) * g.n + inner0 + m] = y;
            }
        }
    }
done:
    tc::fence_before();
    __syncthreads();
    if (warp == W_MMA) tc::tmem_free<TMEM_COLS>(tmem);
}

// ---------------------------------------------------------------------------
// host: tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry
// point: no link-time libcuda dependency)
typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}
// 3-D map: dims {inner, outer, batch}, element strides of outer / batch;
// esz 4 (fp32) or 2 (fp16)
static bool make_map(CUtensorMap *m, const void *base, uint64_t inner, uint64_t outer, uint64_t batch,
                     uint64_t outer_stride, uint64_t batch_stride, uint32_t box_in, uint32_t box_out, bool sw128,
                     int esz = 4) {
    EncodeFn fn = encode_fn();
    if (!fn) return false;
    const cuuint64_t dims[3] = {inner, outer, batch};
    const cuuint64_t strides[2] = {outer_stride * esz, (batch > 1 ? batch_stride : outer_stride * outer) * esz};
    const cuuint32_t box[3] = {box_in, box_out, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
              const_cast<void *>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace ftc

bool flat_tc_supported(int ts, int elem_bytes) {
    if (const char *s = getenv("BSVD_FLAT_TC"))
        if (atoi(s) == 0) return false;
    return ts == 128 && (elem_bytes == 4 || elem_bytes == 2) && ftc::encode_fn() != nullptr;
}

struct FlatTcPlan {
    ftc::Maps maps[2];   // by V ping-pong parity
    bool half;           // FP16 storage
};

FlatTcPlan *flat_tc_plan(void *a, int elem_bytes, int64_t n, int64_t batch, int64_t a_bstride, const float *vcm0,
                         const float *vcm1, const float *vrm0, const float *vrm1, const float *w2t,
                         int64_t ws_bstride) {
    auto *p = new FlatTcPlan;
    p->half = elem_bytes == 2;
    const int es = p->half ? 2 : 4;
    bool ok = true;
    for (int par = 0; par < 2; ++par) {
        ftc::Maps &m = p->maps[par];
        // fp16 X: raw unswizzled boxes (widened by the split warps)
        ok = ok && ftc::make_map(&m.Xk, a, n, n, batch, n, a_bstride, 32, 128, !p->half, es);
        ok = ok && ftc::make_map(&m.Xm, a, n, n, batch, n, a_bstride, 128, 32, false, es);
        ok = ok && ftc::make_map(&m.Xt, a, n, n, batch, n, a_bstride, 128, 128, false, es);
        ok = ok && ftc::make_map(&m.Vcm, par ? vcm1 : vcm0, n, 128, batch, n, ws_bstride, 32, 128, true);
        ok = ok && ftc::make_map(&m.Vrm, par ? vrm1 : vrm0, 128, n, batch, 128, ws_bstride, 32, 128, true);
        ok = ok && ftc::make_map(&m.W2T, w2t, 128, n, batch, 128, ws_bstride, 32, 128, true);
    }
    if (!ok) {
        delete p;
        return nullptr;
    }
    return p;
}
void flat_tc_plan_free(FlatTcPlan *p) { delete p; }

cudaError_t launch_flat_tc(const FlatTcPlan *plan, int par, int mode, bool lq, int M, int C, int row_base,
                           int col_base, float *Wp, float *Gp, int64_t ws_bstride, int ns, int rps, void *a,
                           int64_t n, int64_t a_bstride, int64_t batch, cudaStream_t st) {
    using namespace ftc;
    static const int no_pf = getenv("BSVD_TC_NOPF") ? 1 : 0;
    Args g{M, C, row_base, col_base, rps, Wp, Gp, ws_bstride, a, n, a_bstride, no_pf};
    const Maps &maps = plan->maps[par];
    dim3 grid;
    cudaError_t e;
    if (mode == 1 || mode == 3 || mode == 4) {
        // 1: W tiles + the Gram tile; 3: the Gram tile alone (C = 0); 4: W tiles alone
        grid = dim3((unsigned)(mode == 3 ? 1 : C / BN + (mode == 1 ? 1 : 0)), (unsigned)ns, (unsigned)batch);
        if (mode == 3) g.C = 0;
        auto kern = plan->half ? (lq ? k_tgemm<1, true, true> : k_tgemm<1, false, true>)
                               : (lq ? k_tgemm<1, true, false> : k_tgemm<1, false, false>);
        if ((e = ensure_smem(kern, Cfg<1>::SMEM)) != cudaSuccess) return e;
        kern<<<grid, Cfg<1>::NTH, Cfg<1>::SMEM, st>>>(maps, g);
    } else {
        grid = dim3((unsigned)((M - TS) / BM), (unsigned)(C / BN), (unsigned)batch);
        auto kern = plan->half ? (lq ? k_tgemm<2, true, true> : k_tgemm<2, false, true>)
                               : (lq ? k_tgemm<2, true, false> : k_tgemm<2, false, false>);
        if ((e = ensure_smem(kern, Cfg<2>::SMEM)) != cudaSuccess) return e;
        kern<<<grid, Cfg<2>::NTH, Cfg<2>::SMEM, st>>>(maps, g);
    }
    bsvd_host::count_launch();
    return cudaGetLastError();
}

}  // namespace bsvd
