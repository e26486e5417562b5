// stage1_apply.cu -- WY trailing updates of the tree stage 1, one launch per
// tree level (the reference's UNMQR / TSMQR, kernels.py:364-421, in
// compact-WY form):
//
//   leaf level  (every panel tile row l, in parallel):
//       W = V_l^T X_l ;  X_l -= U_l W                      (U = V T^T)
//   tree level j (every node with two children, in parallel):
//       W = X_top + Vb^T X_bot ;  X_top -= T^T W ;  X_bot -= U W
//
// Grid = (column blocks) x (tile rows or node pairs) x (batch): thousands of
// CTAs per launch instead of one CTA per column block walking the tree.
// Each product is a BM x BN x K (= ts x BN x ts) register-blocked FMA GEMM:
// the ts x ts operand is streamed through shared memory in K-chunks with
// cp.async double buffering, the X / W tiles sit in shared memory, and the
// warp layout (4 x 8 or 8 x 4 lanes, 8x4 / 4x4 per thread) keeps shared
// traffic at <= 3 wavefronts per 32-lane FMA instruction group.
#include "common.cuh"
#include "kernels.cuh"

namespace bsvd {

namespace apply {

constexpr int kNT = 256;

// Geometry per (compute type, ts).  BM = ts rows, BN columns per CTA.
template <typename C, int TS> struct Geo;
// fp32 / fp16-storage: 16 KiB... 32 KiB tiles, 8x4 per thread
template <int TS> struct Geo<float, TS> {
    static constexpr int BM = TS;
    static constexpr int BN = 8192 / TS;               // ts*BN = 8192 elements
    static constexpr int WGM = TS >= 128 ? 4 : (TS >= 64 ? 2 : 1);
    static constexpr int WGN = 8 / WGM;
    static constexpr int LM = TS >= 32 ? 4 : 2;
    static constexpr int LN = 32 / LM;
    static constexpr int MR = BM / (WGM * LM);
    static constexpr int NR = BN / (WGN * LN);
    static constexpr int KC = 32;
    // balanced rows: warp row wm owns the 16-row half-blocks wm and 7 - wm,
    // so a triangular operand gives every warp the same number of nonzero
    // K-chunks (each warp's two halves skip independently)
    static constexpr bool BAL = (TS == 128);
};
template <int TS> struct Geo<double, TS> {
    static constexpr int BM = TS;
    static constexpr int BN = 4096 / TS;
    static constexpr int WGM = TS >= 128 ? 4 : (TS >= 64 ? 2 : 1);
    static constexpr int WGN = 8 / WGM;
    static constexpr int LM = TS >= 32 ? 8 : 4;
    static constexpr int LN = 32 / LM;
    static constexpr int MR = BM / (WGM * LM);
    static constexpr int NR = BN / (WGN * LN);
    static constexpr int KC = 16;
    static constexpr bool BAL = false;
};

template <typename C> struct Vec;
template <> struct Vec<float> { using t4 = float4; };
template <> struct Vec<double> { using t4 = double2; };   // 16-byte granule

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Thread's microtile coordinates: rows m0.. (first half of the microtile)
// and m1.. (second half), columns n0..
template <typename G>
struct Lane {
    int m0, m1, n0, wm;
    __device__ Lane() {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        wm = warp % G::WGM;
        const int wn = warp / G::WGM;
        const int lm = lane % G::LM, ln = lane / G::LM;
        if constexpr (G::BAL) {
            constexpr int HB = G::BM / (2 * G::WGM);        // half-block rows
            m0 = wm * HB + lm * (G::MR / 2);
            m1 = (2 * G::WGM - 1 - wm) * HB + lm * (G::MR / 2);
        } else {
            m0 = wm * (G::BM / G::WGM) + lm * G::MR;
            m1 = m0 + G::MR / 2;
        }
        n0 = wn * (G::BN / G::WGN) + ln * G::NR;
    }
    __device__ __forceinline__ int row(int i) const { return i < G::MR / 2 ? m0 + i : m1 + (i - G::MR / 2); }
};

// acc[i][j] += sign * sum_k A[k][m0+i] * Bs[k][n0+j]; A global [TS][TS] streamed
// in KC-row chunks through Abuf (2 x KC x TS), Bs shared [TS][BNP].
// TRI: structure of the A operand A(k, m) = Ag[k][m] -- 0 dense, 1 zero for
// k > m, 2 zero for k < m (the triangular reflector factors).  When a K-chunk
// lines up with a warp's row block, warps skip the chunks that are entirely
// zero for their rows (the CTA still walks every chunk for the buffer sync).
template <typename C, int TS, typename G, bool NEG, int BNP, int TRI = 0>
__device__ __forceinline__ void gemm(const C *__restrict__ Ag, const C *Bs, C *Abuf,
                                     C (&acc)[G::MR][G::NR], const Lane<G> &ln) {
    constexpr int bnp = BNP;
    constexpr int KC = (G::KC < TS) ? G::KC : TS;
    constexpr int NCH = TS / KC;
    constexpr int CH = KC * TS;                       // elements per chunk
    constexpr int PER16 = 16 / (int)sizeof(C);        // elements per 16 B
    constexpr int NV = CH / PER16;                    // 16 B granules per chunk
    // Triangular operands on the balanced layout: chunk ch holds the
    // interleaved rows k = NCH i + ch, so every chunk has the same zero profile
    // and each warp skips the same share of every chunk (contiguous chunks
    // leave the barrier waiting on the warp whose rows are all nonzero there).
    constexpr bool ILV = TRI != 0 && G::BAL && KC == 32 && NCH == 4;
    auto issue = [&](int ch) {
        C *dst = Abuf + (ch & 1) * CH;
        if constexpr (ILV) {
            constexpr int GR = TS / PER16;                // granules per row
            for (int v = threadIdx.x; v < NV; v += kNT) {
                const int i = v / GR, gc = v % GR;
                cp_async16(dst + i * TS + gc * PER16, Ag + (size_t)(NCH * i + ch) * TS + gc * PER16);
            }
        } else {
            const C *src = Ag + (size_t)ch * CH;
            for (int v = threadIdx.x; v < NV; v += kNT) cp_async16(dst + v * PER16, src + v * PER16);
        }
        cp_async_commit();
    };
    issue(0);
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
        if (ch + 1 < NCH) {
            issue(ch + 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const C *As = Abuf + (ch & 1) * CH;
        constexpr int H = G::MR / 2;
        if constexpr (ILV) {
            // i ranges (k = NCH i + ch) where each half-block of rows is nonzero
            constexpr int HB = G::BM / (2 * G::WGM);
            const int ha = ln.wm, hb = 2 * G::WGM - 1 - ln.wm;
            auto cnt_le = [&](int kmax) { return kmax < ch ? 0 : min(KC, (kmax - ch) / NCH + 1); };   // #{i: k <= kmax}
            auto cnt_lt = [&](int kmin) { return kmin <= ch ? 0 : min(KC, (kmin - ch + NCH - 1) / NCH); };   // #{i: k < kmin}
            int alo = 0, ahi = KC, blo = 0, bhi = KC;
            if constexpr (TRI == 1) { ahi = cnt_le(HB * ha + HB - 1); bhi = cnt_le(HB * hb + HB - 1); }
            else { alo = cnt_lt(HB * ha); blo = cnt_lt(HB * hb); }
            const int b0 = max(alo, blo), b1 = min(ahi, bhi);
            auto full = [&](int i0, int i1) {
#pragma unroll 4
                for (int i = i0; i < i1; ++i) {
                    const int k = NCH * i + ch;
                    C a[G::MR], b[G::NR];
#pragma unroll
                    for (int t = 0; t < H; ++t) a[t] = As[i * TS + ln.m0 + t];
#pragma unroll
                    for (int t = 0; t < H; ++t) a[H + t] = As[i * TS + ln.m1 + t];
#pragma unroll
                    for (int j = 0; j < G::NR; ++j) b[j] = Bs[(size_t)k * bnp + ln.n0 + j];
#pragma unroll
                    for (int t = 0; t < G::MR; ++t)
#pragma unroll
                        for (int j = 0; j < G::NR; ++j) {
                            if (NEG) acc[t][j] -= a[t] * b[j];
                            else acc[t][j] += a[t] * b[j];
                        }
                }
            };
            auto half = [&](bool second, int i0, int i1) {
                const int mh = second ? ln.m1 : ln.m0;
#pragma unroll 4
                for (int i = i0; i < i1; ++i) {
                    const int k = NCH * i + ch;
                    C a[H], b[G::NR];
#pragma unroll
                    for (int t = 0; t < H; ++t) a[t] = As[i * TS + mh + t];
#pragma unroll
                    for (int j = 0; j < G::NR; ++j) b[j] = Bs[(size_t)k * bnp + ln.n0 + j];
                    if (second) {
#pragma unroll
                        for (int t = 0; t < H; ++t)
#pragma unroll
                            for (int j = 0; j < G::NR; ++j) {
                                if (NEG) acc[H + t][j] -= a[t] * b[j];
                                else acc[H + t][j] += a[t] * b[j];
                            }
                    } else {
#pragma unroll
                        for (int t = 0; t < H; ++t)
#pragma unroll
                            for (int j = 0; j < G::NR; ++j) {
                                if (NEG) acc[t][j] -= a[t] * b[j];
                                else acc[t][j] += a[t] * b[j];
                            }
                    }
                }
            };
            if (b0 < b1) full(b0, b1);
            // the rest of each half's range (an interval sharing one end with the overlap)
            if (alo < ahi) {
                if (alo < b0) half(false, alo, min(ahi, b0));
                if (ahi > b1) half(false, max(alo, b1), ahi);
            }
            if (blo < bhi) {
                if (blo < b0) half(true, blo, min(bhi, b0));
                if (bhi > b1) half(true, max(blo, b1), bhi);
            }
            __syncthreads();   // buffer (ch & 1) is refilled by issue(ch + 2)
            continue;
        }
        const C *Bk = Bs + (size_t)ch * KC * bnp;
        bool za = false, zb = false;                      // microtile halves entirely zero
        if constexpr (TRI != 0 && G::BAL && KC == 2 * (G::BM / (2 * G::WGM))) {
            const int ha = ln.wm, hb = 2 * G::WGM - 1 - ln.wm;   // half-block indices
            za = TRI == 1 ? ch > (ha >> 1) : ch < (ha >> 1);
            zb = TRI == 1 ? ch > (hb >> 1) : ch < (hb >> 1);
        } else if constexpr (TRI != 0 && !G::BAL && KC == G::BM / G::WGM) {
            za = zb = TRI == 1 ? ch > ln.wm : ch < ln.wm;
        }
        if (!za && !zb) {
#pragma unroll 4
            for (int k = 0; k < KC; ++k) {
                C a[G::MR], b[G::NR];
#pragma unroll
                for (int i = 0; i < H; ++i) a[i] = As[k * TS + ln.m0 + i];
#pragma unroll
                for (int i = 0; i < H; ++i) a[H + i] = As[k * TS + ln.m1 + i];
#pragma unroll
                for (int j = 0; j < G::NR; ++j) b[j] = Bk[k * bnp + ln.n0 + j];
#pragma unroll
                for (int i = 0; i < G::MR; ++i)
#pragma unroll
                    for (int j = 0; j < G::NR; ++j) {
                        if (NEG) acc[i][j] -= a[i] * b[j];
                        else acc[i][j] += a[i] * b[j];
                    }
            }
        } else if (!za || !zb) {                          // one half only
            const int mh = za ? ln.m1 : ln.m0, io = za ? H : 0;
#pragma unroll 4
            for (int k = 0; k < KC; ++k) {
                C a[H], b[G::NR];
#pragma unroll
                for (int i = 0; i < H; ++i) a[i] = As[k * TS + mh + i];
#pragma unroll
                for (int j = 0; j < G::NR; ++j) b[j] = Bk[k * bnp + ln.n0 + j];
                if (za) {
#pragma unroll
                    for (int i = 0; i < H; ++i)
#pragma unroll
                        for (int j = 0; j < G::NR; ++j) {
                            if (NEG) acc[H + i][j] -= a[i] * b[j];
                            else acc[H + i][j] += a[i] * b[j];
                        }
                } else {
#pragma unroll
                    for (int i = 0; i < H; ++i)
#pragma unroll
                        for (int j = 0; j < G::NR; ++j) {
                            if (NEG) acc[i][j] -= a[i] * b[j];
                            else acc[i][j] += a[i] * b[j];
                        }
                }
                (void)io;
            }
        }
        __syncthreads();   // buffer (ch & 1) is refilled by issue(ch + 2)
    }
}

template <typename S>
struct View {
    S *base;
    int64_t rs, cs;
    __device__ __forceinline__ S *ptr(int64_t r, int64_t c) const { return base + r * rs + c * cs; }
};

// X tile (TS rows from view row r0, BN columns from view column c0, columns
// >= cmax masked) -> Xs[r][c] (row stride bnp).  fp32 full tiles: 16-byte
// loads -- along the contiguous dimension of either view (column-major RQ
// side: 8 rows of one column per thread, a full 32-byte sector; LQ side: 4
// columns of one row).
template <typename S, typename C, int TS, int BN>
__device__ __forceinline__ void load_x(const View<S> &V, int64_t r0, int64_t c0, int64_t cmax,
                                       C *Xs, int bnp) {
    using CV = Conv<S, C>;
    if constexpr (sizeof(S) == 4 && sizeof(C) == 4 && TS % 8 == 0 && BN % 4 == 0) {
        if (c0 + BN <= cmax) {
            if (V.rs == 1) {
                for (int idx = threadIdx.x; idx < (TS / 8) * BN; idx += kNT) {
                    const int c = idx % BN, u = idx / BN;
                    const float4 *p = reinterpret_cast<const float4 *>(V.ptr(r0 + 8 * u, c0 + c));
                    const float4 a = __ldcg(p), b = __ldcg(p + 1);
                    float *d = Xs + (8 * u) * bnp + c;
                    d[0] = a.x; d[bnp] = a.y; d[2 * bnp] = a.z; d[3 * bnp] = a.w;
                    d[4 * bnp] = b.x; d[5 * bnp] = b.y; d[6 * bnp] = b.z; d[7 * bnp] = b.w;
                }
            } else {
                for (int idx = threadIdx.x; idx < TS * (BN / 4); idx += kNT) {
                    const int c4 = idx % (BN / 4), r = idx / (BN / 4);
                    const float4 a = __ldcg(reinterpret_cast<const float4 *>(V.ptr(r0 + r, c0 + 4 * c4)));
                    *reinterpret_cast<float4 *>(Xs + r * bnp + 4 * c4) = a;
                }
            }
            return;
        }
    }
    for (int idx = threadIdx.x; idx < TS * BN; idx += kNT) {
        int r, c;
        if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % BN; r = idx / BN; }
        Xs[r * bnp + c] = (c0 + c < cmax) ? CV::ld(*V.ptr(r0 + r, c0 + c)) : C(0);
    }
}

// Store the thread's microtile straight from registers (fp32 full tiles:
// 16-byte stores along the contiguous dimension of the view).
template <typename S, typename C, typename G>
__device__ __forceinline__ void store_acc(const View<S> &V, int64_t r0, int64_t c0, int64_t cmax,
                                          const C (&acc)[G::MR][G::NR], const Lane<G> &ln) {
    using CV = Conv<S, C>;
    if constexpr (sizeof(S) == 4 && sizeof(C) == 4 && G::MR % 4 == 0 && G::NR % 4 == 0) {
        if (c0 + G::BN <= cmax) {
            if (V.rs == 1) {
#pragma unroll
                for (int j = 0; j < G::NR; ++j)
#pragma unroll
                    for (int i = 0; i < G::MR; i += 4)
                        __stcg(reinterpret_cast<float4 *>(V.ptr(r0 + ln.row(i), c0 + ln.n0 + j)),
                               make_float4(acc[i][j], acc[i + 1][j], acc[i + 2][j], acc[i + 3][j]));
            } else {
#pragma unroll
                for (int i = 0; i < G::MR; ++i)
#pragma unroll
                    for (int j = 0; j < G::NR; j += 4)
                        __stcg(reinterpret_cast<float4 *>(V.ptr(r0 + ln.row(i), c0 + ln.n0 + j)),
                               make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]));
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < G::MR; ++i)
#pragma unroll
        for (int j = 0; j < G::NR; ++j)
            if (c0 + ln.n0 + j < cmax) *V.ptr(r0 + ln.row(i), c0 + ln.n0 + j) = CV::st(acc[i][j]);
}

template <typename C, typename G>
__device__ __forceinline__ void init_from(C (&acc)[G::MR][G::NR], const C *Xs, int bnp,
                                          const Lane<G> &ln) {
#pragma unroll
    for (int i = 0; i < G::MR; ++i)
#pragma unroll
        for (int j = 0; j < G::NR; ++j) acc[i][j] = Xs[ln.row(i) * bnp + ln.n0 + j];
}

template <typename C, typename G>
__device__ __forceinline__ void zero(C (&acc)[G::MR][G::NR]) {
#pragma unroll
    for (int i = 0; i < G::MR; ++i)
#pragma unroll
        for (int j = 0; j < G::NR; ++j) acc[i][j] = C(0);
}

template <typename C, typename G>
__device__ __forceinline__ void to_smem(const C (&acc)[G::MR][G::NR], C *Ws, int bnp,
                                        const Lane<G> &ln) {
#pragma unroll
    for (int i = 0; i < G::MR; ++i)
#pragma unroll
        for (int j = 0; j < G::NR; ++j) Ws[ln.row(i) * bnp + ln.n0 + j] = acc[i][j];
}

}  // namespace apply

using namespace apply;

// Leaf level: grid (column blocks, m tile rows, batch).
template <typename S, typename C, int TS>
__global__ void __launch_bounds__(apply::kNT, 3) k_apply_leaf(View<S> V, int64_t top, int64_t cbase,
                                                           int64_t ncols, const C *nodes,
                                                           int64_t ts2x3, int64_t ws_bstride,
                                                           int64_t a_bstride) {
    using G = Geo<C, TS>;
    constexpr int BNP = G::BN + 16 / (int)sizeof(C);
    constexpr int KC = (G::KC < TS) ? G::KC : TS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *Abuf = (C *)smem_raw;
    C *Xs = Abuf + 2 * KC * TS;                  // X, then W (one tile: 3 CTAs/SM)
    const int64_t b = blockIdx.z, l = blockIdx.y;
    V.base += b * a_bstride;
    nodes += b * ws_bstride;
    const C *Vk = nodes + l * ts2x3, *Um = Vk + (int64_t)TS * TS;
    const int64_t c0 = cbase + (int64_t)blockIdx.x * G::BN, cmax = cbase + ncols;
    const int64_t r0 = (top + l) * TS;
    const Lane<G> ln;
    load_x<S, C, TS, G::BN>(V, r0, c0, cmax, Xs, BNP);
    __syncthreads();
    C acc[G::MR][G::NR];
    zero<C, G>(acc);
    gemm<C, TS, G, false, BNP, 2>(Vk, Xs, Abuf, acc, ln);   // W = V^T X (ends on a barrier)
    C xr[G::MR][G::NR];
    init_from<C, G>(xr, Xs, BNP, ln);                       // the thread's X microtile
    __syncthreads();                                        // every X read before W lands
    to_smem<C, G>(acc, Xs, BNP, ln);
#pragma unroll
    for (int i = 0; i < G::MR; ++i)
#pragma unroll
        for (int j = 0; j < G::NR; ++j) acc[i][j] = xr[i][j];
    __syncthreads();
    gemm<C, TS, G, true, BNP>(Um, Xs, Abuf, acc, ln);       // X -= U W
    store_acc<S, C, G>(V, r0, c0, cmax, acc, ln);
}

// Tree level j: grid (column blocks, node pairs, batch).  Node (j, p) combines
// leaves a = (2p) << (j-1) (top) and bb = (2p+1) << (j-1) (bottom); its
// reflector slot is slot0 + p.
template <typename S, typename C, int TS>
__global__ void __launch_bounds__(apply::kNT) k_apply_tt(View<S> V, int64_t top, int64_t cbase,
                                                         int64_t ncols, const C *nodes,
                                                         int64_t ts2x3, int64_t slot0, int j,
                                                         int64_t ws_bstride, int64_t a_bstride,
                                                         int lstride) {
    using G = Geo<C, TS>;
    constexpr int BNP = G::BN + 16 / (int)sizeof(C);
    constexpr int KC = (G::KC < TS) ? G::KC : TS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *Abuf = (C *)smem_raw;
    C *Xt = Abuf + 2 * KC * TS;
    C *Xb = Xt + TS * BNP;
    const int64_t b = blockIdx.z, p = blockIdx.y;
    V.base += b * a_bstride;
    nodes += b * ws_bstride;
    const C *Vk = nodes + (slot0 + p) * ts2x3, *Um = Vk + (int64_t)TS * TS, *Tt = Um + (int64_t)TS * TS;
    const int64_t c0 = cbase + (int64_t)blockIdx.x * G::BN, cmax = cbase + ncols;
    const int64_t rt = (top + lstride * ((2 * p) << (j - 1))) * TS;
    const int64_t rb = (top + lstride * ((2 * p + 1) << (j - 1))) * TS;
    const Lane<G> ln;
    load_x<S, C, TS, G::BN>(V, rt, c0, cmax, Xt, BNP);
    load_x<S, C, TS, G::BN>(V, rb, c0, cmax, Xb, BNP);
    __syncthreads();
    // X_top's microtile stays in registers, so its shared buffer carries W
    // and then W2 (two tiles of shared memory instead of three: 2 CTAs/SM)
    C xt[G::MR][G::NR], acc[G::MR][G::NR];
    init_from<C, G>(xt, Xt, BNP, ln);
#pragma unroll
    for (int i = 0; i < G::MR; ++i)
#pragma unroll
        for (int jx = 0; jx < G::NR; ++jx) acc[i][jx] = xt[i][jx];
    gemm<C, TS, G, false, BNP, 1>(Vk, Xb, Abuf, acc, ln);   // W = X_top + Vb^T X_bot (Vb upper)
    to_smem<C, G>(acc, Xt, BNP, ln);                        // (gemm ended on a barrier)
    __syncthreads();
    zero<C, G>(acc);
    gemm<C, TS, G, false, BNP, 1>(Tt, Xt, Abuf, acc, ln);   // W2 = T^T W (T upper)
#pragma unroll
    for (int i = 0; i < G::MR; ++i)
#pragma unroll
        for (int jx = 0; jx < G::NR; ++jx) xt[i][jx] -= acc[i][jx];
    store_acc<S, C, G>(V, rt, c0, cmax, xt, ln);            // X_top -= W2
    to_smem<C, G>(acc, Xt, BNP, ln);                        // W2 (gemm ended on a barrier)
    __syncthreads();
    init_from<C, G>(acc, Xb, BNP, ln);
    gemm<C, TS, G, true, BNP, 2>(Um, Xt, Abuf, acc, ln);    // X_bot -= Vb W2 (Um = Vb^T layout)
    store_acc<S, C, G>(V, rb, c0, cmax, acc, ln);
}

// Two-tile leaves (stage1_tree.cu k_panel_leaf2): grid (column blocks,
// super-leaves, batch).  V = [V1; V2] (V1 unit lower, V2 dense), U = [U1; U2]:
//   W = V1^T X1 + V2^T X2 ;  X1 -= U1 W ;  X2 -= U2 W
// (the second tile absent past the panel's end).  X1's tile carries W once
// X1's microtile is in registers: two shared tiles, 2 CTAs/SM.
template <typename S, typename C, int TS>
__global__ void __launch_bounds__(apply::kNT, 2) k_apply_leaf2(View<S> V, int64_t top, int64_t m,
                                                              int64_t cbase, int64_t ncols, const C *nodes,
                                                              const C *ext, int64_t ts2x3,
                                                              int64_t ws_bstride, int64_t a_bstride) {
    using G = Geo<C, TS>;
    constexpr int BNP = G::BN + 16 / (int)sizeof(C);
    constexpr int KC = (G::KC < TS) ? G::KC : TS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *Abuf = (C *)smem_raw;
    C *X1 = Abuf + 2 * KC * TS;
    C *X2 = X1 + TS * BNP;
    const int64_t b = blockIdx.z, l = blockIdx.y;
    const int64_t ts2 = (int64_t)TS * TS;
    V.base += b * a_bstride;
    nodes += b * ws_bstride;
    ext += b * ws_bstride;
    const C *Vk = nodes + l * ts2x3, *Um = Vk + ts2;
    const C *V2 = ext + l * 2 * ts2, *U2 = V2 + ts2;
    const int64_t c0 = cbase + (int64_t)blockIdx.x * G::BN, cmax = cbase + ncols;
    const int64_t r1 = (top + 2 * l) * TS, r2 = r1 + TS;
    const bool two = 2 * l + 1 < m;
    const Lane<G> ln;
    load_x<S, C, TS, G::BN>(V, r1, c0, cmax, X1, BNP);
    if (two) load_x<S, C, TS, G::BN>(V, r2, c0, cmax, X2, BNP);
    __syncthreads();
    C acc[G::MR][G::NR];
    zero<C, G>(acc);
    gemm<C, TS, G, false, BNP, 2>(Vk, X1, Abuf, acc, ln);      // V1^T X1 (V1 unit lower)
    if (two) gemm<C, TS, G, false, BNP>(V2, X2, Abuf, acc, ln);   // + V2^T X2
    C xr[G::MR][G::NR];
    init_from<C, G>(xr, X1, BNP, ln);
    __syncthreads();
    to_smem<C, G>(acc, X1, BNP, ln);                           // W
#pragma unroll
    for (int i = 0; i < G::MR; ++i)
#pragma unroll
        for (int jx = 0; jx < G::NR; ++jx) acc[i][jx] = xr[i][jx];
    __syncthreads();
    gemm<C, TS, G, true, BNP>(Um, X1, Abuf, acc, ln);          // X1 -= U1 W
    store_acc<S, C, G>(V, r1, c0, cmax, acc, ln);
    if (two) {
        init_from<C, G>(acc, X2, BNP, ln);
        gemm<C, TS, G, true, BNP>(U2, X1, Abuf, acc, ln);      // X2 -= U2 W
        store_acc<S, C, G>(V, r2, c0, cmax, acc, ln);
    }
}

template <typename C, int TS>
size_t apply_smem(bool tt) {
    using G = Geo<C, TS>;
    constexpr int BNP = G::BN + 16 / (int)sizeof(C);
    constexpr int KC = (G::KC < TS) ? G::KC : TS;
    return (size_t)(2 * KC * TS + (tt ? 2 : 1) * TS * BNP) * sizeof(C);
}

// Host side: one launch for the leaves, one per tree level.
template <typename S, typename C, int TS>
cudaError_t launch_apply_levels(S *a, int64_t n, int64_t batch, int64_t a_bstride, bool lq,
                                int64_t top, int64_t k, int64_t m, const C *nodes,
                                int64_t ws_bstride, cudaStream_t st) {
    using G = Geo<C, TS>;
    const int64_t ncols = (n / TS - 1 - k) * TS;
    if (ncols <= 0) return cudaSuccess;
    View<S> V{a, lq ? n : 1, lq ? 1 : n};
    const int64_t cbase = (k + 1) * TS;
    const int64_t ts2x3 = 3 * (int64_t)TS * TS;
    const unsigned gx = (unsigned)((ncols + G::BN - 1) / G::BN);
    const size_t sl = apply_smem<C, TS>(false), stt = apply_smem<C, TS>(true);
    cudaError_t e;
    if ((e = ensure_smem(k_apply_leaf<S, C, TS>, sl)) != cudaSuccess) return e;
    if ((e = ensure_smem(k_apply_tt<S, C, TS>, stt)) != cudaSuccess) return e;
    k_apply_leaf<S, C, TS><<<dim3(gx, (unsigned)m, (unsigned)batch), apply::kNT, sl, st>>>(
        V, top, cbase, ncols, nodes, ts2x3, ws_bstride, a_bstride);
    bsvd_host::count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // tree levels: count(j) = ceil(m / 2^j); node (j, p) has two children iff 2p+1 < count(j-1)
    int64_t off = 0, cnt_prev = m;
    for (int j = 1; ((int64_t)1 << (j - 1)) < m; ++j) {
        off += cnt_prev;                                   // tree_offset(m, j)
        const int64_t cnt = (m + ((int64_t)1 << j) - 1) >> j;
        const int64_t pairs = cnt_prev / 2;                // nodes with a right child
        if (pairs > 0) {
            k_apply_tt<S, C, TS><<<dim3(gx, (unsigned)pairs, (unsigned)batch), apply::kNT, stt, st>>>(
                V, top, cbase, ncols, nodes, ts2x3, off, j, ws_bstride, a_bstride, 1);
            bsvd_host::count_launch();
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        cnt_prev = cnt;
    }
    return cudaSuccess;
}

// One tree level only (0 = the leaves, j >= 1 = the TT nodes of level j), for
// the overlapped schedule where level j's update starts as soon as the panel
// has produced level j's reflectors.
template <typename S, typename C, int TS>
cudaError_t launch_apply_level(S *a, int64_t n, int64_t batch, int64_t a_bstride, bool lq,
                               int64_t top, int64_t k, int64_t m, const C *nodes,
                               int64_t ws_bstride, int j, cudaStream_t st, const C *ext,
                               int64_t mtiles) {
    using G = Geo<C, TS>;
    const int64_t ncols = (n / TS - 1 - k) * TS;
    if (ncols <= 0) return cudaSuccess;
    View<S> V{a, lq ? n : 1, lq ? 1 : n};
    const int64_t cbase = (k + 1) * TS;
    const int64_t ts2x3 = 3 * (int64_t)TS * TS;
    const unsigned gx = (unsigned)((ncols + G::BN - 1) / G::BN);
    const size_t sl = apply_smem<C, TS>(false), stt = apply_smem<C, TS>(true);
    cudaError_t e;
    const int lstride = ext ? 2 : 1;                    // m counts two-tile leaves
    if (j == 0 && ext) {
        const size_t s2 = apply_smem<C, TS>(true);
        if ((e = ensure_smem(k_apply_leaf2<S, C, TS>, s2)) != cudaSuccess) return e;
        k_apply_leaf2<S, C, TS><<<dim3(gx, (unsigned)m, (unsigned)batch), apply::kNT, s2, st>>>(
            V, top, mtiles, cbase, ncols, nodes, ext, ts2x3, ws_bstride, a_bstride);
        bsvd_host::count_launch();
        return cudaGetLastError();
    }
    if (j == 0) {
        if ((e = ensure_smem(k_apply_leaf<S, C, TS>, sl)) != cudaSuccess) return e;
        k_apply_leaf<S, C, TS><<<dim3(gx, (unsigned)m, (unsigned)batch), apply::kNT, sl, st>>>(
            V, top, cbase, ncols, nodes, ts2x3, ws_bstride, a_bstride);
        bsvd_host::count_launch();
        return cudaGetLastError();
    }
    if ((e = ensure_smem(k_apply_tt<S, C, TS>, stt)) != cudaSuccess) return e;
    int64_t off = 0, cnt_prev = m;
    for (int q = 1; q < j; ++q) {
        off += cnt_prev;
        cnt_prev = (m + ((int64_t)1 << q) - 1) >> q;
    }
    off += cnt_prev;                                     // tree_offset(m, j)
    const int64_t pairs = cnt_prev / 2;
    if (pairs <= 0) return cudaSuccess;
    k_apply_tt<S, C, TS><<<dim3(gx, (unsigned)pairs, (unsigned)batch), apply::kNT, stt, st>>>(
        V, top, cbase, ncols, nodes, ts2x3, off, j, ws_bstride, a_bstride, lstride);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

#define INST(S, C, TS)                                                                         \
    template cudaError_t launch_apply_levels<S, C, TS>(S *, int64_t, int64_t, int64_t, bool,    \
                                                       int64_t, int64_t, int64_t, const C *,    \
                                                       int64_t, cudaStream_t);                  \
    template cudaError_t launch_apply_level<S, C, TS>(S *, int64_t, int64_t, int64_t, bool,     \
                                                      int64_t, int64_t, int64_t, const C *,     \
                                                      int64_t, int, cudaStream_t, const C *,    \
                                                      int64_t);
#define INST3(TS) INST(double, double, TS) INST(float, float, TS) INST(__half, float, TS)
INST3(16)
INST3(32)
INST3(64)
INST3(128)
#undef INST3
#undef INST

}  // namespace bsvd
