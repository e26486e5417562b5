// stage1_flat.cu -- stage 1 (dense -> band) as ONE flat Householder panel and
// ONE compact-WY trailing update per sweep side, fp32 compute (FP32 and FP16
// storage), ts in {64, 128}.
//
// Same sweep structure and tile operators as the reference stage 1
// (bandreduce.py:31-120 getsmqrt / banddiag; kernels.py:205-421 geqrt,
// tsqrt, unmqr, tsmqr): per sweep side (RQ on the matrix, LQ on its lazy
// transpose -- a stride swap, no copy) the panel -- view tile column k, tile
// rows top..N-1, M = (N-top)*ts rows -- is reduced to [R; 0] by ts
// Householder reflectors, and the trailing columns X (M x C) are replaced by
// Q^T X.  The reference factors the panel as a flat TSQRT chain of tile QRs
// and applies it tile by tile (4*ts flops per column per reflector,
// kernels.py:180-188); here the panel is one Householder QR of the whole
// M x ts block and the update is the aggregated compact-WY form
//     W = V^T X,  W2 = T^T W,  X -= V W2             (4*M*ts*C flops)
// -- the reference's algorithmic flop count, no tree-level
// overhead, two GEMM-shaped products per side.  The orthogonal factor is the
// panel's (unique up to signs) Householder QR; the band differs from the
// reference's tile-chain band by those signs only, the values do not.
//
// Kernels per side (streams: P = high priority panel chain, U = update):
//   k_fpanel  [P]  one thread-block cluster (<= 16 CTAs, rows split across
//                  CTAs, 512 threads each).  32-column sub-panels live in
//                  registers; per column ONE cluster-wide reduction (the dot
//                  products of the pivot column with every sub-panel column,
//                  which yield the norm, the update coefficients and the
//                  V^T v column of T at once) pushed through DSMEM; the rest
//                  of the panel gets the sub-panel's block reflector.  Writes
//                  R in place, V (fp32, row- and column-major) and tau.
//   k_fgram   [P]  G = V^T V split over rows, the last CTA merges the parts in
//                  a fixed order and builds T (recursive larft).  Overlaps
//                  k_fgemm1.
//   k_fgemm1  [U]  W_s = V[rows_s]^T X[rows_s]  (split-K partials).
//   k_fw2x1   [P]  W2 = T^T sum_s W_s; X[0:ts] -= V[0:ts] W2 -- the top tile
//                  row is the NEXT side's panel, so it is finished first
//                  (look-ahead) and the next panel starts while ...
//   k_fgemm2  [U]  X[ts:M] -= V[ts:M] W2  runs on the other stream.
// All reductions have a fixed order (deterministic, no float atomics).
#include <stdio.h>
#include <stdlib.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "panel_qr.cuh"

namespace bsvd {
namespace flat {

constexpr int NB = 32;       // sub-panel width (columns held in registers)
constexpr int kPT = 512;     // panel threads: 128 row groups x 4 column groups
constexpr int kMaxCS = 16;   // cluster size limit (non-portable)
constexpr int kGT = 256;     // GEMM threads
constexpr int KC = 16;       // GEMM k-chunk
constexpr int kMaxSplit = 16;

// ---------------------------------------------------------------------------
// storage helpers (FP16 = storage only: widen on load, round-to-nearest on store)
__device__ __forceinline__ float ldf(const float *p) { return *p; }
__device__ __forceinline__ float ldf(const __half *p) { return __half2float(*p); }
__device__ __forceinline__ void stf(float *p, float v) { *p = v; }
__device__ __forceinline__ void stf(__half *p, float v) { *p = __float2half_rn(v); }
__device__ __forceinline__ float4 ld4(const float *p) { return *reinterpret_cast<const float4 *>(p); }
__device__ __forceinline__ float4 ld4(const __half *p) {
    const uint2 u = *reinterpret_cast<const uint2 *>(p);
    const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ void st4(float *p, float4 v) { *reinterpret_cast<float4 *>(p) = v; }
__device__ __forceinline__ void st4(__half *p, float4 v) {
    __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<unsigned *>(&a);
    u.y = *reinterpret_cast<unsigned *>(&b);
    *reinterpret_cast<uint2 *>(p) = u;
}
__device__ __forceinline__ float4 f4zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ float f4get(const float4 &v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// cluster plumbing (PTX)
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_remote(uint32_t cluster_addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(cluster_addr), "f"(v) : "memory");
}

// LAPACK dlarfg convention (scale-invariant, tau = 0 for a zero tail); same
// scalar formula as the tree path's house_scalars (stage1_tree.cu).
__device__ __forceinline__ void house(float alpha, float sig, float &beta, float &tau, float &scale) {
    if (sig == 0.f) {
        beta = alpha;
        tau = 0.f;
        scale = 0.f;   // v tail is zero either way
    } else {
        beta = -copysignf(__fsqrt_rn(fmaf(alpha, alpha, sig)), alpha);
        const float d = alpha - beta;
        scale = __frcp_rn(d);
        tau = -d * __frcp_rn(beta);
    }
}

// ---------------------------------------------------------------------------
// Workspace of one matrix (floats):
//   Vrm[2][n][TS] | Vcm[2][TS][n] (leading dim n; ping-pong: the next panel writes V while the
//   previous side's k_fgemm2 still reads it) | tau[TS] | T[TS][TS] |
//   Wp[nsplit][TS][n] | W2[TS][n] | Gp[kGSplit][TS][TS] | counter
constexpr int kGSplit = 16;
struct Ws {
    float *Vrm0, *Vrm1, *Vcm0, *Vcm1, *tau, *T, *Wp, *W2, *W2T, *Gp;
    __host__ __device__ float *vrm(int par) const { return par ? Vrm1 : Vrm0; }
    int *cnt;
};
__host__ __device__ inline size_t ws_floats(int64_t n, int ts, int nsplit) {
    const size_t a = (size_t)n * ts * 4 + ts + (size_t)ts * ts + (size_t)nsplit * ts * n +
                     2 * (size_t)ts * n + (size_t)kGSplit * ts * ts + 64;
    return (a + 63) & ~(size_t)63;
}
__host__ __device__ inline Ws ws_carve(float *base, int64_t n, int ts, int nsplit) {
    Ws w;
    w.Vrm0 = base;
    w.Vrm1 = w.Vrm0 + (size_t)n * ts;
    w.Vcm0 = w.Vrm1 + (size_t)n * ts;
    w.Vcm1 = w.Vcm0 + (size_t)n * ts;
    w.tau = w.Vcm1 + (size_t)n * ts;
    w.T = w.tau + ts;
    w.Wp = w.T + (size_t)ts * ts;
    w.W2 = w.Wp + (size_t)nsplit * ts * n;
    w.W2T = w.W2 + (size_t)ts * n;
    w.Gp = w.W2T + (size_t)ts * n;
    w.cnt = (int *)(w.Gp + (size_t)kGSplit * ts * ts);
    return w;
}

// ---------------------------------------------------------------------------
// Panel.  One cluster of CS = gridDim.x CTAs per matrix (blockIdx.y = batch
// member).  CTA c owns panel rows [c*RPC, (c+1)*RPC), RPC = 128*RPT; thread
// (rg, q) -- rg = tid/4 in [0,128), q = tid%4 -- holds rows rg + 128 i
// (i < RPT) x the 8 columns q*8..q*8+7 of the current 32-column sub-panel.
template <int TS, int RPT>
struct PanelSmem {
    static constexpr int RPC = 128 * RPT;
    static constexpr int VLD = 36;   // Vs row stride: conflict-free LDS.128 for (rg, q) lanes
    static constexpr int WE = NB * (TS - NB > 0 ? TS - NB : 1);   // rest-block W elements
    // Vs [RPC][VLD] | red8 [16][8][32] | Wc [WE] | W2s [WE] | RS [WE + kMaxCS]
    static constexpr size_t floats = (size_t)RPC * VLD + 16 * 8 * 32 + 3 * WE + kMaxCS;
    static constexpr size_t dyn = floats * 4;
};

template <typename S, int TS, int RPT>
__global__ void __launch_bounds__(kPT, 1)
k_fpanel(S *__restrict__ P, int64_t rs, int64_t cs, int64_t a_bstride, int M, float *ws0,
         int64_t ws_bstride, int64_t n, int nsplit, int par) {
    using PS = PanelSmem<TS, RPT>;
    constexpr int RPC = PS::RPC, VLD = PS::VLD;
    __shared__ __align__(16) float red[16][32];
    __shared__ __align__(16) float slots[2][kMaxCS][32];
    __shared__ __align__(16) float prow_loc[32];
    __shared__ __align__(16) float prow_slot[2][32];
    __shared__ __align__(16) float fco[32];
    __shared__ float scal[2];
    __shared__ float Y[NB][NB + 1];
    __shared__ float Ts[NB][NB + 1];
    __shared__ float taus[NB];
    extern __shared__ __align__(16) float dsm[];
    float *Vs = dsm;                                  // [RPC][VLD]
    float *red8 = dsm + (size_t)RPC * VLD;           // [16 warps][8][32]
    float *Wc = red8 + 16 * 8 * 32;                  // [NB][Rc]
    float *W2s = Wc + PS::WE;
    float *RS = W2s + PS::WE;

    const int b = blockIdx.y;
    P += (int64_t)b * a_bstride;
    Ws w = ws_carve(ws0 + (int64_t)b * ws_bstride, n, TS, nsplit);
    float *Vcm = par ? w.Vcm1 : w.Vcm0;
    const int CS = gridDim.x;
    const int rank = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, rgw = lane >> 2, rg = warp * 8 + rgw;
    const int rbase = rank * RPC + rg;   // row of i = 0
    const unsigned FULL = 0xffffffffu;
    const bool lqv = (cs == 1);          // columns contiguous in memory

    auto elem = [&](int r, int c) -> S * { return P + (int64_t)r * rs + (int64_t)c * cs; };

    // rows of the 8-column group q, cols [c0, c0+8), into x[8] (0 beyond M)
    auto load8 = [&](int r, int c0, float (&x)[8]) {
        if (r >= M) {
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = 0.f;
            return;
        }
        if (lqv) {
            const float4 u = ld4(elem(r, c0)), v = ld4(elem(r, c0 + 4));
            x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w;
            x[4] = v.x; x[5] = v.y; x[6] = v.z; x[7] = v.w;
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = ldf(elem(r, c0 + c));
        }
    };

    for (int s = 0; s < TS / NB; ++s) {
        const int col0 = s * NB;
        float a[RPT][8];
#pragma unroll
        for (int i = 0; i < RPT; ++i) load8(rbase + 128 * i, col0 + q * 8, a[i]);

        // ---- 32 column steps, one cluster reduction each --------------------
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            const int jg = col0 + j;
            const int qj = j >> 3, cj = j & 7;
            const int pb = j & 1;
            const int src = (lane & ~3) | qj;
            float p[RPT];
#pragma unroll
            for (int i = 0; i < RPT; ++i) p[i] = __shfl_sync(FULL, a[i][cj], src);
            float d[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) d[c] = 0.f;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const float pm = (rbase + 128 * i > jg) ? p[i] : 0.f;
#pragma unroll
                for (int c = 0; c < 8; ++c) d[c] = fmaf(pm, a[i][c], d[c]);
            }
            // pivot row (row jg < TS <= RPC: CTA 0, i = 0, rg = jg)
            if (rank == 0 && rg == jg) {
#pragma unroll
                for (int c = 0; c < 8; ++c) prow_loc[q * 8 + c] = a[0][c];
            }
            // reduce-scatter d over the 8 row groups of the warp (lane bits 2..4)
            float e4[4], e2[2], dsum;
            {
                const bool hb = lane & 16;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float mine = hb ? d[4 + t] : d[t], oth = hb ? d[t] : d[4 + t];
                    e4[t] = mine + __shfl_xor_sync(FULL, oth, 16);
                }
                const bool mb = lane & 8;
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const float mine = mb ? e4[2 + t] : e4[t], oth = mb ? e4[t] : e4[2 + t];
                    e2[t] = mine + __shfl_xor_sync(FULL, oth, 8);
                }
                const bool lb = lane & 4;
                const float mine = lb ? e2[1] : e2[0], oth = lb ? e2[0] : e2[1];
                dsum = mine + __shfl_xor_sync(FULL, oth, 4);
            }
            red[warp][q * 8 + rgw] = dsum;   // column q*8 + rgw
            __syncthreads();
            float g = 0.f;
            if (warp == 0) {
#pragma unroll
                for (int ww = 0; ww < 16; ++ww) g += red[ww][lane];
                if (CS > 1) {
                    const uint32_t sa = smem_u32(&slots[pb][rank][lane]);
                    const uint32_t pa = smem_u32(&prow_slot[pb][lane]);
                    const float pr = prow_loc[lane];
                    for (int t = 0; t < CS; ++t) {
                        st_remote(mapa(sa, t), g);
                        if (rank == 0) st_remote(mapa(pa, t), pr);
                    }
                }
            }
            if (CS > 1) csync();
            if (warp == 0) {
                float pr;
                if (CS > 1) {
                    g = 0.f;
                    for (int t = 0; t < CS; ++t) g += slots[pb][t][lane];
                    pr = prow_slot[pb][lane];
                } else {
                    pr = prow_loc[lane];
                }
                const float sigma = __shfl_sync(FULL, g, j), alpha = __shfl_sync(FULL, pr, j);
                float beta, tau, scale;
                house(alpha, sigma, beta, tau, scale);
                const float wv = fmaf(g, scale, pr);   // v_j^T x_l (l > j) / v_l^T v_j (l < j)
                fco[lane] = lane > j ? tau * wv : 0.f;
                if (lane < j) Y[j][lane] = wv;
                if (lane == 0) {
                    scal[0] = scale;
                    scal[1] = beta;
                    taus[j] = tau;
                }
            }
            __syncthreads();
            const float scale = scal[0], beta = scal[1];
            const float4 f0 = *reinterpret_cast<const float4 *>(&fco[q * 8]);
            const float4 f1 = *reinterpret_cast<const float4 *>(&fco[q * 8 + 4]);
            const float f[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = rbase + 128 * i;
                const float v = (r > jg) ? p[i] * scale : (r == jg ? 1.f : 0.f);
#pragma unroll
                for (int c = 0; c < 8; ++c) a[i][c] = fmaf(-f[c], v, a[i][c]);
                if (q == qj) a[i][cj] = (r > jg) ? v : (r == jg ? beta : a[i][cj]);
            }
        }

        // ---- T of the sub-panel (forward larft from the V^T v columns) -----
        if (warp == 0) {
            if (lane < NB) Ts[lane][lane] = taus[lane];
            __syncwarp();
            for (int j = 1; j < NB; ++j) {
                float t = 0.f;
                if (lane < j)
                    for (int c = lane; c < j; ++c) t = fmaf(Ts[lane][c], Y[j][c], t);
                __syncwarp();
                if (lane < j) Ts[lane][j] = -taus[j] * t;
                __syncwarp();
            }
            if (rank == 0) w.tau[col0 + lane] = taus[lane];
        }

        // ---- write back: R / tails into the matrix, clean V to Vrm, Vcm, Vs --
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = rbase + 128 * i;
            const int lr = rg + 128 * i;
            float v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int cg = col0 + q * 8 + c;
                v[c] = (r > cg) ? a[i][c] : (r == cg ? 1.f : 0.f);
            }
            *reinterpret_cast<float4 *>(&Vs[lr * VLD + q * 8]) = make_float4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<float4 *>(&Vs[lr * VLD + q * 8 + 4]) = make_float4(v[4], v[5], v[6], v[7]);
            if (r < M) {
                if (lqv) {
                    st4(elem(r, col0 + q * 8), make_float4(a[i][0], a[i][1], a[i][2], a[i][3]));
                    st4(elem(r, col0 + q * 8 + 4), make_float4(a[i][4], a[i][5], a[i][6], a[i][7]));
                } else {
#pragma unroll
                    for (int c = 0; c < 8; ++c) stf(elem(r, col0 + q * 8 + c), a[i][c]);
                }
                float *vr = w.vrm(par) + (int64_t)r * TS + col0 + q * 8;
                *reinterpret_cast<float4 *>(vr) = make_float4(v[0], v[1], v[2], v[3]);
                *reinterpret_cast<float4 *>(vr + 4) = make_float4(v[4], v[5], v[6], v[7]);
#pragma unroll
                for (int c = 0; c < 8; ++c) Vcm[(int64_t)(col0 + q * 8 + c) * n + r] = v[c];
            }
        }
        __syncthreads();
        if (s == TS / NB - 1) break;

        // ---- block reflector of the sub-panel on the panel's rest columns ---
        const int rc0 = col0 + NB;             // first rest column
        const int Rc = TS - rc0;               // rest width (multiple of 32)
        // W_cta = Vs^T A_rest over this CTA's rows, 8 rest columns per chunk
        for (int cc = 0; cc < Rc / 8; ++cc) {
            float acc[8][8];   // [c' (rest col in chunk)][c (V col in group q)]
#pragma unroll
            for (int x = 0; x < 8; ++x)
#pragma unroll
                for (int c = 0; c < 8; ++c) acc[x][c] = 0.f;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = rbase + 128 * i, lr = rg + 128 * i;
                if (r < col0) continue;   // V rows above the sub-panel are zero
                const float4 v0 = *reinterpret_cast<const float4 *>(&Vs[lr * VLD + q * 8]);
                const float4 v1 = *reinterpret_cast<const float4 *>(&Vs[lr * VLD + q * 8 + 4]);
                const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                float x[8];
                load8(r, rc0 + cc * 8, x);
#pragma unroll
                for (int xx = 0; xx < 8; ++xx)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[xx][c] = fmaf(v[c], x[xx], acc[xx][c]);
            }
            // reduce-scatter over the warp's 8 row groups: lane keeps c' = rgw
            float h4[4][8], h2[2][8], h1[8];
            {
                const bool hb = lane & 16;
#pragma unroll
                for (int t = 0; t < 4; ++t)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float mine = hb ? acc[4 + t][c] : acc[t][c], oth = hb ? acc[t][c] : acc[4 + t][c];
                        h4[t][c] = mine + __shfl_xor_sync(FULL, oth, 16);
                    }
                const bool mb = lane & 8;
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float mine = mb ? h4[2 + t][c] : h4[t][c], oth = mb ? h4[t][c] : h4[2 + t][c];
                        h2[t][c] = mine + __shfl_xor_sync(FULL, oth, 8);
                    }
                const bool lb = lane & 4;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const float mine = lb ? h2[1][c] : h2[0][c], oth = lb ? h2[0][c] : h2[1][c];
                    h1[c] = mine + __shfl_xor_sync(FULL, oth, 4);
                }
            }
            float *rb = red8 + (warp * 8 + rgw) * 32 + q * 8;   // [warp][c'][c]
            *reinterpret_cast<float4 *>(rb) = make_float4(h1[0], h1[1], h1[2], h1[3]);
            *reinterpret_cast<float4 *>(rb + 4) = make_float4(h1[4], h1[5], h1[6], h1[7]);
            __syncthreads();
            if (tid < 256) {
                const int xx = tid >> 5, c = tid & 31;
                float sum = 0.f;
#pragma unroll
                for (int ww = 0; ww < 16; ++ww) sum += red8[(ww * 8 + xx) * 32 + c];
                Wc[c * Rc + cc * 8 + xx] = sum;   // Wc[c][c']
            }
            __syncthreads();
        }
        // cluster all-reduce of Wc (NB x Rc): reduce-scatter then all-gather
        if (CS > 1) {
            const int E = NB * Rc, slice = (E + CS - 1) / CS;
            for (int e = tid; e < E; e += kPT) {
                const int dst = e / slice, pos = e - dst * slice;
                st_remote(mapa(smem_u32(&RS[rank * slice + pos]), dst), Wc[e]);
            }
            csync();
            for (int pos = tid; pos < slice; pos += kPT) {
                const int e = rank * slice + pos;
                if (e < E) {
                    float sum = 0.f;
                    for (int t = 0; t < CS; ++t) sum += RS[t * slice + pos];
                    const uint32_t la = smem_u32(&Wc[e]);
                    for (int t = 0; t < CS; ++t) st_remote(mapa(la, t), sum);
                }
            }
            csync();
        }
        // W2 = Ts^T Wc  (W2[c][x] = sum_{j<=c} Ts[j][c] Wc[j][x])
        for (int e = tid; e < NB * Rc; e += kPT) {
            const int c = e / Rc, x = e - c * Rc;
            float sum = 0.f;
            for (int j = 0; j <= c; ++j) sum = fmaf(Ts[j][c], Wc[j * Rc + x], sum);
            W2s[e] = sum;
        }
        __syncthreads();
        // A_rest -= Vs W2 (own rows): thread (rg, q) sums its 8 V columns, the
        // 4 q lanes of a row reduce-scatter so lane q owns rest cols 2q, 2q+1
        for (int cc = 0; cc < Rc / 8; ++cc) {
            float wr[8][8];   // [c in group q][x in chunk]
#pragma unroll
            for (int c = 0; c < 8; ++c)
#pragma unroll
                for (int x = 0; x < 8; ++x) wr[c][x] = W2s[(q * 8 + c) * Rc + cc * 8 + x];
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int r = rbase + 128 * i, lr = rg + 128 * i;
                const float4 v0 = *reinterpret_cast<const float4 *>(&Vs[lr * VLD + q * 8]);
                const float4 v1 = *reinterpret_cast<const float4 *>(&Vs[lr * VLD + q * 8 + 4]);
                const float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                float u[8];
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    float t = 0.f;
#pragma unroll
                    for (int c = 0; c < 8; ++c) t = fmaf(v[c], wr[c][x], t);
                    u[x] = t;
                }
                // reduce-scatter over q (lane bits 0, 1)
                float u4[4], u2[2];
                const bool qb1 = lane & 2;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float mine = qb1 ? u[4 + t] : u[t], oth = qb1 ? u[t] : u[4 + t];
                    u4[t] = mine + __shfl_xor_sync(FULL, oth, 2);
                }
                const bool qb0 = lane & 1;
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const float mine = qb0 ? u4[2 + t] : u4[t], oth = qb0 ? u4[t] : u4[2 + t];
                    u2[t] = mine + __shfl_xor_sync(FULL, oth, 1);
                }
                if (r < M && r >= col0) {
                    const int x0 = rc0 + cc * 8 + q * 2;
                    S *e0 = elem(r, x0), *e1 = elem(r, x0 + 1);
                    stf(e0, ldf(e0) - u2[0]);
                    stf(e1, ldf(e1) - u2[1]);
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Panel v2.  Same row/column mapping as k_fpanel, restructured for latency:
//  * per column ONE __syncthreads: every warp sums the 16 warp partials of
//    the column dots itself and forms the reflector redundantly (no serial
//    single-warp phase and no second barrier); warp partials are double
//    buffered by column parity;
//  * the cluster exchange is one-way: warp 0 pushes its CTA's 32 partial dots
//    (rank 0 also the pivot row) into every other CTA's slot with st.async,
//    counted in bytes on the receiver's mbarrier (no cluster barrier, no L1
//    flush); every CTA sums the slots in rank order, so all CTAs form
//    bit-identical reflectors;
//  * the 32 column steps run as 4 x 8 (only the 8 columns a thread holds are
//    unrolled: the body stays in the instruction cache);
//  * the sub-panel T is built row-parallel (lane i owns row i) while the
//    other warps write the sub-panel back;
//  * the rest of the panel streams through a 3-stage cp.async ring (no
//    exposed load latency), V comes from registers, and the W = V^T A_rest
//    all-reduce is a reduce-scatter + all-gather over st.async/mbarriers.
// The panel's full T is NOT built here: k_fgemm1 forms G = V^T V as one more
// column block and its last CTA builds T (off the panel chain).
namespace p2 {
// development instrumentation (BSVD_FPANEL_TRACE): phase timestamps of CTA 0
__device__ unsigned long long *g_trace = nullptr;
__device__ __forceinline__ void stamp(int i, int who = 0) {
    if (g_trace && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == who) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_trace[i] = t;
    }
}
__device__ __forceinline__ void mbar_init(uint64_t *m, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *m, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *m, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}\n" ::"r"(smem_u32(m)),
        "r"(parity)
        : "memory");
}
// 4-byte / 16-byte remote store into CTA `rank`'s shared memory, completion
// counted on that CTA's mbarrier (same offset as `bar` locally)
__device__ __forceinline__ void put1(const float *dst_local, uint64_t *bar_local, unsigned rank, float v) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                     mapa(smem_u32(dst_local), rank)),
                 "r"(__float_as_uint(v)), "r"(mapa(smem_u32(bar_local), rank))
                 : "memory");
}
__device__ __forceinline__ void put4(const float *dst_local, uint64_t *bar_local, unsigned rank, float4 v) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     mapa(smem_u32(dst_local), rank)),
                 "r"(__float_as_uint(v.x)), "r"(__float_as_uint(v.y)), "r"(__float_as_uint(v.z)),
                 "r"(__float_as_uint(v.w)), "r"(mapa(smem_u32(bar_local), rank))
                 : "memory");
}
__device__ __forceinline__ void cp16(void *smem, const void *gmem, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Sum over the 8 lanes that differ in lane bits 2..4 (the warp's 8 row groups),
// scattered: the lane with bits (h, m, l) keeps elements h*K/2 + m*K/4 + l*K/8 + t.
template <int K>
__device__ __forceinline__ void rs8(const float (&v)[K], float (&out)[K / 8], int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    float e1[K / 2], e2[K / 4];
    const bool hb = lane & 16, mb = lane & 8, lb = lane & 4;
#pragma unroll
    for (int t = 0; t < K / 2; ++t) {
        const float mine = hb ? v[K / 2 + t] : v[t], oth = hb ? v[t] : v[K / 2 + t];
        e1[t] = mine + __shfl_xor_sync(FULL, oth, 16);
    }
#pragma unroll
    for (int t = 0; t < K / 4; ++t) {
        const float mine = mb ? e1[K / 4 + t] : e1[t], oth = mb ? e1[t] : e1[K / 4 + t];
        e2[t] = mine + __shfl_xor_sync(FULL, oth, 8);
    }
#pragma unroll
    for (int t = 0; t < K / 8; ++t) {
        const float mine = lb ? e2[K / 8 + t] : e2[t], oth = lb ? e2[t] : e2[K / 8 + t];
        out[t] = mine + __shfl_xor_sync(FULL, oth, 4);
    }
}
}  // namespace p2

template <typename S, int TS, int RPT>
struct Panel2 {
    static constexpr int RPC = 128 * RPT;
    static constexpr int XW = (RPT >= 8 && sizeof(S) == 4) ? 4 : 8;   // rest columns per staged chunk
    static constexpr int KV = XW * 8;                      // per-thread chunk partials
    static constexpr int CHB = RPC * XW * (int)sizeof(S);  // bytes per staged chunk
    static constexpr int CHF = (CHB + 15) / 16 * 4;        // in floats (16-B aligned)
    static constexpr int NST = 3;
    static constexpr int WE = NB * (TS - NB > 0 ? TS - NB : 1);
    static constexpr int R8 = 16 * XW * 33;               // red8 buffer (row stride 33)
    // ring [NST][CHF] | red8 [2][R8] | Wc [WE] (x-major [x][32]) | W2 [WE] ([x][32]) | RS [WE + 4*kMaxCS]
    static constexpr size_t floats = (size_t)NST * CHF + 2 * R8 + 3 * (size_t)WE + 4 * kMaxCS;
    static constexpr size_t dyn = floats * 4;
};

template <typename S, int TS, int RPT>
__global__ void __launch_bounds__(kPT, 1)
k_fpanel2(S *__restrict__ P, int64_t rs, int64_t cs, int64_t a_bstride, int M, float *ws0,
          int64_t ws_bstride, int64_t n, int nsplit, int par) {
    using PS = Panel2<S, TS, RPT>;
    constexpr int RPC = PS::RPC, XW = PS::XW, KV = PS::KV;
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ __align__(16) float red[2][16][32];
    __shared__ __align__(16) float slot[2][kMaxCS][32];
    __shared__ __align__(16) float pslot[2][32];
    __shared__ __align__(16) float prow[2][32];
    __shared__ __align__(16) float Ts[NB][NB + 1];
    __shared__ float Y[NB][NB + 1];
    __shared__ float Xm[2 * 8 * 8 + 16 * 16];
    __shared__ float taus[NB];
    __shared__ __align__(8) uint64_t mbar[4];   // [0,1] column exchange, [2] RS, [3] AG
    extern __shared__ __align__(16) float dsm[];
    float *ring = dsm;
    float *red8 = ring + PS::NST * PS::CHF;        // [2][16][XW][33]
    float *Wc = red8 + 2 * PS::R8;
    float *W2s = Wc + PS::WE;
    float *RS = W2s + PS::WE;

    const int b = blockIdx.y;
    P += (int64_t)b * a_bstride;
    Ws w = ws_carve(ws0 + (int64_t)b * ws_bstride, n, TS, nsplit);
    float *Vcm = par ? w.Vcm1 : w.Vcm0;
    const int CS = gridDim.x;
    const int rank = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int q = lane & 3, rgw = lane >> 2, rg = warp * 8 + rgw;
    const int row0 = rank * RPC;
    const int rbase = row0 + rg;
    const bool lqv = (cs == 1);
    auto elem = [&](int r, int c) -> S * { return P + (int64_t)r * rs + (int64_t)c * cs; };
    auto load8 = [&](int r, int c0, float (&x)[8]) {
        if (r >= M) {
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = 0.f;
            return;
        }
        if (lqv) {
            const float4 u = ld4(elem(r, c0)), v = ld4(elem(r, c0 + 4));
            x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w;
            x[4] = v.x; x[5] = v.y; x[6] = v.z; x[7] = v.w;
        } else {
#pragma unroll
            for (int c = 0; c < 8; ++c) x[c] = ldf(elem(r, c0 + c));
        }
    };
    if (CS > 1) {
        if (tid == 0) {
            for (int i = 0; i < 4; ++i) p2::mbar_init(&mbar[i], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        csync();
    }
    // bytes this CTA receives per column exchange: CS-1 partial-dot vectors
    // (+ the pivot row from rank 0)
    const unsigned col_bytes = (unsigned)(CS - 1) * 128u + (rank != 0 ? 128u : 0u);
    int t_col = 0;    // column exchanges so far (buffer = t & 1, phase = (t >> 1) & 1)
    int t_bnd = 0;    // boundary all-reduces so far

    // stage XW rest columns [rc, rc + XW) of this CTA's rows into ring slot
    auto stage = [&](int slot_i, int rc) {
        S *dst = reinterpret_cast<S *>(ring + (size_t)slot_i * PS::CHF);
        constexpr int EPV = 16 / (int)sizeof(S);
        if (!lqv) {     // rows contiguous: [XW cols][RPC rows]
            constexpr int SEGC = RPC / EPV;
            for (int sg = tid; sg < XW * SEGC; sg += kPT) {
                const int x = sg / SEGC, rr = (sg - x * SEGC) * EPV, r = row0 + rr;
                const bool ok = r < M;
                p2::cp16(dst + x * RPC + rr, ok ? elem(r, rc + x) : P, ok);
            }
        } else {        // columns contiguous: [RPC rows][XW cols]
            constexpr int SPR = XW / EPV > 0 ? XW / EPV : 1;
            for (int sg = tid; sg < RPC * SPR; sg += kPT) {
                const int lr = sg / SPR, part = sg - lr * SPR, r = row0 + lr;
                const bool ok = r < M;
                p2::cp16(dst + lr * XW + part * EPV, ok ? elem(r, rc + part * EPV) : P, ok);
            }
        }
        p2::cp_commit();
    };
    auto staged = [&](int slot_i, int lr, int x) -> float {
        const S *src = reinterpret_cast<const S *>(ring + (size_t)slot_i * PS::CHF);
        return lqv ? ldf(src + lr * XW + x) : ldf(src + x * RPC + lr);
    };

    float a[RPT][8];
#pragma unroll
    for (int i = 0; i < RPT; ++i) load8(rbase + 128 * i, q * 8, a[i]);

    p2::stamp(0);
    for (int s = 0; s < TS / NB; ++s) {
        const int col0 = s * NB;
        // ---- 32 column steps (4 x 8: only the thread's 8 columns unrolled) --
#pragma unroll 1
        for (int qj = 0; qj < 4; ++qj) {
            p2::stamp(1 + s * 12 + qj);
#pragma unroll
            for (int cj = 0; cj < 8; ++cj) {
                const int j = qj * 8 + cj, jg = col0 + j;
                const int bf = t_col & 1;
                const int src = (lane & ~3) | qj;
                float p[RPT];
#pragma unroll
                for (int i = 0; i < RPT; ++i) p[i] = __shfl_sync(FULL, a[i][cj], src);
                float d[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) d[c] = 0.f;
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const float pm = (rbase + 128 * i > jg) ? p[i] : 0.f;
#pragma unroll
                    for (int c = 0; c < 8; ++c) d[c] = fmaf(pm, a[i][c], d[c]);
                }
                if (rank == 0 && rg == jg) {
#pragma unroll
                    for (int c = 0; c < 8; ++c) prow[bf][q * 8 + c] = a[0][c];
                }
                float dsum[1];
                p2::rs8<8>(d, dsum, lane);
                red[bf][warp][q * 8 + rgw] = dsum[0];
                __syncthreads();
                // every warp: the CTA's partial dot of column `lane` (fixed tree)
                float g;
                {
                    float v[16];
#pragma unroll
                    for (int ww = 0; ww < 16; ++ww) v[ww] = red[bf][ww][lane];
#pragma unroll
                    for (int h = 8; h > 0; h >>= 1)
#pragma unroll
                        for (int u = 0; u < h; ++u) v[u] += v[u + h];
                    g = v[0];
                }
                float pr;
                if (CS > 1) {
                    // warp t pushes to CTA t (every warp holds g): the sends of
                    // one column leave in parallel, not 15 deep from one warp
                    if (warp == 0 && lane == 0) p2::mbar_expect(&mbar[bf], col_bytes);
                    if (warp < CS && warp != rank) {
                        p2::put1(&slot[bf][rank][lane], &mbar[bf], (unsigned)warp, g);
                        if (rank == 0) p2::put1(&pslot[bf][lane], &mbar[bf], (unsigned)warp, prow[bf][lane]);
                    }
                    p2::mbar_wait(&mbar[bf], (unsigned)((t_col >> 1) & 1));
                    // same tree on every CTA (own term from registers): identical sums
                    float v[kMaxCS];
#pragma unroll
                    for (int t = 0; t < kMaxCS; ++t)
                        v[t] = t < CS ? (t == rank ? g : slot[bf][t][lane]) : 0.f;
#pragma unroll
                    for (int h = kMaxCS / 2; h > 0; h >>= 1)
#pragma unroll
                        for (int u = 0; u < h; ++u) v[u] += v[u + h];
                    g = v[0];
                    pr = rank == 0 ? prow[bf][lane] : pslot[bf][lane];
                } else {
                    pr = prow[bf][lane];
                }
                ++t_col;
                const float sigma = __shfl_sync(FULL, g, j), alpha = __shfl_sync(FULL, pr, j);
                float beta, tau, scale;
                house(alpha, sigma, beta, tau, scale);
                const float wv = fmaf(g, scale, pr);   // v_j^T x_l (l > j) / v_l^T v_j (l < j)
                const float fco = lane > j ? tau * wv : 0.f;
                if (warp == 0) {
                    if (lane < j) Y[j][lane] = wv;   // v_l^T v_j, l < j
                    if (lane == 0) taus[j] = tau;
                }
                float f[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) f[c] = __shfl_sync(FULL, fco, q * 8 + c);
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int r = rbase + 128 * i;
                    const float v = (r > jg) ? p[i] * scale : (r == jg ? 1.f : 0.f);
#pragma unroll
                    for (int c = 0; c < 8; ++c) a[i][c] = fmaf(-f[c], v, a[i][c]);
                    if (q == qj) a[i][cj] = (r > jg) ? v : (r == jg ? beta : a[i][cj]);
                }
            }
        }
        __syncthreads();   // T_s, taus complete
        p2::stamp(1 + s * 12 + 4);

        // ---- T_s (compact WY of the sub-panel) by block recursion: 8 x 8
        // diagonal blocks (one warp each), then T12 = -T11 (G12 T22) merges
        // with G[c][j] = v_c^T v_j = Y[j][c]; ~1k cycles on the whole CTA -----
        if (warp < 4 && lane < 8) {
            const int o = warp * 8, i = lane;
            float tr[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float acc = 0.f;
#pragma unroll
                for (int c = 0; c < j; ++c) acc = (c >= i) ? fmaf(tr[c], Y[o + j][o + c], acc) : acc;
                tr[j] = (j < i) ? 0.f : (j == i ? taus[o + j] : -taus[o + j] * acc);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) Ts[o + i][o + j] = tr[j];
        }
        if (warp == 0 && rank == 0) w.tau[col0 + lane] = taus[lane];
        __syncthreads();
#pragma unroll
        for (int h = 8; h < NB; h *= 2) {
            const int nm = NB / (2 * h), per = h * h;
            if (tid < nm * per) {      // X = G12 T22 (T22 upper triangular)
                const int mg = tid / per, r = (tid % per) / h, c = tid % h;
                const int a = mg * 2 * h, bb = a + h;
                float acc = 0.f;
                for (int k = 0; k <= c; ++k) acc = fmaf(Y[bb + k][a + r], Ts[bb + k][bb + c], acc);
                Xm[tid] = acc;
            }
            __syncthreads();
            if (tid < nm * per) {      // T12 = -T11 X (T11 upper triangular)
                const int mg = tid / per, r = (tid % per) / h, c = tid % h;
                const int a = mg * 2 * h, bb = a + h;
                float acc = 0.f;
                for (int k = r; k < h; ++k) acc = fmaf(Ts[a + r][a + k], Xm[mg * per + k * h + c], acc);
                Ts[a + r][bb + c] = -acc;
            }
            __syncthreads();
        }
        // ---- write back R, clean V -> Vrm, Vcm -----------------------------
#pragma unroll
        for (int i = 0; i < RPT; ++i) {
            const int r = rbase + 128 * i;
            float v[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const int cg = col0 + q * 8 + c;
                v[c] = (r > cg) ? a[i][c] : (r == cg ? 1.f : 0.f);
            }
            if (r < M) {
                // only the top TS rows (R) are band: the V tails below them lie
                // outside the band and are never read again (the band packer
                // reads rows [c - b, c]; banddiag clears outside the band)
                if (r < TS) {
                    if (lqv) {
                        st4(elem(r, col0 + q * 8), make_float4(a[i][0], a[i][1], a[i][2], a[i][3]));
                        st4(elem(r, col0 + q * 8 + 4), make_float4(a[i][4], a[i][5], a[i][6], a[i][7]));
                    } else {
#pragma unroll
                        for (int c = 0; c < 8; ++c) stf(elem(r, col0 + q * 8 + c), a[i][c]);
                    }
                }
                float *vr = w.vrm(par) + (int64_t)r * TS + col0 + q * 8;
                *reinterpret_cast<float4 *>(vr) = make_float4(v[0], v[1], v[2], v[3]);
                *reinterpret_cast<float4 *>(vr + 4) = make_float4(v[4], v[5], v[6], v[7]);
#pragma unroll
                for (int c = 0; c < 8; ++c) Vcm[(int64_t)(col0 + q * 8 + c) * n + r] = v[c];
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) a[i][c] = v[c];   // a := clean V from here on
        }
        p2::stamp(1 + s * 12 + 10, 32);   // warp 1's write-back done
        p2::stamp(1 + s * 12 + 5);
        if (s == TS / NB - 1) break;

        // ---- block reflector of the sub-panel on the rest of the panel -------
        const int rc0 = col0 + NB, Rc = TS - rc0;
        const int nch = Rc / XW;
        stage(0, rc0);
        if (nch > 1) stage(1, rc0 + XW);
        // W_cta[c][x] = sum over own rows of V(r, c) A(r, rc0 + x)
#pragma unroll 1
        for (int cc = 0; cc <= nch; ++cc) {
            if (cc < nch) {
                if (cc + 1 < nch) p2::cp_wait<1>();
                else p2::cp_wait<0>();
            }
            __syncthreads();   // chunk cc landed (all threads' copies); red8[(cc-1)&1] complete
            if (cc + 2 < nch) stage((cc + 2) % PS::NST, rc0 + (cc + 2) * XW);
            if (cc > 0 && tid < XW * 32) {       // fold chunk cc-1 over the 16 warps
                const float *rb = red8 + ((cc - 1) & 1) * PS::R8;
                const int xx = tid >> 5, c = tid & 31;
                float v[16];
#pragma unroll
                for (int ww = 0; ww < 16; ++ww) v[ww] = rb[(ww * XW + xx) * 33 + c];
#pragma unroll
                for (int h = 8; h > 0; h >>= 1)
#pragma unroll
                    for (int u = 0; u < h; ++u) v[u] += v[u + h];
                Wc[((cc - 1) * XW + xx) * 32 + c] = v[0];
            }
            if (cc == nch) break;
            float acc[KV];   // [xx][c]
#pragma unroll
            for (int e = 0; e < KV; ++e) acc[e] = 0.f;
            const int sl = cc % PS::NST;
#pragma unroll
            for (int i = 0; i < RPT; ++i) {
                const int lr = rg + 128 * i;
                if (row0 + lr < col0) continue;   // V rows above the sub-panel are zero
                float x[XW];
                if (lqv && sizeof(S) == 4) {
                    const float *src = ring + (size_t)sl * PS::CHF + lr * XW;
#pragma unroll
                    for (int x4 = 0; x4 < XW; x4 += 4) {
                        const float4 t = *reinterpret_cast<const float4 *>(src + x4);
                        x[x4] = t.x; x[x4 + 1] = t.y; x[x4 + 2] = t.z; x[x4 + 3] = t.w;
                    }
                } else {
#pragma unroll
                    for (int xx = 0; xx < XW; ++xx) x[xx] = staged(sl, lr, xx);
                }
#pragma unroll
                for (int xx = 0; xx < XW; ++xx)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[xx * 8 + c] = fmaf(a[i][c], x[xx], acc[xx * 8 + c]);
            }
            float h[KV / 8];
            p2::rs8<KV>(acc, h, lane);
            // lane keeps idx = rgw' * (KV/8) + t  ->  (xx, c) = divmod(idx, 8)
            float *rb = red8 + (cc & 1) * PS::R8;
#pragma unroll
            for (int t = 0; t < KV / 8; ++t) {
                const int idx = rgw * (KV / 8) + t, xx = idx >> 3, c = idx & 7;
                rb[(warp * XW + xx) * 33 + q * 8 + c] = h[t];
            }
        }
        __syncthreads();   // Wc complete (the last chunk's fold)
        p2::stamp(1 + s * 12 + 6);
        // cluster all-reduce of Wc (NB x Rc): reduce-scatter + all-gather
        if (CS > 1) {
            const int E = NB * Rc;
            const int slice = ((E + CS - 1) / CS + 3) & ~3;
            const int own_lo = rank * slice, own_len = max(0, min(slice, E - own_lo));
            const unsigned ph = (unsigned)(t_bnd & 1);
            if (tid == 0) {
                p2::mbar_expect(&mbar[2], (unsigned)((CS - 1) * own_len * 4));
                p2::mbar_expect(&mbar[3], (unsigned)((E - own_len) * 4));
            }
            for (int e4 = tid * 4; e4 < E; e4 += kPT * 4) {
                const int dst = e4 / slice;
                if (dst == rank) continue;
                const float4 v = *reinterpret_cast<const float4 *>(&Wc[e4]);
                p2::put4(&RS[rank * slice + (e4 - dst * slice)], &mbar[2], (unsigned)dst, v);
            }
            p2::mbar_wait(&mbar[2], ph);
            for (int p4 = tid * 4; p4 < own_len; p4 += kPT * 4) {
                float4 sum = f4zero();
                for (int t = 0; t < CS; ++t) {
                    const float4 v = (t == rank) ? *reinterpret_cast<const float4 *>(&Wc[own_lo + p4])
                                                 : *reinterpret_cast<const float4 *>(&RS[t * slice + p4]);
                    sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
                }
                *reinterpret_cast<float4 *>(&Wc[own_lo + p4]) = sum;
                for (int t = 0; t < CS; ++t)
                    if (t != rank) p2::put4(&Wc[own_lo + p4], &mbar[3], (unsigned)t, sum);
            }
            p2::mbar_wait(&mbar[3], ph);
            ++t_bnd;
            __syncthreads();   // own slice (local stores) visible
        }
        p2::stamp(1 + s * 12 + 7);
        // W2 = Ts^T Wc  (W2[x][c] = sum_{j<=c} Ts[j][c] Wc[x][j]); lanes run over c
        for (int e = tid; e < NB * Rc; e += kPT) {
            const int x = e >> 5, c = e & 31;
            const float *wx = Wc + x * 32;
            float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
            for (int j = 0; j < NB; j += 4) {
                if (j <= c) s0 = fmaf(Ts[j][c], wx[j], s0);
                if (j + 1 <= c) s1 = fmaf(Ts[j + 1][c], wx[j + 1], s1);
                if (j + 2 <= c) s2 = fmaf(Ts[j + 2][c], wx[j + 2], s2);
                if (j + 3 <= c) s3 = fmaf(Ts[j + 3][c], wx[j + 3], s3);
            }
            W2s[e] = (s0 + s1) + (s2 + s3);
        }
        __syncthreads();
        // A_rest -= V W2 (own rows): the 4 q lanes of a row reduce-scatter so
        // lane q owns rest columns 2q, 2q+1 of each 8-column chunk
        {
            auto ld2 = [&](int r, int x0, float &u0, float &u1) {
                if (r >= M || r < col0) { u0 = u1 = 0.f; return; }
                if (lqv && sizeof(S) == 4) {
                    const float2 t = *reinterpret_cast<const float2 *>(elem(r, x0));
                    u0 = t.x; u1 = t.y;
                } else {
                    u0 = ldf(elem(r, x0));
                    u1 = ldf(elem(r, x0 + 1));
                }
            };
            float cur[RPT][2], nxt[RPT][2];
#pragma unroll
            for (int i = 0; i < RPT; ++i) ld2(rbase + 128 * i, rc0 + q * 2, cur[i][0], cur[i][1]);
#pragma unroll 1
            for (int cc = 0; cc < Rc / 8; ++cc) {
                if (cc + 1 < Rc / 8) {
#pragma unroll
                    for (int i = 0; i < RPT; ++i) ld2(rbase + 128 * i, rc0 + (cc + 1) * 8 + q * 2, nxt[i][0], nxt[i][1]);
                }
                float wr[8][8];   // [c in group q][x in chunk]
#pragma unroll
                for (int x = 0; x < 8; ++x) {
                    const float4 w0 = *reinterpret_cast<const float4 *>(&W2s[(cc * 8 + x) * 32 + q * 8]);
                    const float4 w1 = *reinterpret_cast<const float4 *>(&W2s[(cc * 8 + x) * 32 + q * 8 + 4]);
                    wr[0][x] = w0.x; wr[1][x] = w0.y; wr[2][x] = w0.z; wr[3][x] = w0.w;
                    wr[4][x] = w1.x; wr[5][x] = w1.y; wr[6][x] = w1.z; wr[7][x] = w1.w;
                }
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int r = rbase + 128 * i;
                    float u[8];
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        float t = 0.f;
#pragma unroll
                        for (int c = 0; c < 8; ++c) t = fmaf(a[i][c], wr[c][x], t);
                        u[x] = t;
                    }
                    float u4[4], u2[2];
                    const bool qb1 = lane & 2, qb0 = lane & 1;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float mine = qb1 ? u[4 + t] : u[t], oth = qb1 ? u[t] : u[4 + t];
                        u4[t] = mine + __shfl_xor_sync(FULL, oth, 2);
                    }
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const float mine = qb0 ? u4[2 + t] : u4[t], oth = qb0 ? u4[t] : u4[2 + t];
                        u2[t] = mine + __shfl_xor_sync(FULL, oth, 1);
                    }
                    if (r < M && r >= col0) {
                        const int x0 = rc0 + cc * 8 + q * 2;
                        const float o0 = cur[i][0] - u2[0], o1 = cur[i][1] - u2[1];
                        if (lqv && sizeof(S) == 4) {
                            *reinterpret_cast<float2 *>(elem(r, x0)) = make_float2(o0, o1);
                        } else {
                            stf(elem(r, x0), o0);
                            stf(elem(r, x0 + 1), o1);
                        }
                    }
                }
                if (cc + 1 < Rc / 8) {
#pragma unroll
                    for (int i = 0; i < RPT; ++i) { cur[i][0] = nxt[i][0]; cur[i][1] = nxt[i][1]; }
                }
            }
        }
        __syncthreads();   // updated rest columns visible to the next sub-panel's loads
        p2::stamp(1 + s * 12 + 8);
#pragma unroll
        for (int i = 0; i < RPT; ++i) load8(rbase + 128 * i, rc0 + q * 8, a[i]);
    }
    p2::stamp(60);
    if (CS > 1) csync();   // no CTA exits while cluster peers may still address it
}

// ---------------------------------------------------------------------------
// FMA GEMM core: C tile BM x BN, 256 threads, per-thread microtile TM x TN
// (rows tm*4+{0..3} [+ BM/2 + ...], cols tn*4+{0..3} [+ BN/2 + ...]).
// Operands staged in shared memory k-major: As[k][BM], Bs[k][BN+4].
template <int BM, int BN>
struct Tile {
    static constexpr int TM = BM / 16, TN = BN / 16;
    static constexpr int BNP = BN + 4;
    static constexpr int A_EL = KC * BM, B_EL = KC * BNP;
    __device__ static __forceinline__ int row(int tm, int ii) {
        return (TM == 8) ? ((ii < 4) ? tm * 4 + ii : BM / 2 + tm * 4 + ii - 4) : tm * 4 + ii;
    }
    __device__ static __forceinline__ int col(int tn, int jj) {
        return (TN == 8) ? ((jj < 4) ? tn * 4 + jj : BN / 2 + tn * 4 + jj - 4) : tn * 4 + jj;
    }
    // acc (+/-)= As^T Bs over one KC chunk
    template <bool SUB>
    __device__ static __forceinline__ void mma(const float *As, const float *Bs, float (&acc)[TM][TN],
                                               int tm, int tn, int kmax = KC) {
#pragma unroll
        for (int k = 0; k < KC; ++k) {
            if (k >= kmax) break;
            float av[TM], bv[TN];
            const float4 a0 = *reinterpret_cast<const float4 *>(&As[k * BM + tm * 4]);
            av[0] = a0.x; av[1] = a0.y; av[2] = a0.z; av[3] = a0.w;
            if (TM == 8) {
                const float4 a1 = *reinterpret_cast<const float4 *>(&As[k * BM + BM / 2 + tm * 4]);
                av[TM == 8 ? 4 : 0] = a1.x; av[TM == 8 ? 5 : 1] = a1.y;
                av[TM == 8 ? 6 : 2] = a1.z; av[TM == 8 ? 7 : 3] = a1.w;
            }
            const float4 b0 = *reinterpret_cast<const float4 *>(&Bs[k * BNP + tn * 4]);
            bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
            if (TN == 8) {
                const float4 b1 = *reinterpret_cast<const float4 *>(&Bs[k * BNP + BN / 2 + tn * 4]);
                bv[TN == 8 ? 4 : 0] = b1.x; bv[TN == 8 ? 5 : 1] = b1.y;
                bv[TN == 8 ? 6 : 2] = b1.z; bv[TN == 8 ? 7 : 3] = b1.w;
            }
#pragma unroll
            for (int ii = 0; ii < TM; ++ii)
#pragma unroll
                for (int jj = 0; jj < TN; ++jj)
                    acc[ii][jj] = SUB ? fmaf(-av[ii], bv[jj], acc[ii][jj]) : fmaf(av[ii], bv[jj], acc[ii][jj]);
        }
    }
};

// Chunk loaders: fetch one KC-chunk into registers, then commit to smem.
// K-major source: element (k, m) at src[k*ld + m] (m contiguous), W columns.
template <typename T, int W>
struct LdKM {
    static constexpr int PER = (KC * W / 4 + kGT - 1) / kGT;   // float4 per thread
    float4 r[PER];
    __device__ __forceinline__ void fetch(const T *src, int64_t ld, int k0, int kmax, int m0, int mmax) {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const int id = threadIdx.x + p * kGT;
            const int k = id / (W / 4), m4 = (id % (W / 4)) * 4;
            r[p] = f4zero();
            if (id < KC * W / 4 && k0 + k < kmax && m0 + m4 < mmax) r[p] = ld4(src + (int64_t)(k0 + k) * ld + m0 + m4);
        }
    }
    // sum of `cnt` equally strided sources (split-K partials), fixed order
    __device__ __forceinline__ void fetch_sum(const float *src, int64_t ld, int64_t sstride, int cnt, int k0,
                                              int kmax, int m0, int mmax) {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const int id = threadIdx.x + p * kGT;
            const int k = id / (W / 4), m4 = (id % (W / 4)) * 4;
            float4 acc = f4zero();
            if (id < KC * W / 4 && k0 + k < kmax && m0 + m4 < mmax) {
                const float *s0 = src + (int64_t)(k0 + k) * ld + m0 + m4;
                // four partials in flight per round trip, summed in split order
                int s = 0;
                for (; s + 4 <= cnt; s += 4) {
                    float4 v[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) v[u] = ld4(s0 + (int64_t)(s + u) * sstride);
#pragma unroll
                    for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
                }
                for (; s < cnt; ++s) {
                    const float4 v = ld4(s0 + (int64_t)s * sstride);
                    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
                }
            }
            r[p] = acc;
        }
    }
    __device__ __forceinline__ void commit(float *dst, int ldd) const {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const int id = threadIdx.x + p * kGT;
            if (id < KC * W / 4) {
                const int k = id / (W / 4), m4 = (id % (W / 4)) * 4;
                *reinterpret_cast<float4 *>(&dst[k * ldd + m4]) = r[p];
            }
        }
    }
};
// M-major source (k contiguous): element (k, m) at src[m*ld + k]; transposed
// into the k-major smem tile.
template <typename T, int W>
struct LdMK {
    static constexpr int PER = (KC * W / 4 + kGT - 1) / kGT;
    float4 r[PER];
    __device__ __forceinline__ void fetch(const T *src, int64_t ld, int k0, int kmax, int m0, int mmax) {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const int id = threadIdx.x + p * kGT;
            const int kq = id % (KC / 4), m = id / (KC / 4);
            r[p] = f4zero();
            if (id < KC * W / 4 && k0 + kq * 4 < kmax && m0 + m < mmax) r[p] = ld4(src + (int64_t)(m0 + m) * ld + k0 + kq * 4);
        }
    }
    __device__ __forceinline__ void commit(float *dst, int ldd) const {
#pragma unroll
        for (int p = 0; p < PER; ++p) {
            const int id = threadIdx.x + p * kGT;
            if (id < KC * W / 4) {
                const int kq = id % (KC / 4), m = id / (KC / 4);
                dst[(kq * 4 + 0) * ldd + m] = r[p].x;
                dst[(kq * 4 + 1) * ldd + m] = r[p].y;
                dst[(kq * 4 + 2) * ldd + m] = r[p].z;
                dst[(kq * 4 + 3) * ldd + m] = r[p].w;
            }
        }
    }
};

// C-tile I/O in the matrix view: element (r, c) at X[r*rs + c*cs]; one of rs,
// cs is 1 (CM: rows contiguous, else columns contiguous).
template <typename S, int BM, int BN, bool CM>
__device__ __forceinline__ void tile_io(S *X, int64_t ld, int r0, int rmax, int c0, int cmax, int tm, int tn,
                                        float (&acc)[BM / 16][BN / 16], bool store) {
    using TL = Tile<BM, BN>;
    constexpr int TM = TL::TM, TN = TL::TN;
    if (CM) {   // rows contiguous: float4 along rows (r = row(tm, 4h..4h+3))
#pragma unroll
        for (int jj = 0; jj < TN; ++jj) {
            const int c = c0 + TL::col(tn, jj);
            if (c >= cmax) continue;
#pragma unroll
            for (int h = 0; h < TM / 4; ++h) {
                const int r = r0 + TL::row(tm, h * 4);
                if (r >= rmax) continue;
                S *p = X + (int64_t)c * ld + r;
                if (store) {
                    st4(p, make_float4(acc[h * 4][jj], acc[h * 4 + 1][jj], acc[h * 4 + 2][jj], acc[h * 4 + 3][jj]));
                } else {
                    const float4 v = ld4(p);
                    acc[h * 4][jj] = v.x; acc[h * 4 + 1][jj] = v.y; acc[h * 4 + 2][jj] = v.z; acc[h * 4 + 3][jj] = v.w;
                }
            }
        }
    } else {    // columns contiguous
#pragma unroll
        for (int ii = 0; ii < TM; ++ii) {
            const int r = r0 + TL::row(tm, ii);
            if (r >= rmax) continue;
#pragma unroll
            for (int h = 0; h < TN / 4; ++h) {
                const int c = c0 + TL::col(tn, h * 4);
                if (c >= cmax) continue;
                S *p = X + (int64_t)r * ld + c;
                if (store) {
                    st4(p, make_float4(acc[ii][h * 4], acc[ii][h * 4 + 1], acc[ii][h * 4 + 2], acc[ii][h * 4 + 3]));
                } else {
                    const float4 v = ld4(p);
                    acc[ii][h * 4] = v.x; acc[ii][h * 4 + 1] = v.y; acc[ii][h * 4 + 2] = v.z; acc[ii][h * 4 + 3] = v.w;
                }
            }
        }
    }
}

// thread -> (tm, tn): the fast lane index runs along the contiguous axis of
// the tile the kernel reads/writes in the matrix (coalesced 256-B rows)
template <bool CM>
__device__ __forceinline__ void tmtn(int &tm, int &tn) {
    if (CM) { tm = threadIdx.x & 15; tn = threadIdx.x >> 4; }
    else { tn = threadIdx.x & 15; tm = threadIdx.x >> 4; }
}

// ---------------------------------------------------------------------------
// k_fgemm2: X[TS:M, :] -= V[TS:M, :] W2  (tile 128 x 128, K = TS).
template <typename S, int TS, bool CM>
__global__ void __launch_bounds__(kGT, 1)
k_fgemm2(S *__restrict__ X, int64_t ld, int64_t a_bstride, int M, int C, const float *ws0,
         int64_t ws_bstride, int64_t n, int nsplit, int par) {
    constexpr int BM = 128, BN = 128;
    using TL = Tile<BM, BN>;
    __shared__ __align__(16) float As[2][TL::A_EL];
    __shared__ __align__(16) float Bs[2][TL::B_EL];
    const int b = blockIdx.z;
    X += (int64_t)b * a_bstride;
    const Ws w = ws_carve(const_cast<float *>(ws0) + (int64_t)b * ws_bstride, n, TS, nsplit);
    const float *Vcm = par ? w.Vcm1 : w.Vcm0;
    const int r0 = TS + blockIdx.x * BM, c0 = blockIdx.y * BN;
    int tm, tn;
    tmtn<CM>(tm, tn);
    float acc[TL::TM][TL::TN];
    tile_io<S, BM, BN, CM>(X, ld, r0, M, c0, C, tm, tn, acc, false);
    LdKM<float, BM> la;
    LdKM<float, BN> lb;
    la.fetch(Vcm, n, 0, TS, r0, M);
    lb.fetch(w.W2, C, 0, TS, c0, C);
    la.commit(As[0], BM);
    lb.commit(Bs[0], TL::BNP);
    __syncthreads();
    constexpr int NCH = TS / KC;
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
        const int cur = ch & 1;
        if (ch + 1 < NCH) {
            la.fetch(Vcm, n, (ch + 1) * KC, TS, r0, M);
            lb.fetch(w.W2, C, (ch + 1) * KC, TS, c0, C);
        }
        TL::template mma<true>(As[cur], Bs[cur], acc, tm, tn);
        if (ch + 1 < NCH) {
            la.commit(As[cur ^ 1], BM);
            lb.commit(Bs[cur ^ 1], TL::BNP);
        }
        __syncthreads();
    }
    tile_io<S, BM, BN, CM>(X, ld, r0, M, c0, C, tm, tn, acc, true);
}

// k_fgemm1: Wp[s] = V[rows_s]^T X[rows_s]  (tile TS x 128, K = rows of split s)
template <typename S, int TS, bool CM>
__global__ void __launch_bounds__(kGT, 1)
k_fgemm1(const S *__restrict__ X, int64_t ld, int64_t a_bstride, int M, int C, float *ws0,
         int64_t ws_bstride, int64_t n, int nsplit, int rps, int par) {
    constexpr int BM = TS < 64 ? 64 : TS, BN = 128;   // ts = 32: rows >= TS zero-filled, masked
    using TL = Tile<BM, BN>;
    __shared__ __align__(16) float As[2][TL::A_EL];
    __shared__ __align__(16) float Bs[2][TL::B_EL];
    const int b = blockIdx.z;
    X += (int64_t)b * a_bstride;
    const Ws w = ws_carve(ws0 + (int64_t)b * ws_bstride, n, TS, nsplit);
    const int c0 = blockIdx.x * BN, sp = blockIdx.y;
    const int k_lo = sp * rps, k_hi = min(M, k_lo + rps);
    int tm, tn;
    tmtn<false>(tm, tn);
    float acc[TL::TM][TL::TN];
#pragma unroll
    for (int ii = 0; ii < TL::TM; ++ii)
#pragma unroll
        for (int jj = 0; jj < TL::TN; ++jj) acc[ii][jj] = 0.f;
    LdKM<float, BM> la;
    LdKM<S, BN> lbr;    // columns contiguous (LQ view)
    LdMK<S, BN> lbc;    // rows contiguous (RQ view): transposed on commit
    auto fetch = [&](int k0) {
        la.fetch(w.vrm(par), TS, k0, k_hi, 0, TS);
        if (CM) lbc.fetch(X, ld, k0, k_hi, c0, C);
        else lbr.fetch(X, ld, k0, k_hi, c0, C);
    };
    auto commit = [&](int buf) {
        la.commit(As[buf], BM);
        if (CM) lbc.commit(Bs[buf], TL::BNP);
        else lbr.commit(Bs[buf], TL::BNP);
    };
    if (k_lo < k_hi) {
        fetch(k_lo);
        commit(0);
        __syncthreads();
        const int nch = (k_hi - k_lo + KC - 1) / KC;
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
            const int cur = ch & 1;
            if (ch + 1 < nch) fetch(k_lo + (ch + 1) * KC);
            TL::template mma<false>(As[cur], Bs[cur], acc, tm, tn);
            if (ch + 1 < nch) commit(cur ^ 1);
            __syncthreads();
        }
    }
    float *Wp = w.Wp + (int64_t)sp * TS * C;
    tile_io<float, BM, BN, false>(Wp, C, 0, TS, c0, C, tm, tn, acc, true);
}

// k_fw2x1: W2 = T^T sum_s Wp[s]  and  X[0:TS] -= V[0:TS] W2  (tile TS x 64)
template <typename S, int TS, bool CM>
__global__ void __launch_bounds__(kGT, 1)
k_fw2x1(S *__restrict__ X, int64_t ld, int64_t a_bstride, int M, int C, float *ws0, int64_t ws_bstride,
        int64_t n, int nsplit, int nused, int par, int w2t) {
    constexpr int BM = TS < 64 ? 64 : TS, BN = 64;    // ts = 32: rows >= TS zero-filled, masked
    using TL = Tile<BM, BN>;
    __shared__ __align__(16) float As[2][TL::A_EL];
    __shared__ __align__(16) float Bs[2][TL::B_EL];
    extern __shared__ __align__(16) float W2s[];   // [BM][BNP]
    const int b = blockIdx.z;
    X += (int64_t)b * a_bstride;
    const Ws w = ws_carve(ws0 + (int64_t)b * ws_bstride, n, TS, nsplit);
    const float *Vcm = par ? w.Vcm1 : w.Vcm0;
    const int c0 = blockIdx.x * BN;
    int tm, tn;
    tmtn<CM>(tm, tn);
    float acc[TL::TM][TL::TN];
#pragma unroll
    for (int ii = 0; ii < TL::TM; ++ii)
#pragma unroll
        for (int jj = 0; jj < TL::TN; ++jj) acc[ii][jj] = 0.f;
    // pass 1: W2 = T^T W  (A(k=j, m=i) = T(j, i): T stored row-major)
    LdKM<float, BM> la;
    LdKM<float, BN> lb;
    constexpr int NCH = TS / KC;
    la.fetch(w.T, TS, 0, TS, 0, TS);
    lb.fetch_sum(w.Wp, C, (int64_t)TS * C, nused, 0, TS, c0, C);
    la.commit(As[0], BM);
    lb.commit(Bs[0], TL::BNP);
    __syncthreads();
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
        const int cur = ch & 1;
        if (ch + 1 < NCH) {
            la.fetch(w.T, TS, (ch + 1) * KC, TS, 0, TS);
            lb.fetch_sum(w.Wp, C, (int64_t)TS * C, nused, (ch + 1) * KC, TS, c0, C);
        }
        TL::template mma<false>(As[cur], Bs[cur], acc, tm, tn);
        if (ch + 1 < NCH) {
            la.commit(As[cur ^ 1], BM);
            lb.commit(Bs[cur ^ 1], TL::BNP);
        }
        __syncthreads();
    }
    // W2 -> global (for k_fgemm2) and smem (B operand of pass 2)
#pragma unroll
    for (int ii = 0; ii < TL::TM; ++ii) {
        const int r = TL::row(tm, ii);
#pragma unroll
        for (int h = 0; h < TL::TN / 4; ++h) {
            const int c = TL::col(tn, h * 4);
            const float4 v = make_float4(acc[ii][h * 4], acc[ii][h * 4 + 1], acc[ii][h * 4 + 2], acc[ii][h * 4 + 3]);
            *reinterpret_cast<float4 *>(&W2s[r * TL::BNP + c]) = v;
            if (c0 + c < C && r < TS) {
                *reinterpret_cast<float4 *>(&w.W2[(int64_t)r * C + c0 + c]) = v;
                if (w2t) {   // K-major copy for the tensor-core update: W2T[c][j]
                    float *t = w.W2T + (int64_t)(c0 + c) * TS + r;
                    t[0] = v.x; t[TS] = v.y; t[2 * TS] = v.z; t[3 * TS] = v.w;
                }
            }
        }
    }
    // pass 2: X[0:TS] -= V[0:TS] W2
    tile_io<S, BM, BN, CM>(X, ld, 0, TS, c0, C, tm, tn, acc, false);
    la.fetch(Vcm, n, 0, TS, 0, TS);
    la.commit(As[0], BM);
    __syncthreads();
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
        const int cur = ch & 1;
        if (ch + 1 < NCH) la.fetch(Vcm, n, (ch + 1) * KC, TS, 0, TS);
        TL::template mma<true>(As[cur], W2s + ch * KC * TL::BNP, acc, tm, tn);
        if (ch + 1 < NCH) la.commit(As[cur ^ 1], BM);
        __syncthreads();
    }
    tile_io<S, BM, BN, CM>(X, ld, 0, TS, c0, C, tm, tn, acc, true);
}

// k_fgram: G = V^T V over row splits; the last CTA merges the partials (fixed
// order) and builds T (compact WY, forward) -> w.T row-major.
template <int TS>
__global__ void __launch_bounds__(kGT, 1)
k_fgram(float *ws0, int64_t ws_bstride, int64_t n, int nsplit, int M, int rps, int par) {
    constexpr int BM = TS < 64 ? 64 : TS, BN = BM;    // ts = 32: zero-filled beyond TS, masked
    using TL = Tile<BM, BN>;
    __shared__ __align__(16) float As[2][TL::A_EL];
    __shared__ __align__(16) float Bs[2][TL::B_EL];
    __shared__ int s_last;
    extern __shared__ __align__(16) float Tsm[];   // [TS][TS+1] T, then tmp TS*TS/4
    const int b = blockIdx.y;
    const Ws w = ws_carve(ws0 + (int64_t)b * ws_bstride, n, TS, nsplit);
    const int sp = blockIdx.x, ns = gridDim.x;
    const int k_lo = sp * rps, k_hi = min(M, k_lo + rps);
    const float *Vrm = w.vrm(par);
    int tm, tn;
    tmtn<false>(tm, tn);
    float acc[TL::TM][TL::TN];
#pragma unroll
    for (int ii = 0; ii < TL::TM; ++ii)
#pragma unroll
        for (int jj = 0; jj < TL::TN; ++jj) acc[ii][jj] = 0.f;
    LdKM<float, BM> la;
    LdKM<float, BN> lb;
    if (k_lo < k_hi) {
        la.fetch(Vrm, TS, k_lo, k_hi, 0, TS);
        lb.fetch(Vrm, TS, k_lo, k_hi, 0, TS);
        la.commit(As[0], BM);
        lb.commit(Bs[0], TL::BNP);
        __syncthreads();
        const int nch = (k_hi - k_lo + KC - 1) / KC;
#pragma unroll 1
        for (int ch = 0; ch < nch; ++ch) {
            const int cur = ch & 1;
            if (ch + 1 < nch) {
                la.fetch(Vrm, TS, k_lo + (ch + 1) * KC, k_hi, 0, TS);
                lb.fetch(Vrm, TS, k_lo + (ch + 1) * KC, k_hi, 0, TS);
            }
            TL::template mma<false>(As[cur], Bs[cur], acc, tm, tn);
            if (ch + 1 < nch) {
                la.commit(As[cur ^ 1], BM);
                lb.commit(Bs[cur ^ 1], TL::BNP);
            }
            __syncthreads();
        }
    }
    float *Gp = w.Gp + (int64_t)sp * TS * TS;
    tile_io<float, BM, BN, false>(Gp, TS, 0, TS, 0, TS, tm, tn, acc, true);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(w.cnt, 1) == ns - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    constexpr int LDT = TS + 1;
    float *tmp = Tsm + TS * LDT;
    for (int e = threadIdx.x; e < TS * TS; e += kGT) {
        const int i = e / TS, j = e % TS;   // G(i, j), i < j kept (strict upper)
        float sum = 0.f;
        float v[kGSplit];            // all partials in flight, summed in split order
#pragma unroll
        for (int s = 0; s < kGSplit; ++s) v[s] = s < ns ? __ldcg(&w.Gp[(int64_t)s * TS * TS + e]) : 0.f;
#pragma unroll
        for (int s = 0; s < kGSplit; ++s) if (s < ns) sum += v[s];
        Tsm[j * LDT + i] = (i < j) ? sum : 0.f;
    }
    __syncthreads();
    panel::build_T_rec<float, TS, kGT>(w.tau, tmp, [&](int i, int j) -> float & { return Tsm[j * LDT + i]; });
    __syncthreads();
    for (int e = threadIdx.x; e < TS * TS; e += kGT) {
        const int i = e / TS, jj = e % TS;   // w.T[i*TS + jj] = T(i, jj) (row-major), zero below
        w.T[e] = (jj >= i) ? Tsm[jj * LDT + i] : 0.f;
    }
    if (threadIdx.x == 0) *w.cnt = 0;
}


// ---------------------------------------------------------------------------
// k_tbuild: T (compact WY, forward) of the whole panel from the Gram matrix
// G = V^T V that the tensor-core W product computed as its extra column tile
// (ns split-K partials, summed here in a fixed order) and tau:
//   diagonal 32 x 32 blocks by the row-parallel recurrence (lane i owns row i:
//     T[i][j] = -tau_j sum_{i<=c<j} T[i][c] G[c][j]),
//   then two merge levels T12 = -T11 (G12 T22) of 32- and 64-wide blocks.
// One CTA of 256 threads per batch member; w.T row-major, zero below the
// diagonal (the layout k_fw2x1 reads).
constexpr int kTB = 256;
template <int TS>
__global__ void __launch_bounds__(kTB, 1) k_tbuild(float *ws0, int64_t ws_bstride, int64_t n, int nsplit, int ns) {
    static_assert(TS == 128, "k_tbuild: ts = 128");
    constexpr int LD = TS + 1;
    extern __shared__ float tsm[];
    float *G = tsm;                 // [TS][LD]
    float *T = G + TS * LD;         // [TS][LD]
    float *Xs = T + TS * LD;        // [64][65] product scratch
    const Ws w = ws_carve(ws0 + (int64_t)blockIdx.x * ws_bstride, n, TS, nsplit);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int e4 = tid * 4; e4 < TS * TS; e4 += kTB * 4) {
        float4 acc = f4zero();
        float4 v[kGSplit];
#pragma unroll
        for (int s = 0; s < kGSplit; ++s)
            v[s] = s < ns ? __ldcg(reinterpret_cast<const float4 *>(w.Gp + (int64_t)s * TS * TS + e4)) : f4zero();
#pragma unroll
        for (int s = 0; s < kGSplit; ++s) {   // fixed order
            acc.x += v[s].x; acc.y += v[s].y; acc.z += v[s].z; acc.w += v[s].w;
        }
        const int i = e4 / TS, j = e4 % TS;
        G[i * LD + j] = acc.x; G[i * LD + j + 1] = acc.y; G[i * LD + j + 2] = acc.z; G[i * LD + j + 3] = acc.w;
        T[i * LD + j] = 0.f; T[i * LD + j + 1] = 0.f; T[i * LD + j + 2] = 0.f; T[i * LD + j + 3] = 0.f;
    }
    __syncthreads();
    if (warp < 4) {                 // diagonal block `warp`
        const int o = warp * 32, i = lane;
        float tr[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            float s0 = 0.f, s1 = 0.f;
#pragma unroll
            for (int c = 0; c < j; ++c) {
                const float gcj = G[(o + c) * LD + o + j];
                if (c & 1) s1 = (c >= i) ? fmaf(tr[c], gcj, s1) : s1;
                else s0 = (c >= i) ? fmaf(tr[c], gcj, s0) : s0;
            }
            const float tj = __ldcg(&w.tau[o + j]);
            tr[j] = (j < i) ? 0.f : (j == i ? tj : -tj * (s0 + s1));
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) T[(o + i) * LD + o + j] = tr[j];
    }
    __syncthreads();
    // merges: T[a:a+h, b:b+h] = -T[a:a+h, a:a+h] * (G[a:a+h, b:b+h] * T[b:b+h, b:b+h]), b = a + h;
    // 4 x 4 register tiles per thread (independent accumulators, the K loop
    // streams one A column and one B row per step)
    for (int h = 32; h < TS; h *= 2) {
        const int nm = TS / (2 * h);               // merges at this level
        const int tpr = h / 4;                      // tiles per row
        const int ntile = nm * tpr * tpr;           // <= 256
        const int LX = h + 1;
        for (int pass = 0; pass < 2; ++pass) {
            if (tid < ntile) {
                const int mg = tid / (tpr * tpr), rem = tid % (tpr * tpr);
                const int r0 = (rem / tpr) * 4, c0 = (rem % tpr) * 4;
                const int a = mg * 2 * h, bb = a + h;
                float acc[4][4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
                float *X = Xs + mg * h * LX;
                if (pass == 0) {   // X = G12 * T22 (T22 upper triangular: rows k <= c0 + 3)
                    for (int k = 0; k <= c0 + 3; ++k) {
                        float av[4], bv[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) av[i] = G[(a + r0 + i) * LD + bb + k];
#pragma unroll
                        for (int j = 0; j < 4; ++j) bv[j] = T[(bb + k) * LD + bb + c0 + j];
#pragma unroll
                        for (int i = 0; i < 4; ++i)
#pragma unroll
                            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) X[(r0 + i) * LX + c0 + j] = acc[i][j];
                } else {           // T12 = -T11 * X (T11 upper triangular: columns k >= r0)
                    for (int k = r0; k < h; ++k) {
                        float av[4], bv[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) av[i] = T[(a + r0 + i) * LD + a + k];
#pragma unroll
                        for (int j = 0; j < 4; ++j) bv[j] = X[k * LX + c0 + j];
#pragma unroll
                        for (int i = 0; i < 4; ++i)
#pragma unroll
                            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
                    }
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) T[(a + r0 + i) * LD + bb + c0 + j] = -acc[i][j];
                }
            }
            __syncthreads();
        }
    }
    for (int e = tid; e < TS * TS; e += kTB) {
        const int i = e / TS, j = e % TS;
        w.T[e] = (j >= i) ? T[i * LD + j] : 0.f;
    }
}

__global__ void k_zero_cnt(float *ws0, int64_t ws_bstride, int64_t n, int ts, int nsplit, int64_t batch) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b < batch) *ws_carve(ws0 + b * ws_bstride, n, ts, nsplit).cnt = 0;
}

// ---------------------------------------------------------------------------
// host side

struct DevCtx {
    std::mutex enqueue_mu;   // one call's enqueue at a time per device (shared streams/events)
    cudaStream_t sp = nullptr, su = nullptr, sg = nullptr;
    cudaEvent_t ev[8] = {};
    bool attr_set = false;
    int nsm = 148;
};
static std::mutex g_mu;
static DevCtx g_ctx[64];

static cudaError_t dev_ctx(DevCtx *&out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(g_mu);
    DevCtx &c = g_ctx[dev & 63];
    if (!c.sp) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if ((e = cudaStreamCreateWithPriority(&c.sp, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&c.su, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithPriority(&c.sg, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
        for (auto &ev : c.ev)
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
        cudaDeviceGetAttribute(&c.nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    out = &c;
    return cudaSuccess;
}

static int pick_rpt(int m, int64_t batch) {
    if (const char *s = getenv("BSVD_FLAT_RPT")) {
        const int v = atoi(s);
        if (v == 1 || v == 2 || v == 4 || v == 8) return (m + v - 1) / v <= kMaxCS ? v : 8;
    }
    if (batch > 1 && m <= 8) return m <= 1 ? 1 : (m <= 2 ? 2 : (m <= 4 ? 4 : 8));
    if (m <= 4) return 1;
    if (m <= 16) return 2;
    if (m <= 64) return 4;
    return 8;
}

static int nsplit_for(int64_t batch) { return batch >= 8 ? 1 : kMaxSplit; }

template <typename S, int TS, int RPT>
static cudaError_t launch_panel(S *P, int64_t rs, int64_t cs, int64_t a_bstride, int M, float *ws,
                                int64_t ws_bstride, int64_t n, int nsplit, int par, int CS, int64_t batch,
                                cudaStream_t st) {
    static const bool v1 = getenv("BSVD_FPANEL_V1") && atoi(getenv("BSVD_FPANEL_V1")) != 0;
    auto kern = v1 ? k_fpanel<S, TS, RPT> : k_fpanel2<S, TS, RPT>;
    const size_t dyn = v1 ? PanelSmem<TS, RPT>::dyn : Panel2<S, TS, RPT>::dyn;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (e != cudaSuccess) return e;
    if (CS > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
        return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)CS, (unsigned)batch, 1);
    cfg.blockDim = dim3(kPT, 1, 1);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = CS > 1 ? 1 : 0;
    e = cudaLaunchKernelEx(&cfg, kern, P, rs, cs, a_bstride, M, ws, ws_bstride, n, nsplit, par);
    bsvd_host::count_launch();
    return e;
}

template <typename S, int TS>
static cudaError_t run_flat(S *a, int64_t n, int64_t batch, int64_t a_bstride, float *ws, cudaStream_t st,
                            double *pms, double *tms, bool timed) {
    DevCtx *cx = nullptr;
    cudaError_t e = dev_ctx(cx);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> enqueue_lock(cx->enqueue_mu);
    const int64_t N = n / TS;
    const int nsplit = nsplit_for(batch);
    constexpr int W2BM = TS < 64 ? 64 : TS;   // k_fw2x1's tile rows
    const int64_t wsb = (int64_t)ws_floats(n, TS, nsplit);
    cudaStream_t sp = cx->sp, su = cx->su, sg = cx->sg;
    cudaEvent_t evStart = cx->ev[0], evP = cx->ev[1], ev1 = cx->ev[2], evW = cx->ev[3], evEndP = cx->ev[4],
                evEndU = cx->ev[5], evT = cx->ev[6], evEndG = cx->ev[7];
    {   // (function attributes are per device: set before every stage)
        e = cudaFuncSetAttribute(k_fw2x1<S, TS, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(W2BM * (64 + 4) * sizeof(float)));
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(k_fw2x1<S, TS, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(W2BM * (64 + 4) * sizeof(float)));
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(k_fgram<TS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)((TS * (TS + 1) + TS * TS / 4) * sizeof(float)));
        if (e != cudaSuccess) return e;
    }
    // the T-build arrival counter of every batch member starts at zero
    k_zero_cnt<<<(unsigned)((batch + 255) / 256), 256, 0, st>>>(ws, wsb, n, TS, nsplit, batch);
    bsvd_host::count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    cudaEventRecord(evStart, st);
    cudaStreamWaitEvent(sp, evStart, 0);
    cudaStreamWaitEvent(su, evStart, 0);
    cudaStreamWaitEvent(sg, evStart, 0);
    cudaEvent_t tp0 = nullptr, tp1 = nullptr;
    if (timed) {
        cudaEventCreate(&tp0);
        cudaEventCreate(&tp1);
        cudaEventRecord(tp0, sp);
    }
    int par = 0;
    const bool use_tc = TS == 128 && flat_tc_supported(TS, (int)sizeof(S));
    FlatTcPlan *tcp = nullptr;
    const size_t tbuild_smem = (2 * (size_t)TS * (TS + 1) + 64 * 65 + 64) * sizeof(float);
    if (use_tc) {
        if constexpr (TS == 128)
            if ((e = ensure_smem(k_tbuild<TS>, tbuild_smem)) != cudaSuccess) return e;
        const Ws w0 = ws_carve(ws, n, TS, nsplit);
        tcp = flat_tc_plan(a, (int)sizeof(S), n, batch, a_bstride, w0.Vcm0, w0.Vcm1, w0.Vrm0, w0.Vrm1, w0.W2T, wsb);
        if (!tcp) return cudaErrorNotSupported;
    }
    // development knob: BSVD_FLAT_TC=2 -> only the W product on the tensor
    // cores, 3 -> only the X update
    const int tc_sel = getenv("BSVD_FLAT_TC") ? atoi(getenv("BSVD_FLAT_TC")) : 1;
    const bool tc1 = use_tc && tc_sel != 3, tc2 = use_tc && tc_sel != 2;
    const char *trace_path = getenv("BSVD_FPANEL_TRACE");
    const int trace_side = getenv("BSVD_FPANEL_TRACE_SIDE") ? atoi(getenv("BSVD_FPANEL_TRACE_SIDE")) : 0;
    unsigned long long *trace_buf = nullptr;
    int side_no = 0;
    if (trace_path) {
        cudaMalloc(&trace_buf, 64 * 8);
        cudaMemset(trace_buf, 0, 64 * 8);
    }
    auto side = [&](int64_t k, bool lq) -> cudaError_t {
        const int64_t top = lq ? k + 1 : k;
        if (top >= N) return cudaSuccess;
        const int M = (int)((N - top) * TS);
        const int C = (int)((N - 1 - k) * TS);
        const int64_t rs = lq ? n : 1, cs = lq ? 1 : n;
        S *P = a + top * TS * rs + k * TS * cs;
        S *X = P + TS * cs;
        const int m = (M + 127) / 128;
        const int rpt = pick_rpt(m, batch);
        const int CS = (m + rpt - 1) / rpt;
        cudaError_t e2;
        const bool tr_this = trace_buf && side_no++ == trace_side;
        if (tr_this) cudaMemcpyToSymbolAsync(p2::g_trace, &trace_buf, sizeof(void *), 0, cudaMemcpyHostToDevice, sp);
        switch (rpt) {
        case 1: e2 = launch_panel<S, TS, 1>(P, rs, cs, a_bstride, M, ws, wsb, n, nsplit, par, CS, batch, sp); break;
        case 2: e2 = launch_panel<S, TS, 2>(P, rs, cs, a_bstride, M, ws, wsb, n, nsplit, par, CS, batch, sp); break;
        case 4: e2 = launch_panel<S, TS, 4>(P, rs, cs, a_bstride, M, ws, wsb, n, nsplit, par, CS, batch, sp); break;
        default: e2 = launch_panel<S, TS, 8>(P, rs, cs, a_bstride, M, ws, wsb, n, nsplit, par, CS, batch, sp); break;
        }
        if (e2 != cudaSuccess) return e2;
        if (tr_this) {
            void *null_ptr = nullptr;
            cudaMemcpyToSymbolAsync(p2::g_trace, &null_ptr, sizeof(void *), 0, cudaMemcpyHostToDevice, sp);
            unsigned long long h[64];
            cudaMemcpyAsync(h, trace_buf, sizeof(h), cudaMemcpyDeviceToHost, sp);
            cudaStreamSynchronize(sp);
            if (FILE *f = fopen(trace_path, "w")) {
                fprintf(f, "side %d M %d CS %d RPT %d\n", trace_side, M, CS, rpt);
                for (int i = 0; i < 64; ++i)
                    if (h[i]) fprintf(f, "%d %.3f\n", i, (double)(h[i] - h[0]) * 1e-3);
                fclose(f);
            }
        }
        if (C > 0) {
            cudaEventRecord(evP, sp);
            if (!tc1) {   // T from V^T V (overlaps the first product on the update stream)
                // >= 64 rows per split: short panels (small n) are bound by the
                // chunk loop's latency, not by the CTA count
                // (batches: the matrices fill the GPU; one 512-row split each)
                const int gs = (int)std::min<int64_t>(kGSplit, std::max<int64_t>(1, M / (batch > 1 ? 512 : 64)));
                const int grps = ((M + gs - 1) / gs + KC - 1) / KC * KC;
                k_fgram<TS><<<dim3((unsigned)gs, (unsigned)batch), kGT, (TS * (TS + 1) + TS * TS / 4) * sizeof(float), sp>>>(
                    ws, wsb, n, nsplit, M, grps, par);
                bsvd_host::count_launch();
                if ((e2 = cudaGetLastError()) != cudaSuccess) return e2;
            }
            // W partials over row splits
            const int cblk = (C + 127) / 128;
            int ns = 1;
            // single matrices: the Gram matrix G = V^T V gets its own ng-way
            // split launch on the third stream, and k_tbuild forms T from it
            // while the W tiles are still running -- off the critical path
            const bool gsep = tc1 && batch == 1 && !getenv("BSVD_GRAM_JOINT");
            const int ng = gsep ? std::max(1, std::min(std::min(nsplit, 8), M / 512)) : 0;
            if (batch == 1 && tc1) {
                // one wave: (cblk W tiles + the Gram tiles) x ns CTAs at one CTA
                // per SM (a second, partial wave doubles the product's time)
                ns = gsep ? std::max(1, std::min(nsplit, (cx->nsm - ng) / cblk))
                          : std::max(1, std::min(nsplit, cx->nsm / (cblk + 1)));
                ns = std::min(ns, std::max(1, M / 256));
                if (getenv("BSVD_TC_NS")) ns = std::max(1, std::min(nsplit, std::min(M / 32, atoi(getenv("BSVD_TC_NS")))));
            } else if (batch == 1) {
                ns = (int)std::max<int64_t>(1, std::min<int64_t>(nsplit, ((tc1 ? 1 : 2) * 148 + cblk - 1) / cblk));
                ns = std::min(ns, std::max(1, M / (tc1 ? 256 : 64)));
                if (tc1 && getenv("BSVD_TC_NS")) ns = std::max(1, std::min(nsplit, std::min(M / 32, atoi(getenv("BSVD_TC_NS")))));
            }
            const int rps = ((M + ns - 1) / ns + (tc1 ? 31 : KC - 1)) / (tc1 ? 32 : KC) * (tc1 ? 32 : KC);
            cudaStreamWaitEvent(su, evP, 0);
            Ws w0 = ws_carve(ws, n, TS, nsplit);
            if (gsep) {
                const int rpg = ((M + std::max(ng, 1) - 1) / std::max(ng, 1) + 31) / 32 * 32;
                cudaStreamWaitEvent(sg, evP, 0);
                e2 = launch_flat_tc(tcp, par, 3, lq, M, 0, (int)(top * TS), (int)((k + 1) * TS), w0.Wp, w0.Gp, wsb, ng,
                                    rpg, a, n, a_bstride, batch, sg);
                if (e2 == cudaSuccess) {
                    if constexpr (TS == 128) {
                        k_tbuild<TS><<<(unsigned)batch, kTB, tbuild_smem, sg>>>(ws, wsb, n, nsplit, ng);
                        bsvd_host::count_launch();
                        e2 = cudaGetLastError();
                    }
                }
                cudaEventRecord(evT, sg);
                if (e2 == cudaSuccess)
                    e2 = launch_flat_tc(tcp, par, 4, lq, M, C, (int)(top * TS), (int)((k + 1) * TS), w0.Wp, w0.Gp, wsb,
                                        ns, rps, a, n, a_bstride, batch, su);
            } else if (tc1)
            {
                e2 = launch_flat_tc(tcp, par, 1, lq, M, C, (int)(top * TS), (int)((k + 1) * TS), w0.Wp, w0.Gp, wsb, ns,
                                    rps, a, n, a_bstride, batch, su);
                if (e2 == cudaSuccess) {
                    if constexpr (TS == 128) {
                        k_tbuild<TS><<<(unsigned)batch, kTB, tbuild_smem, su>>>(ws, wsb, n, nsplit, ns);
                        bsvd_host::count_launch();
                        e2 = cudaGetLastError();
                    }
                }
            }
            else if (lq)
                k_fgemm1<S, TS, false><<<dim3((unsigned)cblk, (unsigned)ns, (unsigned)batch), kGT, 0, su>>>(
                    X, rs, a_bstride, M, C, ws, wsb, n, nsplit, rps, par);
            else
                k_fgemm1<S, TS, true><<<dim3((unsigned)cblk, (unsigned)ns, (unsigned)batch), kGT, 0, su>>>(
                    X, cs, a_bstride, M, C, ws, wsb, n, nsplit, rps, par);
            if (!tc1) {
                bsvd_host::count_launch();
                e2 = cudaGetLastError();
            }
            if (e2 != cudaSuccess) return e2;
            cudaEventRecord(ev1, su);
            cudaStreamWaitEvent(sp, ev1, 0);
            if (gsep) cudaStreamWaitEvent(sp, evT, 0);
            const size_t w2sm = W2BM * (64 + 4) * sizeof(float);
            if (lq)
                k_fw2x1<S, TS, false><<<dim3((unsigned)((C + 63) / 64), 1, (unsigned)batch), kGT, w2sm, sp>>>(
                    X, rs, a_bstride, M, C, ws, wsb, n, nsplit, ns, par, tc2 ? 1 : 0);
            else
                k_fw2x1<S, TS, true><<<dim3((unsigned)((C + 63) / 64), 1, (unsigned)batch), kGT, w2sm, sp>>>(
                    X, cs, a_bstride, M, C, ws, wsb, n, nsplit, ns, par, tc2 ? 1 : 0);
            bsvd_host::count_launch();
            if ((e2 = cudaGetLastError()) != cudaSuccess) return e2;
            if (M > TS) {
                cudaEventRecord(evW, sp);
                cudaStreamWaitEvent(su, evW, 0);
                const dim3 g2((unsigned)((M - TS + 127) / 128), (unsigned)cblk, (unsigned)batch);
                if (tc2) {
                    e2 = launch_flat_tc(tcp, par, 2, lq, M, C, (int)(top * TS), (int)((k + 1) * TS), w0.Wp, w0.Gp, wsb,
                                        1, 0, a, n, a_bstride, batch, su);
                    if (e2 != cudaSuccess) return e2;
                } else if (lq)
                    k_fgemm2<S, TS, false><<<g2, kGT, 0, su>>>(X, rs, a_bstride, M, C, ws, wsb, n, nsplit, par);
                else
                    k_fgemm2<S, TS, true><<<g2, kGT, 0, su>>>(X, cs, a_bstride, M, C, ws, wsb, n, nsplit, par);
                if (!tc2) {
                    bsvd_host::count_launch();
                    if ((e2 = cudaGetLastError()) != cudaSuccess) return e2;
                }
            }
        }
        par ^= 1;
        return cudaSuccess;
    };
    for (int64_t k = 0; k < N - 1 && e == cudaSuccess; ++k) {
        if ((e = side(k, false)) != cudaSuccess) break;
        e = side(k, true);
    }
    if (e == cudaSuccess) e = side(N - 1, false);
    cudaEventRecord(evEndP, sp);
    cudaEventRecord(evEndU, su);
    cudaEventRecord(evEndG, sg);
    cudaStreamWaitEvent(st, evEndP, 0);
    cudaStreamWaitEvent(st, evEndU, 0);
    cudaStreamWaitEvent(st, evEndG, 0);
    if (timed) {
        cudaEventRecord(tp1, st);
        cudaEventSynchronize(tp1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tp0, tp1);
        *pms += ms;   // the whole stage (panel chain and updates overlap)
        *tms += ms;
        cudaEventDestroy(tp0);
        cudaEventDestroy(tp1);
    }
    if (trace_buf) cudaFree(trace_buf);
    if (tcp) flat_tc_plan_free(tcp);
    return e;
}

}  // namespace flat

size_t flat_workspace_bytes(int64_t n, int ts, int64_t batch) {
    return flat::ws_floats(n, ts, flat::nsplit_for(batch)) * sizeof(float) * (size_t)batch;
}

bool flat_supported(int ts, int elem_bytes) {
    if (const char *s = getenv("BSVD_FLAT")) {
        if (atoi(s) == 0) return false;
    }
    return (ts == 32 || ts == 64 || ts == 128) && elem_bytes <= 4;
}

template <typename S>
cudaError_t banddiag_flat(S *a, int64_t n, int ts, int64_t batch, int64_t a_bstride, void *ws, cudaStream_t st,
                          double *panel_ms, double *trail_ms) {
    const bool timed = panel_ms != nullptr;
    if (ts == 128) return flat::run_flat<S, 128>(a, n, batch, a_bstride, (float *)ws, st, panel_ms, trail_ms, timed);
    if (ts == 64) return flat::run_flat<S, 64>(a, n, batch, a_bstride, (float *)ws, st, panel_ms, trail_ms, timed);
    return flat::run_flat<S, 32>(a, n, batch, a_bstride, (float *)ws, st, panel_ms, trail_ms, timed);
}

template cudaError_t banddiag_flat<float>(float *, int64_t, int, int64_t, int64_t, void *, cudaStream_t, double *, double *);
template cudaError_t banddiag_flat<__half>(__half *, int64_t, int, int64_t, int64_t, void *, cudaStream_t, double *, double *);

}  // namespace bsvd
