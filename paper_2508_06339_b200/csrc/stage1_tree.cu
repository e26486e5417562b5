// stage1_tree.cu -- fast stage 1 (dense -> band) for sm_100a.
//
// Same tile operators as the reference stage 1 (bandreduce.py:31-120,
// kernels.py:205-559): GEQRT on ts x ts tiles, a triangle-on-triangle TSQRT
// (kernels.py:286-313 with B upper triangular), and WY-form UNMQR / TSMQR
// trailing updates.  What changes is the panel's reduction tree: the
// reference walks each panel as ONE flat TSQRT chain (critical path ~N^2
// tile QRs per matrix); here every panel tile is factored
// in parallel and the R factors are combined by a binary tree (depth
// ceil(log2 m)).  The orthogonal factor differs from the reference's, the
// band differs, the singular values do not (parity is on values).
//
// Per sweep side (RQ on the matrix, LQ on its lazy transpose -- a stride
// swap, no copy) there are exactly two launches:
//
//  k_panel_tree   one CTA per panel tile.  Leaf: Householder QR of the tile
//                 in shared memory (reference reflector scalars, incl. the
//                 10*eps guard), then the compact-WY factor T (larft) and
//                 U = V T^T.  Tree: the second child CTA to arrive at a node
//                 (atomic arrival counter) combines [R_left; R_right] with a
//                 TT-QR and climbs; the root writes R into the band tile.
//  k_trail_tree   one CTA per CB-column block of the trailing matrix.  Walks
//                 the same tree in post-order with an on-chip stack of
//                 ts x CB tiles, so every trailing tile is read once and
//                 written once per sweep side:
//                   leaf:  W = V^T X;                 X -= U W
//                   node:  W = X_top + V^T X_bot;     X_top -= T^T W;
//                          X_bot -= U W
//                 Each product is a register-blocked FMA GEMM (K = ts) with
//                 the ts x ts operand streamed through shared memory.
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_sm100.cuh"

namespace bsvd {

constexpr int kNT = 256;          // threads per CTA for both kernels

template <typename C> struct TileCfg {
    // trailing column-block width: a ts x CB tile is 16 KiB
    static constexpr int elems = 16384 / (int)sizeof(C);
};

__host__ __device__ inline int64_t tree_count(int64_t m, int j) {  // nodes at level j
    return (m + ((int64_t)1 << j) - 1) >> j;
}
__host__ __device__ inline int tree_levels(int64_t m) {           // ceil(log2 m)
    int L = 0;
    while (((int64_t)1 << L) < m) ++L;
    return L;
}
__host__ __device__ inline int64_t tree_offset(int64_t m, int j) { // first slot of level j
    int64_t off = 0;
    for (int q = 0; q < j; ++q) off += tree_count(m, q);
    return off;
}

// Workspace of one sweep side for one matrix:
//   node slots (tree_slots(N)): Vk | Um | Tt   (3 ts^2 C each)
//   R slots (N): ts^2 C each
//   arrival counters (N ints)
template <typename C>
struct TreeWs {
    C *nodes;   // slot s at nodes + s * 3 * ts2
    C *R;       // leaf l at R + l * ts2
    int *cnt;
    int64_t ts2;
    __host__ __device__ C *Vk(int64_t s) const { return nodes + s * 3 * ts2; }
    __host__ __device__ C *Um(int64_t s) const { return nodes + s * 3 * ts2 + ts2; }
    __host__ __device__ C *Tt(int64_t s) const { return nodes + s * 3 * ts2 + 2 * ts2; }
};

// Exact slot count sum_j ceil(N / 2^j) down to the root (it can exceed 2N:
// 5+3+2+1 = 11); the count is nondecreasing in m, so N bounds every side.
__host__ __device__ inline int64_t tree_slots(int64_t N) {
    int64_t s = 1;
    for (int64_t c = N; c > 1; c = (c + 1) / 2) s += c;
    return s + 8;
}

// Tensor-core trailing update (stage1_apply_tc.cu): fp32 compute, ts = 128.
template <typename C>
__host__ __device__ inline bool tree_tc(int ts) { return sizeof(C) == 4 && ts == 128; }

// Elements before the tensor-core operand images (nodes | R | counters).
template <typename C>
__host__ __device__ inline size_t tree_img_offset(int64_t N, int ts) {
    const int64_t ts2 = (int64_t)ts * ts;
    const size_t e = (size_t)(tree_slots(N) * 3 * ts2 + N * ts2) + (size_t)(N + 64) * sizeof(int) / sizeof(C) + 64;
    return (e + 63) & ~(size_t)63;
}

// Elements before the two-tile-leaf region (per super-leaf: V and U rows
// ts..2ts-1, ts^2 each; the first ts rows stay in the leaf's Vk / Um slots).
template <typename C>
__host__ __device__ inline size_t tree_leaf2_offset(int64_t N, int ts) {
    size_t e = tree_img_offset<C>(N, ts);
    if (tree_tc<C>(ts)) e += (size_t)tree_slots(N) * 6 * ts * ts;   // hi/lo images, 3 per node
    return (e + 63) & ~(size_t)63;
}
template <typename C>
__host__ __device__ inline size_t tree_ws_elems(int64_t N, int ts) {
    // rounded to 64 elements: every batch member's slice stays 256-byte
    // aligned for the 16-byte cp.async / bulk-copy tile loads
    const size_t e = tree_leaf2_offset<C>(N, ts) + (size_t)N * 2 * ts * ts;
    return (e + 63) & ~(size_t)63;
}

template <typename C>
__device__ __forceinline__ C warp_sum_t(C v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename C, int G>
__device__ __forceinline__ C group_sum(C v) {   // sum over G consecutive lanes
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Scale-invariant Householder scalars (LAPACK dlarfg convention): the
// column (alpha, tail) with ||tail||^2 = sig maps to (beta, 0) with
// H = I - tau v v^T, v = (1, tail*scale).  A zero tail gives tau = 0 (H = I).
// Unlike the reference's absolute 10*eps guard (kernels.py:109)
// this commutes with scaling, so tiny-scaled inputs keep full accuracy; the
// faithful path (faithful.cu) keeps the reference's guard bit-for-bit.
template <typename C>
__device__ __forceinline__ void house_scalars(C alpha, C sig, C &beta, C &tau, C &scale) {
    if (sig == C(0)) {
        beta = alpha;
        tau = C(0);
        scale = C(1);
    } else {
        beta = -copysign(dsqrt(alpha * alpha + sig), alpha);
        tau = (beta - alpha) / beta;
        scale = C(1) / (alpha - beta);
    }
}

// fp32: one correctly rounded sqrt and two correctly rounded reciprocals in
// place of two IEEE divisions (shorter dependent chain in the panel's column
// step; tau and scale stay within an ulp or two).
__device__ __forceinline__ void house_scalars(float alpha, float sig, float &beta, float &tau, float &scale) {
    if (sig == 0.f) {
        beta = alpha;
        tau = 0.f;
        scale = 1.f;
    } else {
        beta = -copysignf(__fsqrt_rn(fmaf(alpha, alpha, sig)), alpha);
        const float d = alpha - beta;
        scale = __frcp_rn(d);
        tau = -d * __frcp_rn(beta);
    }
}

// ---------------------------------------------------------------------------
// Leaf: Householder QR of one ts x ts tile held column-major in smem (ld =
// ts+1), reference reflector scalars.  Afterwards: R in the upper triangle,
// v (unit implied) strictly below, tau[] in smem (house_scalars).
template <typename C, int TS>
__device__ void leaf_qr(C *A, C *tau, C *scal) {
    constexpr int LD = TS + 1;
    constexpr int TPC = (kNT / TS) < 32 ? (kNT / TS) : 32;   // threads per column
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int kk = 0; kk < TS - 1; ++kk) {
        if (warp == 0) {
            C sig = C(0);
            for (int r = kk + 1 + lane; r < TS; r += 32) sig += A[kk * LD + r] * A[kk * LD + r];
            sig = warp_sum_t(sig);
            const C alpha = A[kk * LD + kk];
            C beta, t, scale;
            house_scalars(alpha, sig, beta, t, scale);
            for (int r = kk + 1 + lane; r < TS; r += 32) A[kk * LD + r] *= scale;
            if (lane == 0) {
                A[kk * LD + kk] = beta;
                tau[kk] = t;
            }
        }
        __syncthreads();
        const C t = tau[kk];
        // columns c > kk: TPC threads per column
        const int g = tid / TPC, q = tid % TPC;
        for (int cb = kk + 1; cb < TS; cb += kNT / TPC) {   // warp-uniform trip count
            const int c = cb + g;
            const bool act = c < TS;
            C w = C(0);
            if (act)
                for (int r = kk + 1 + q; r < TS; r += TPC) w += A[kk * LD + r] * A[c * LD + r];
            w = group_sum<C, TPC>(w);
            if (act) {
                w = (w + A[c * LD + kk]) * t;
                for (int r = kk + 1 + q; r < TS; r += TPC) A[c * LD + r] -= w * A[kk * LD + r];
                if (q == 0) A[c * LD + kk] -= w;
            }
        }
        __syncthreads();
    }
    if (tid == 0) tau[TS - 1] = C(0);   // A8: last tile column has no reflector
    __syncthreads();
    (void)scal;
}

// T (upper, compact WY, forward columnwise) from G = V^T V and tau.
// getG(i, j) for i < j, Tset/Tget store T(i, j) for i <= j.  tmp: ts vector.
template <typename C, int TS, typename GetG, typename TGet, typename TSet>
__device__ void build_T(const C *tau, C *tmp, GetG getG, TGet tget, TSet tset) {
    const int tid = threadIdx.x;
    for (int j = 0; j < TS; ++j) {
        for (int i = tid; i < j; i += kNT) tmp[i] = getG(i, j);
        __syncthreads();
        C v = C(0);
        if (tid < j) {
            C s = C(0);
            for (int q = tid; q < j; ++q) s += tget(tid, q) * tmp[q];
            v = -tau[j] * s;
        }
        __syncthreads();
        if (tid < j) tset(tid, j, v);
        if (tid == 0) tset(j, j, tau[j]);
        __syncthreads();
    }
}

// Packed upper-triangular column-major index (r <= c).
__host__ __device__ __forceinline__ int pk(int r, int c) { return c * (c + 1) / 2 + r; }

// TT-QR of [R_top; R_bot], both upper triangular, packed in smem.  After:
// R_top updated, R_bot holds V_b (upper), tau[] (house_scalars).
template <typename C, int TS>
__device__ void tt_qr(C *Rt, C *Rb, C *tau, C *scal) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int kk = 0; kk < TS; ++kk) {
        if (warp == 0) {
            C sig = C(0);
            for (int r = lane; r <= kk; r += 32) sig += Rb[pk(r, kk)] * Rb[pk(r, kk)];
            sig = warp_sum_t(sig);
            const C alpha = Rt[pk(kk, kk)];
            C beta, t, scale;
            house_scalars(alpha, sig, beta, t, scale);
            for (int r = lane; r <= kk; r += 32) Rb[pk(r, kk)] *= scale;
            if (lane == 0) {
                Rt[pk(kk, kk)] = beta;
                tau[kk] = t;
            }
        }
        __syncthreads();
        const C t = tau[kk];
        constexpr int TPC = (kNT / TS) < 32 ? (kNT / TS) : 32;
        const int g = tid / TPC, q = tid % TPC;
        for (int cb = kk + 1; cb < TS; cb += kNT / TPC) {   // warp-uniform trip count
            const int c = cb + g;
            const bool act = c < TS;
            C w = C(0);
            if (act)
                for (int r = q; r <= kk; r += TPC) w += Rb[pk(r, kk)] * Rb[pk(r, c)];
            w = group_sum<C, TPC>(w);
            if (act) {
                w = (w + Rt[pk(kk, c)]) * t;
                for (int r = q; r <= kk; r += TPC) Rb[pk(r, c)] -= w * Rb[pk(r, kk)];
                if (q == 0) Rt[pk(kk, c)] -= w;
            }
        }
        __syncthreads();
    }
    (void)scal;
}

}  // namespace bsvd
#include "panel_qr.cuh"
#include "panel_blocked.cuh"
namespace bsvd {

// Per-device streams (panel chain at high priority, updates, factors at high
// priority) and a reusable event pool for the tree stage 1.
struct TreeCtx {
    std::mutex mu;
    cudaStream_t st1 = nullptr, st2 = nullptr, st3 = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaError_t reserve(size_t k) {
        while (ev.size() < k) {
            cudaEvent_t e;
            cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            if (err != cudaSuccess) return err;
            ev.push_back(e);
        }
        return cudaSuccess;
    }
};
static cudaError_t tree_ctx(TreeCtx *&out) {
    static std::mutex mu;
    static TreeCtx ctx[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    TreeCtx &c = ctx[dev & 63];
    if (!c.st2) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if ((e = cudaStreamCreateWithPriority(&c.st1, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&c.st2, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithPriority(&c.st3, cudaStreamNonBlocking, hi)) != cudaSuccess) return e;
    }
    out = &c;
    return cudaSuccess;
}

// Development instrumentation (BSVD_PANEL_TRACE): leaf-phase timestamps of
// one chosen panel launch.
__device__ unsigned long long *g_panel_trace = nullptr;
__device__ __forceinline__ unsigned long long gtimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// View helpers: tile (tr, tc) of the (possibly transposed) matrix view.
template <typename S>
struct View {
    S *base;
    int64_t rs, cs;
    __device__ __forceinline__ S *ptr(int64_t r, int64_t c) const { return base + r * rs + c * cs; }
};

// ---------------------------------------------------------------------------
// Panel kernel.  Grid: m CTAs (tile rows top..top+m-1 of view tile column k).
template <typename S, typename C, int TS>
__global__ void __launch_bounds__(kNT) k_panel_tree(View<S> V, int64_t m, int64_t top, int64_t k,
                                                   TreeWs<C> ws, int64_t ws_bstride,
                                                   int64_t a_bstride) {
    using CV = Conv<S, C>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *sm = (C *)smem_raw;
    constexpr int LD = TS + 1;
    constexpr int PK = TS * (TS + 1) / 2;
    // layout: [ big: max(TS*LD, 3*PK) ] [tau TS] [tmp TS] [scal 8]
    constexpr int BIG = (TS * LD > 3 * PK) ? TS * LD : 3 * PK;
    C *tau = sm + BIG;
    C *tmp = tau + TS;
    C *scal = tmp + TS;
    __shared__ int s_old;

    const int64_t b = blockIdx.y;
    V.base += b * a_bstride;
    ws.nodes += b * ws_bstride;
    ws.R += b * ws_bstride;
    ws.cnt = (int *)((char *)ws.cnt + b * ws_bstride * (int64_t)sizeof(C));
    const int64_t l = blockIdx.x;
    const int tid = threadIdx.x;
    const int64_t ts2 = (int64_t)TS * TS;
    auto house = [](C a, C s, C &b, C &t, C &sc) { house_scalars(a, s, b, t, sc); };
    unsigned long long *trc = g_panel_trace && b == 0 && l < 64 ? g_panel_trace + l * 8 : nullptr;
    auto mark = [&](int ph) {
        if (trc && tid == 0) trc[ph] = gtimer_ns();
    };

    // ---- leaf: GEQRT of view tile (top + l, k) ----
    {
        C *A = sm;
        mark(0);
        const int64_t r0 = (top + l) * TS, c0 = k * TS;
        for (int idx = tid; idx < TS * TS; idx += kNT) {
            int r, c;
            if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % TS; r = idx / TS; }
            A[c * LD + r] = CV::ld(*V.ptr(r0 + r, c0 + c));
        }
        __syncthreads();
        mark(1);
        panel::leaf_qr_la<C, TS, kNT>(A, tau, house);
        mark(2);
        // R -> ws.R[l] (column-major, upper triangle + zeros)
        C *Rg = ws.R + l * ts2;
        for (int idx = tid; idx < TS * TS; idx += kNT) {
            const int c = idx / TS, r = idx % TS;
            Rg[idx] = (r <= c) ? A[c * LD + r] : C(0);
        }
        __syncthreads();
        // G (i<j) into the upper triangle (R saved), then T in place, tau on the diagonal.
        for (int idx = tid; idx < TS * TS; idx += kNT) {
            const int j = idx / TS, i = idx % TS;
            if (i < j) {
                const C *vi = A + i * LD, *vj = A + j * LD;
                C s0 = vi[j], s1 = C(0);   // V[j][i] (V[j][j] = 1)
                int r = j + 1;
                for (; r + 1 < TS; r += 2) {
                    s0 += vi[r] * vj[r];
                    s1 += vi[r + 1] * vj[r + 1];
                }
                if (r < TS) s0 += vi[r] * vj[r];
                A[j * LD + i] = s0 + s1;
            }
        }
        __syncthreads();
        mark(3);
        panel::build_T_rec<C, TS, kNT>(tau, A + TS * LD, [&](int i, int j) -> C & { return A[j * LD + i]; });
        mark(4);
        // Vk[r][i] = V(r, i);  Um[i][r] = U(r, i) = sum_{j=i..r} V(r,j) T(i,j)
        C *Vk = ws.Vk(l), *Um = ws.Um(l);
        for (int idx = tid; idx < TS * TS; idx += kNT) {
            const int r = idx / TS, i = idx % TS;
            Vk[idx] = (r > i) ? A[i * LD + r] : (r == i ? C(1) : C(0));
        }
        for (int idx = tid; idx < TS * TS; idx += kNT) {
            const int i = idx / TS, r = idx % TS;
            C s0 = C(0), s1 = C(0);
            if (r >= i) {
                s0 = A[i * LD + i] * ((r == i) ? C(1) : A[i * LD + r]);   // j = i: T(i,i)=tau_i
                int j = i + 1;
                for (; j + 1 < r; j += 2) {
                    s0 += A[j * LD + r] * A[j * LD + i];
                    s1 += A[(j + 1) * LD + r] * A[(j + 1) * LD + i];
                }
                for (; j <= r; ++j) s0 += ((j == r) ? C(1) : A[j * LD + r]) * A[j * LD + i];
            }
            Um[idx] = s0 + s1;
        }
        __syncthreads();
        mark(5);
    }

    // ---- tree: climb while we are the second arrival ----
    const int L = tree_levels(m);
    int64_t node = l;   // index at current level
    for (int j = 1; j <= L; ++j) {
        const int64_t parent = node >> 1;
        const bool has_right = ((parent << 1) + 1) < tree_count(m, j - 1);
        if (has_right) {
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                int *c = ws.cnt + tree_offset(m, j) - m + parent;   // level>=1 counters
                s_old = atomicAdd(c, 1);
                if (s_old == 1) *c = 0;   // self-cleaning for the next launch
                __threadfence();
            }
            __syncthreads();
            if (s_old == 0) return;   // first arrival: the sibling continues
            trc = g_panel_trace && b == 0 && parent < 64 ? g_panel_trace + (64 + j * 64 + parent) * 8 : nullptr;
            mark(0);
            // combine: left leaf slot a = (2*parent) << (j-1), right b = (2*parent+1) << (j-1)
            const int64_t a = (parent << 1) << (j - 1);
            const int64_t bb = ((parent << 1) + 1) << (j - 1);
            C *Rt = sm, *Rb = sm + PK, *Tp = sm + 2 * PK;
            const C *Ra_g = ws.R + a * ts2, *Rb_g = ws.R + bb * ts2;
            for (int idx = tid; idx < TS * TS; idx += kNT) {
                const int c = idx / TS, r = idx % TS;
                if (r <= c) {
                    Rt[pk(r, c)] = __ldcg(Ra_g + idx);
                    Rb[pk(r, c)] = __ldcg(Rb_g + idx);
                }
            }
            __syncthreads();
            mark(1);
            panel::tt_qr_la<C, TS, kNT>(Rt, Rb, tau, house);
            mark(2);
            // R_top -> slot a
            C *Rg = ws.R + a * ts2;
            for (int idx = tid; idx < TS * TS; idx += kNT) {
                const int c = idx / TS, r = idx % TS;
                Rg[idx] = (r <= c) ? Rt[pk(r, c)] : C(0);
            }
            // G(i,j) = sum_{r<=i} Vb(r,i) Vb(r,j) into Tp, then T in place
            for (int idx = tid; idx < TS * TS; idx += kNT) {
                const int jj = idx / TS, i = idx % TS;
                if (i < jj) {
                    const C *vi = Rb + pk(0, i), *vj = Rb + pk(0, jj);
                    C s0 = C(0), s1 = C(0);
                    int r = 0;
                    for (; r + 1 <= i; r += 2) {
                        s0 += vi[r] * vj[r];
                        s1 += vi[r + 1] * vj[r + 1];
                    }
                    if (r <= i) s0 += vi[r] * vj[r];
                    Tp[pk(i, jj)] = s0 + s1;
                }
            }
            __syncthreads();
            mark(3);
            // Rt is saved: its space is the T-merge scratch
            panel::build_T_rec<C, TS, kNT>(tau, Rt, [&](int i, int jj) -> C & { return Tp[pk(i, jj)]; });
            mark(4);
            const int64_t slot = tree_offset(m, j) + parent;
            C *Vk = ws.Vk(slot), *Um = ws.Um(slot), *Tt = ws.Tt(slot);
            for (int idx = tid; idx < TS * TS; idx += kNT) {
                const int r = idx / TS, i = idx % TS;   // Vk[r][i] = Vb(r,i); Tt[r][i] = T(r,i)
                Vk[idx] = (r <= i) ? Rb[pk(r, i)] : C(0);
                Tt[idx] = (r <= i) ? Tp[pk(r, i)] : C(0);
            }
            for (int idx = tid; idx < TS * TS; idx += kNT) {
                const int i = idx / TS, r = idx % TS;   // Um[i][r] = U(r,i) = sum_{jj>=max(i,r)} Vb(r,jj) T(i,jj)
                C s = C(0);
                for (int jj = (i > r ? i : r); jj < TS; ++jj) s += Rb[pk(r, jj)] * Tp[pk(i, jj)];
                Um[idx] = s;
            }
            __syncthreads();
            mark(5);
        }
        node = parent;
    }
    // root: R of the whole panel (slot 0) -> upper triangle of view tile (top, k)
    __syncthreads();
    if (L == 0 || node == 0) {
        const C *Rg = ws.R;   // leaf slot 0
        const int64_t r0 = top * TS, c0 = k * TS;
        for (int idx = tid; idx < TS * TS; idx += kNT) {
            int r, c;
            if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % TS; r = idx / TS; }
            if (r <= c) *V.ptr(r0 + r, c0 + c) = CV::st(__ldcg(Rg + c * TS + r));
        }
    }
}

// ---------------------------------------------------------------------------
// Blocked panel kernel (ts >= 16): same tree and workspace contract as
// k_panel_tree, node QRs by blk::qr_blocked (panel_blocked.cuh).  The TT
// operand is held unpacked (2ts x ts) except for fp64 at ts = 128, which
// would not fit shared memory and keeps the packed look-ahead TT-QR.
constexpr int kNTP = 512;         // blocked panel CTA: 16 warps hide the column-step latencies

template <typename C, int TS>
struct PanelBlk {
    static constexpr int NB = blk::NBsel<C, TS>::v;
    static constexpr bool TT_BLOCKED = !(sizeof(C) == 8 && TS >= 128);
    static constexpr int LDL = TS + 1;                        // leaf lda
    static constexpr int LDT = 2 * TS + 1;                    // TT lda (unpacked)
    static constexpr int AUX = blk::aux_elems<C, TS>();
    static constexpr int LEAF = TS * LDL + AUX;
    static constexpr int PK = TS * (TS + 1) / 2;
    static constexpr int TTN = TT_BLOCKED ? (TS * LDT + AUX) : (3 * PK);
    static constexpr int UNION = LEAF > TTN ? LEAF : TTN;
    static constexpr size_t smem = (size_t)(UNION + TS + 8) * sizeof(C);
};

template <typename S, typename C, int TS>
__global__ void __launch_bounds__(kNTP) k_panel_blk(View<S> V, int64_t m, int64_t top, int64_t k,
                                                  TreeWs<C> ws, int64_t ws_bstride,
                                                  int64_t a_bstride) {
    using CV = Conv<S, C>;
    using PB = PanelBlk<C, TS>;
    constexpr int NB = PB::NB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *sm = (C *)smem_raw;
    C *tau = sm + PB::UNION;
    __shared__ int s_old;

    const int64_t b = blockIdx.y;
    V.base += b * a_bstride;
    ws.nodes += b * ws_bstride;
    ws.R += b * ws_bstride;
    ws.cnt = (int *)((char *)ws.cnt + b * ws_bstride * (int64_t)sizeof(C));
    const int64_t l = blockIdx.x;
    const int tid = threadIdx.x;
    const int64_t ts2 = (int64_t)TS * TS;
    auto house = [](C a, C s, C &bb, C &t, C &sc) { house_scalars(a, s, bb, t, sc); };
    unsigned long long *trc = g_panel_trace && b == 0 && l < 64 ? g_panel_trace + l * 8 : nullptr;
    auto mark = [&](int ph) {
        if (trc && tid == 0) trc[ph] = gtimer_ns();
    };

    // ---- leaf: blocked QR of view tile (top + l, k) ----
    {
        constexpr int lda = PB::LDL;
        C *A = sm;
        C *aux = A + TS * lda;
        mark(0);
        const int64_t r0 = (top + l) * TS, c0 = k * TS;
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            int r, c;
            if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % TS; r = idx / TS; }
            A[c * lda + r] = CV::ld(*V.ptr(r0 + r, c0 + c));
        }
        __syncthreads();
        mark(1);
        C *Rg = ws.R + l * ts2;
        // R column blocks are final right after their sub-panel: save them, then T
        // may reuse the upper triangle (qr_blocked writes T block column j0 there).
        blk::qr_blocked<C, TS, false, kNTP>(A, lda, tau, A, lda, aux, house,
            [&](int j0) {
                for (int idx = tid; idx < TS * NB; idx += kNTP) {
                    const int c = j0 + idx / TS, r = idx % TS;
                    Rg[c * TS + r] = (r <= c) ? A[c * lda + r] : C(0);
                }
                __syncthreads();
            }, (g_panel_trace && b == 0 && l == 0) ? g_panel_trace + 64 * 9 * 8 : nullptr);
        mark(4);
        // Vk[r][i] = V(r, i);  Um[i][r] = U(r, i) = sum_{j=i..r} V(r,j) T(i,j)
        C *Vk = ws.Vk(l), *Um = ws.Um(l);
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int r = idx / TS, i = idx % TS;
            Vk[idx] = (r > i) ? A[i * lda + r] : (r == i ? C(1) : C(0));
        }
        blk::sgemm<C, 4, 4, kNTP>(TS, TS, TS,
            [&](int r, int j) { return r == j ? C(1) : (r > j ? A[j * lda + r] : C(0)); },   // V(r, j)
            [&](int j, int i) { return j >= i ? A[j * lda + i] : C(0); },                   // T(i, j)
            [&](int r, int i, C v) { Um[i * TS + r] = v; });
        __syncthreads();
        mark(5);
    }

    // ---- tree: climb while we are the second arrival ----
    const int L = tree_levels(m);
    int64_t node = l;
    for (int j = 1; j <= L; ++j) {
        const int64_t parent = node >> 1;
        const bool has_right = ((parent << 1) + 1) < tree_count(m, j - 1);
        if (has_right) {
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                int *cptr = ws.cnt + tree_offset(m, j) - m + parent;
                s_old = atomicAdd(cptr, 1);
                if (s_old == 1) *cptr = 0;   // self-cleaning for the next launch
                __threadfence();
            }
            __syncthreads();
            if (s_old == 0) return;
            trc = g_panel_trace && b == 0 && parent < 64 ? g_panel_trace + (64 + j * 64 + parent) * 8 : nullptr;
            mark(0);
            const int64_t a = (parent << 1) << (j - 1);
            const int64_t bb = ((parent << 1) + 1) << (j - 1);
            const C *Ra_g = ws.R + a * ts2, *Rb_g = ws.R + bb * ts2;
            C *Rg = ws.R + a * ts2;
            const int64_t slot = tree_offset(m, j) + parent;
            C *Vk = ws.Vk(slot), *Um = ws.Um(slot), *Tt = ws.Tt(slot);
            if constexpr (PB::TT_BLOCKED) {
                constexpr int lda = PB::LDT;
                C *A = sm;
                C *aux = A + TS * lda;
                for (int idx = tid; idx < TS * TS; idx += kNTP) {
                    const int c = idx / TS, r = idx % TS;
                    A[c * lda + r] = (r <= c) ? __ldcg(Ra_g + idx) : C(0);
                    A[c * lda + TS + r] = (r <= c) ? __ldcg(Rb_g + idx) : C(0);
                }
                __syncthreads();
                mark(1);
                blk::qr_blocked<C, TS, true, kNTP>(A, lda, tau, A, lda, aux, house,
                    [&](int j0) {
                        for (int idx = tid; idx < TS * NB; idx += kNTP) {
                            const int c = j0 + idx / TS, r = idx % TS;
                            Rg[c * TS + r] = (r <= c) ? A[c * lda + r] : C(0);
                        }
                        __syncthreads();
                    });
                mark(4);
                for (int idx = tid; idx < TS * TS; idx += kNTP) {
                    const int r = idx / TS, i = idx % TS;   // Vk[r][i] = Vb(r,i); Tt[r][i] = T(r,i)
                    Vk[idx] = (r <= i) ? A[i * lda + TS + r] : C(0);
                    Tt[idx] = (r <= i) ? A[i * lda + r] : C(0);
                }
                // TT update X_bot -= Vb (T^T W): Vb in the transposed operand layout
                for (int idx = tid; idx < TS * TS; idx += kNTP) {
                    const int i = idx / TS, r = idx % TS;
                    Um[idx] = (r <= i) ? A[i * lda + TS + r] : C(0);
                }
                __syncthreads();
            } else {
                constexpr int PK = PB::PK;
                C *Rt = sm, *Rb = sm + PK, *Tp = sm + 2 * PK;
                for (int idx = tid; idx < TS * TS; idx += kNTP) {
                    const int c = idx / TS, r = idx % TS;
                    if (r <= c) {
                        Rt[pk(r, c)] = __ldcg(Ra_g + idx);
                        Rb[pk(r, c)] = __ldcg(Rb_g + idx);
                    }
                }
                __syncthreads();
                mark(1);
                panel::tt_qr_la<C, TS, kNTP>(Rt, Rb, tau, house);
                for (int idx = tid; idx < TS * TS; idx += kNTP) {
                    const int c = idx / TS, r = idx % TS;
                    Rg[idx] = (r <= c) ? Rt[pk(r, c)] : C(0);
                }
                for (int idx = tid; idx < TS * TS; idx += kNTP) {
                    const int jj = idx / TS, i = idx % TS;
                    if (i < jj) {
                        const C *vi = Rb + pk(0, i), *vj = Rb + pk(0, jj);
                        C s0 = C(0);
                        for (int r = 0; r <= i; ++r) s0 += vi[r] * vj[r];
                        Tp[pk(i, jj)] = s0;
                    }
                }
                __syncthreads();
                panel::build_T_rec<C, TS, kNTP>(tau, Rt, [&](int i, int jj) -> C & { return Tp[pk(i, jj)]; });
                mark(4);
                for (int idx = tid; idx < TS * TS; idx += kNTP) {
                    const int r = idx / TS, i = idx % TS;
                    Vk[idx] = (r <= i) ? Rb[pk(r, i)] : C(0);
                    Tt[idx] = (r <= i) ? Tp[pk(r, i)] : C(0);
                }
                for (int idx = tid; idx < TS * TS; idx += kNTP) {   // Vb, transposed operand layout
                    const int i = idx / TS, r = idx % TS;
                    Um[idx] = (r <= i) ? Rb[pk(r, i)] : C(0);
                }
                __syncthreads();
            }
            mark(5);
        }
        node = parent;
    }
    __syncthreads();
    if (L == 0 || node == 0) {
        const C *Rg = ws.R;
        const int64_t r0 = top * TS, c0 = k * TS;
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            int r, c;
            if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % TS; r = idx / TS; }
            if (r <= c) *V.ptr(r0 + r, c0 + c) = CV::st(__ldcg(Rg + c * TS + r));
        }
    }
}

// ---------------------------------------------------------------------------
// Per-level panel kernels (ts >= 16).  Same node math as k_panel_blk, but one
// launch per tree level, so the trailing update of level j (on a second
// stream) can start as soon as level j's reflectors exist: the leaf-level
// update -- the largest -- overlaps the whole TT climb.

template <typename S, typename C, int TS>
__device__ __forceinline__ void write_root_R(const View<S> &V, const C *Rg, int64_t top, int64_t k) {
    using CV = Conv<S, C>;
    const int64_t r0 = top * TS, c0 = k * TS;
    for (int idx = threadIdx.x; idx < TS * TS; idx += blockDim.x) {
        int r, c;
        if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % TS; r = idx / TS; }
        if (r <= c) *V.ptr(r0 + r, c0 + c) = CV::st(__ldcg(Rg + c * TS + r));
    }
}

// Deferred compact-WY factors.  The tree climb only needs each node's R, so
// with DEFER the node kernels stop after the factorisation: they store V (Vk
// slot) and tau (first TS entries of the Tt slot), and k_node_tu -- launched
// on the trailing stream, off the panel's critical path -- builds T from
// G = V^T V (build_T_rec) and U = V T^T for the level's trailing update.
template <typename C, int TS>
struct NodeTU {
    static constexpr int LD = TS + 1;
    static constexpr size_t smem = (size_t)(2 * TS * LD + TS * TS / 4 + TS) * sizeof(C);
    static constexpr bool ok = smem <= 200 * 1024;
};

// With `img` (tensor-core trailing update, stage1_apply_tc.cu) the products
// are written as pre-split, pre-swizzled K-major TF32 operand images instead
// of Um / Tt: per node slot three A images of 2 ts^2 floats -- V^T (rows i,
// K = r), then for a leaf U (rows r, K = i), for a TT node T^T and U -- each
// K-block (32 of K) stored as [hi: ts rows x 32][lo: ts rows x 32].
template <typename C, int TS>
__device__ __forceinline__ void img_put(C *im, int m, int k, C v) {
    if constexpr (sizeof(C) == 4) {
        float h, l;
        tc::split3(v, h, l);
        const int o = (k >> 5) * (2 * TS * 32) + m * 32 + ((((k & 31) >> 2) ^ (m & 7)) << 2) + (k & 3);
        im[o] = h;
        im[o + TS * 32] = l;
    }
}

template <typename C, int TS>
__global__ void __launch_bounds__(kNTP) k_node_tu(C *nodes, int64_t slot0, int64_t ws_bstride,
                                                 bool tt, C *img) {
    using NT_ = NodeTU<C, TS>;
    constexpr int LD = NT_::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *Vs = (C *)smem_raw;                 // Vs[i * LD + r] = V(r, i)
    C *Ts = Vs + TS * LD;                  // Ts[j * LD + i] = T(i, j)
    C *tmp = Ts + TS * LD;
    C *tau = tmp + TS * TS / 4;
    const int tid = threadIdx.x;
    const int64_t ts2 = (int64_t)TS * TS;
    C *base = nodes + blockIdx.y * ws_bstride + (slot0 + blockIdx.x) * 3 * ts2;
    C *Vk = base, *Um = base + ts2, *Tt = base + 2 * ts2;
    C *im = img ? img + blockIdx.y * ws_bstride + (slot0 + blockIdx.x) * 6 * ts2 : nullptr;
    for (int idx = tid; idx < TS * TS; idx += kNTP) {
        const int r = idx / TS, i = idx % TS;
        Vs[i * LD + r] = __ldcg(Vk + idx);
    }
    for (int i = tid; i < TS; i += kNTP) tau[i] = __ldcg(Tt + i);
    __syncthreads();
    // strictly upper G = V^T V (for TT nodes V = [I; Vb]: the identity adds only
    // to the diagonal, so Vk = Vb gives the same G)
    blk::sgemm<C, 4, 4, kNTP>(TS, TS, TS,
        [&](int i, int r) { return Vs[i * LD + r]; },
        [&](int r, int j) { return Vs[j * LD + r]; },
        [&](int i, int j, C v) { if (i < j) Ts[j * LD + i] = v; });
    __syncthreads();
    panel::build_T_rec<C, TS, kNTP>(tau, tmp, [&](int i, int j) -> C & { return Ts[j * LD + i]; });
    __syncthreads();
    if (im) {
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int m = idx / TS, kk = idx % TS;
            img_put<C, TS>(im, m, kk, Vs[m * LD + kk]);                        // V^T: (i, r) = V(r, i)
            if (tt) img_put<C, TS>(im + 2 * ts2, m, kk, kk <= m ? Ts[m * LD + kk] : C(0));   // T^T: (r, i) = T(i, r)
        }
        C *imU = im + (tt ? 4 : 2) * ts2;
        blk::sgemm<C, 4, 4, kNTP>(TS, TS, TS,
            [&](int r, int j) { return Vs[j * LD + r]; },
            [&](int j, int i) { return j >= i ? Ts[j * LD + i] : C(0); },
            [&](int r, int i, C v) { img_put<C, TS>(imU, r, i, v); });
        return;
    }
    if (tt) {
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int r = idx / TS, i = idx % TS;   // Tt[r][i] = T(r, i)
            Tt[idx] = (r <= i) ? Ts[i * LD + r] : C(0);
        }
        // TT nodes apply X_bot -= Vb (T^T W) (stage1_apply.cu): no U, but Vb
        // in the transposed operand layout, Um[i][r] = Vb(r, i)
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int i = idx / TS, r = idx % TS;
            Um[idx] = Vs[i * LD + r];
        }
        return;
    }
    // U(r, i) = sum_{j >= i} V(r, j) T(i, j)
    blk::sgemm<C, 4, 4, kNTP>(TS, TS, TS,
        [&](int r, int j) { return Vs[j * LD + r]; },
        [&](int j, int i) { return j >= i ? Ts[j * LD + i] : C(0); },
        [&](int r, int i, C v) { Um[i * TS + r] = v; });
}

// Leaves: grid (m, batch).
template <typename S, typename C, int TS, bool DEFER>
__global__ void __launch_bounds__(kNTP) k_panel_leaf(View<S> V, int64_t m, int64_t top, int64_t k,
                                                    TreeWs<C> ws, int64_t ws_bstride,
                                                    int64_t a_bstride) {
    using CV = Conv<S, C>;
    using PB = PanelBlk<C, TS>;
    constexpr int NB = PB::NB;
    constexpr int lda = PB::LDL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *sm = (C *)smem_raw;
    C *tau = sm + PB::UNION;
    const int64_t b = blockIdx.y, l = blockIdx.x;
    V.base += b * a_bstride;
    ws.nodes += b * ws_bstride;
    ws.R += b * ws_bstride;
    const int tid = threadIdx.x;
    const int64_t ts2 = (int64_t)TS * TS;
    auto house = [](C a, C s, C &bb, C &t, C &sc) { house_scalars(a, s, bb, t, sc); };
    C *A = sm, *aux = A + TS * lda;
    const int64_t r0 = (top + l) * TS, c0 = k * TS;
    for (int idx = tid; idx < TS * TS; idx += kNTP) {
        int r, c;
        if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % TS; r = idx / TS; }
        A[c * lda + r] = CV::ld(*V.ptr(r0 + r, c0 + c));
    }
    __syncthreads();
    C *Rg = ws.R + l * ts2;
    blk::qr_blocked<C, TS, false, kNTP, !DEFER>(A, lda, tau, A, lda, aux, house, [&](int j0) {
        for (int idx = tid; idx < TS * NB; idx += kNTP) {
            const int c = j0 + idx / TS, r = idx % TS;
            Rg[c * TS + r] = (r <= c) ? A[c * lda + r] : C(0);
        }
        __syncthreads();
    });
    C *Vk = ws.Vk(l), *Um = ws.Um(l);
    for (int idx = tid; idx < TS * TS; idx += kNTP) {
        const int r = idx / TS, i = idx % TS;
        Vk[idx] = (r > i) ? A[i * lda + r] : (r == i ? C(1) : C(0));
    }
    if constexpr (DEFER) {
        for (int i = tid; i < TS; i += kNTP) ws.Tt(l)[i] = tau[i];
    } else {
        blk::sgemm<C, 4, 4, kNTP>(TS, TS, TS,
            [&](int r, int j) { return r == j ? C(1) : (r > j ? A[j * lda + r] : C(0)); },
            [&](int j, int i) { return j >= i ? A[j * lda + i] : C(0); },
            [&](int r, int i, C v) { Um[i * TS + r] = v; });
    }
    if (m == 1) {                         // the leaf is the root
        __syncthreads();
        write_root_R<S, C, TS>(V, Rg, top, k);
    }
}

// Two-tile leaves (fp32 compute, ts = 128): super-leaf l factors the dense
// 2ts x ts panel of tile rows top+2l and top+2l+1 (the second a zero tile
// past the panel's end) in one blocked QR -- the leaf level and the first
// TT level of the single-tile tree in one node.  V rows 0..ts-1 go to the
// leaf's Vk slot, rows ts..2ts-1 to the leaf2 region; tau into Tt.
template <typename C, int TS>
struct Leaf2 {
    static constexpr int LD = 2 * TS + 1;
    static constexpr int AUX = blk::aux_elems<C, TS, 2 * TS>();
    static constexpr size_t smem = (size_t)(TS * LD + AUX + TS + 8) * sizeof(C);
    static constexpr bool ok = sizeof(C) == 4 && TS >= 32 && smem <= 227 * 1024;
};

template <typename S, typename C, int TS, bool FULLT>
__global__ void __launch_bounds__(kNTP) k_panel_leaf2(View<S> V, int64_t m, int64_t m2, int64_t top,
                                                     int64_t k, TreeWs<C> ws, C *ext,
                                                     int64_t ws_bstride, int64_t a_bstride) {
    using CV = Conv<S, C>;
    using L2 = Leaf2<C, TS>;
    constexpr int NB = blk::NBsel<C, TS>::v;
    constexpr int lda = L2::LD;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *A = (C *)smem_raw;
    C *aux = A + TS * lda;
    C *tau = aux + L2::AUX;
    const int64_t b = blockIdx.y, l = blockIdx.x;
    V.base += b * a_bstride;
    ws.nodes += b * ws_bstride;
    ws.R += b * ws_bstride;
    ext += b * ws_bstride;
    const int tid = threadIdx.x;
    const int64_t ts2 = (int64_t)TS * TS;
    auto house = [](C a, C s, C &bb, C &t, C &sc) { house_scalars(a, s, bb, t, sc); };
    const int64_t t0 = top + 2 * l, t1 = t0 + 1;
    const bool two = t1 < top + m;
    const int64_t c0 = k * TS;
    for (int idx = tid; idx < 2 * TS * TS; idx += kNTP) {
        int r, c;
        if (V.rs == 1) { r = idx % (2 * TS); c = idx / (2 * TS); } else { c = idx % TS; r = idx / TS; }
        const int64_t gr = (r < TS ? t0 : t1) * TS + (r % TS);
        A[c * lda + r] = (r < TS || two) ? CV::ld(*V.ptr(gr, c0 + c)) : C(0);
    }
    __syncthreads();
    C *Rg = ws.R + l * ts2;
    // FULLT: the whole compact-WY T comes out of the factorisation, so the
    // leaf update waits only for the short U = V T^T kernel (k_leaf2_u);
    // otherwise k_node_tu2 builds T and U (less work in total: batches)
    blk::qr_blocked<C, TS, false, kNTP, FULLT, 2 * TS>(A, lda, tau, A, lda, aux, house, [&](int j0) {
        for (int idx = tid; idx < TS * NB; idx += kNTP) {
            const int c = j0 + idx / TS, r = idx % TS;
            Rg[c * TS + r] = (r <= c) ? A[c * lda + r] : C(0);
        }
        __syncthreads();
    });
    C *Vk = ws.Vk(l), *V2 = ext + l * 2 * ts2;
    for (int idx = tid; idx < TS * TS; idx += kNTP) {
        const int r = idx / TS, i = idx % TS;
        Vk[idx] = (r > i) ? A[i * lda + r] : (r == i ? C(1) : C(0));
        V2[idx] = A[i * lda + TS + r];
    }
    C *Tg = ws.Tt(l);
    if constexpr (FULLT) {                // T (column-major, upper; zeros below)
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int jj = idx / TS, i = idx % TS;
            Tg[idx] = (i <= jj) ? A[jj * lda + i] : C(0);
        }
    } else {
        for (int i = tid; i < TS; i += kNTP) Tg[i] = tau[i];
    }
    if (m2 == 1) {                        // the super-leaf is the root
        __syncthreads();
        write_root_R<S, C, TS>(V, Rg, top, k);
    }
}

// T and U of two-tile leaves: G = V^T V over 2ts rows, T by recursive
// merging, U = V T^T (rows 0..ts-1 into Um, ts..2ts-1 into the leaf2 region).
template <typename C, int TS>
struct NodeTU2 {
    static constexpr int LD = 2 * TS + 1, LT = TS + 1;
    static constexpr size_t smem = (size_t)(TS * LD + TS * LT + TS * TS / 4 + TS) * sizeof(C);
};
template <typename C, int TS>
__global__ void __launch_bounds__(kNTP) k_node_tu2(C *nodes, C *ext, int64_t ws_bstride) {
    using NT_ = NodeTU2<C, TS>;
    constexpr int LD = NT_::LD, LT = NT_::LT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *Vs = (C *)smem_raw;                 // Vs[i * LD + r] = V(r, i), r < 2 TS
    C *Ts = Vs + TS * LD;                  // Ts[j * LT + i] = T(i, j)
    C *tmp = Ts + TS * LT;
    C *tau = tmp + TS * TS / 4;
    const int tid = threadIdx.x;
    const int64_t ts2 = (int64_t)TS * TS, l = blockIdx.x;
    C *base = nodes + blockIdx.y * ws_bstride + l * 3 * ts2;
    C *Vk = base, *Um = base + ts2, *Tt = base + 2 * ts2;
    C *V2 = ext + blockIdx.y * ws_bstride + l * 2 * ts2, *U2 = V2 + ts2;
    for (int idx = tid; idx < TS * TS; idx += kNTP) {
        const int r = idx / TS, i = idx % TS;
        Vs[i * LD + r] = __ldcg(Vk + idx);
        Vs[i * LD + TS + r] = __ldcg(V2 + idx);
    }
    for (int i = tid; i < TS; i += kNTP) tau[i] = __ldcg(Tt + i);
    __syncthreads();
    blk::sgemm<C, 4, 4, kNTP>(TS, TS, 2 * TS,
        [&](int i, int r) { return Vs[i * LD + r]; },
        [&](int r, int j) { return Vs[j * LD + r]; },
        [&](int i, int j, C v) { if (i < j) Ts[j * LT + i] = v; });
    __syncthreads();
    panel::build_T_rec<C, TS, kNTP>(tau, tmp, [&](int i, int j) -> C & { return Ts[j * LT + i]; });
    __syncthreads();
    // U(r, i) = sum_{j >= i} V(r, j) T(i, j)
    blk::sgemm<C, 4, 4, kNTP>(2 * TS, TS, TS,
        [&](int r, int j) { return Vs[j * LD + r]; },
        [&](int j, int i) { return j >= i ? Ts[j * LT + i] : C(0); },
        [&](int r, int i, C v) {
            if (r < TS) Um[i * TS + r] = v; else U2[i * TS + (r - TS)] = v;
        });
}

// U = V T^T of two-tile leaves from the full T their panel kernel wrote:
// grid (leaves, U2_SLICES, batch), each CTA a slice of the 2ts rows.
constexpr int kU2Slices = 4;
template <typename C, int TS>
struct LeafU2 {
    static constexpr int RS = 2 * TS / kU2Slices;         // rows per CTA
    static constexpr int LT = TS + 1, LV = RS + 1;
    static constexpr size_t smem = (size_t)(TS * LT + TS * LV) * sizeof(C);
};
template <typename C, int TS>
__global__ void __launch_bounds__(kNTP) k_leaf2_u(C *nodes, C *ext, int64_t ws_bstride) {
    using LU = LeafU2<C, TS>;
    constexpr int RS = LU::RS, LT = LU::LT, LV = LU::LV;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *Ts = (C *)smem_raw;                 // Ts[j * LT + i] = T(i, j)
    C *Vs = Ts + TS * LT;                  // Vs[j * LV + r] = V(r0 + r, j)
    const int tid = threadIdx.x;
    const int64_t ts2 = (int64_t)TS * TS, l = blockIdx.x;
    const int r0 = blockIdx.y * RS;
    C *base = nodes + blockIdx.z * ws_bstride + l * 3 * ts2;
    const C *Vk = base, *Tg = base + 2 * ts2;
    C *Um = base + ts2;
    C *V2 = ext + blockIdx.z * ws_bstride + l * 2 * ts2, *U2 = V2 + ts2;
    for (int idx = tid; idx < TS * TS; idx += kNTP) Ts[(idx / TS) * LT + idx % TS] = __ldcg(Tg + idx);
    for (int idx = tid; idx < RS * TS; idx += kNTP) {
        const int r = idx / TS, j = idx % TS, gr = r0 + r;
        Vs[j * LV + r] = gr < TS ? __ldcg(Vk + gr * TS + j) : __ldcg(V2 + (gr - TS) * TS + j);
    }
    __syncthreads();
    // U(r, i) = sum_{j >= i} V(r, j) T(i, j)
    blk::sgemm<C, 4, 4, kNTP>(RS, TS, TS,
        [&](int r, int j) { return Vs[j * LV + r]; },
        [&](int j, int i) { return j >= i ? Ts[j * LT + i] : C(0); },
        [&](int r, int i, C v) {
            const int gr = r0 + r;
            if (gr < TS) Um[i * TS + gr] = v; else U2[i * TS + (gr - TS)] = v;
        });
}

// TT nodes of level j: grid (pairs, batch); node p combines the R factors of
// leaves a = (2p) << (j-1) and bb = (2p+1) << (j-1).
template <typename S, typename C, int TS, bool DEFER>
__global__ void __launch_bounds__(kNTP) k_panel_tt(View<S> V, int64_t m, int64_t top, int64_t k, int j,
                                                  TreeWs<C> ws, int64_t ws_bstride,
                                                  int64_t a_bstride) {
    using PB = PanelBlk<C, TS>;
    constexpr int NB = PB::NB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *sm = (C *)smem_raw;
    C *tau = sm + PB::UNION;
    const int64_t b = blockIdx.y, parent = blockIdx.x;
    V.base += b * a_bstride;
    ws.nodes += b * ws_bstride;
    ws.R += b * ws_bstride;
    const int tid = threadIdx.x;
    const int64_t ts2 = (int64_t)TS * TS;
    auto house = [](C a, C s, C &bb, C &t, C &sc) { house_scalars(a, s, bb, t, sc); };
    const int64_t a = (parent << 1) << (j - 1);
    const int64_t bb = ((parent << 1) + 1) << (j - 1);
    const C *Ra_g = ws.R + a * ts2, *Rb_g = ws.R + bb * ts2;
    C *Rg = ws.R + a * ts2;
    const int64_t slot = tree_offset(m, j) + parent;
    C *Vk = ws.Vk(slot), *Um = ws.Um(slot), *Tt = ws.Tt(slot);
    if constexpr (PB::TT_BLOCKED) {
        constexpr int lda = PB::LDT;
        C *A = sm, *aux = A + TS * lda;
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int c = idx / TS, r = idx % TS;
            A[c * lda + r] = (r <= c) ? __ldcg(Ra_g + idx) : C(0);
            A[c * lda + TS + r] = (r <= c) ? __ldcg(Rb_g + idx) : C(0);
        }
        __syncthreads();
        unsigned long long *pst = (g_panel_trace && b == 0 && parent == 0) ? g_panel_trace : nullptr;
        if (pst && tid == 0) pst[200] = blk::stamp_now();
        blk::qr_blocked<C, TS, true, kNTP, !DEFER>(A, lda, tau, A, lda, aux, house, [&](int j0) {
            for (int idx = tid; idx < TS * NB; idx += kNTP) {
                const int c = j0 + idx / TS, r = idx % TS;
                Rg[c * TS + r] = (r <= c) ? A[c * lda + r] : C(0);
            }
            __syncthreads();
        }, pst);
        if (pst && tid == 0) pst[201] = blk::stamp_now();
        if constexpr (DEFER) {
            for (int idx = tid; idx < TS * TS; idx += kNTP) {
                const int r = idx / TS, i = idx % TS;
                Vk[idx] = (r <= i) ? A[i * lda + TS + r] : C(0);
            }
            for (int i = tid; i < TS; i += kNTP) Tt[i] = tau[i];
        } else {
            for (int idx = tid; idx < TS * TS; idx += kNTP) {
                const int r = idx / TS, i = idx % TS;
                Vk[idx] = (r <= i) ? A[i * lda + TS + r] : C(0);
                Tt[idx] = (r <= i) ? A[i * lda + r] : C(0);
            }
            // TT update X_bot -= Vb (T^T W): Vb in the transposed operand layout
            for (int idx = tid; idx < TS * TS; idx += kNTP) {
                const int i = idx / TS, r = idx % TS;
                Um[idx] = (r <= i) ? A[i * lda + TS + r] : C(0);
            }
        }
    } else {
        constexpr int PK = PB::PK;
        C *Rt = sm, *Rb = sm + PK, *Tp = sm + 2 * PK;
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int c = idx / TS, r = idx % TS;
            if (r <= c) {
                Rt[pk(r, c)] = __ldcg(Ra_g + idx);
                Rb[pk(r, c)] = __ldcg(Rb_g + idx);
            }
        }
        __syncthreads();
        panel::tt_qr_la<C, TS, kNTP>(Rt, Rb, tau, house);
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int c = idx / TS, r = idx % TS;
            Rg[idx] = (r <= c) ? Rt[pk(r, c)] : C(0);
        }
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int jj = idx / TS, i = idx % TS;
            if (i < jj) {
                const C *vi = Rb + pk(0, i), *vj = Rb + pk(0, jj);
                C s0 = C(0);
                for (int r = 0; r <= i; ++r) s0 += vi[r] * vj[r];
                Tp[pk(i, jj)] = s0;
            }
        }
        __syncthreads();
        panel::build_T_rec<C, TS, kNTP>(tau, Rt, [&](int i, int jj) -> C & { return Tp[pk(i, jj)]; });
        for (int idx = tid; idx < TS * TS; idx += kNTP) {
            const int r = idx / TS, i = idx % TS;
            Vk[idx] = (r <= i) ? Rb[pk(r, i)] : C(0);
            Tt[idx] = (r <= i) ? Tp[pk(r, i)] : C(0);
        }
        for (int idx = tid; idx < TS * TS; idx += kNTP) {   // Vb, transposed operand layout
            const int i = idx / TS, r = idx % TS;
            Um[idx] = (r <= i) ? Rb[pk(r, i)] : C(0);
        }
    }
    if (gridDim.x == 1 && ((int64_t)1 << j) >= m) {   // the root level: R into the band tile
        __syncthreads();
        write_root_R<S, C, TS>(V, Rg, top, k);
    }
}

// Overlapped stage 1: panel levels on `st`, trailing levels on a second
// stream, one event per level; the next side's panel waits for the whole
// trailing update (its panel is the top tile row/column of that update).
template <typename S, typename C, int TS>
static cudaError_t run_levels(S *a, int64_t n, int64_t batch, int64_t a_bstride, void *wsp,
                              cudaStream_t st, double *pms, double *tms, bool timed) {
    using PB = PanelBlk<C, TS>;
    constexpr bool DEFER = NodeTU<C, TS>::ok;
    const int64_t N = n / TS;
    const int64_t ws_elems = (int64_t)tree_ws_elems<C>(N, TS);
    const int64_t ts2 = (int64_t)TS * TS;
    TreeWs<C> ws;
    ws.nodes = (C *)wsp;
    ws.R = ws.nodes + tree_slots(N) * 3 * ts2;
    ws.cnt = (int *)(ws.R + N * ts2);
    ws.ts2 = ts2;
    cudaError_t err;
    const size_t psm = PB::smem;
    // Trailing update on the FMA pipe by default.  BSVD_TC=1 selects the
    // tcgen05 3xTF32 kernels (fp32 compute, ts = 128): ~1.8x faster trailing
    // update, but the tensor-core accumulation loses accuracy -- 6e-5 of
    // sigma_max at n = 8192 against 2e-7 on the FMA path.
    C *img = ws.nodes + tree_img_offset<C>(N, TS);
    const bool use_tc = DEFER && tree_tc<C>(TS) && getenv("BSVD_TC") && atoi(getenv("BSVD_TC")) != 0;
    // T and U of `count` nodes from slot0 on, ahead of their trailing level (st2)
    auto node_tu = [&](int64_t slot0, int64_t count, bool tt, cudaStream_t s2) -> cudaError_t {
        if (!DEFER || count <= 0) return cudaSuccess;
        k_node_tu<C, TS><<<dim3((unsigned)count, (unsigned)batch), kNTP, NodeTU<C, TS>::smem, s2>>>(
            ws.nodes, slot0, ws_elems, tt, use_tc ? img : nullptr);
        bsvd_host::count_launch();
        return cudaGetLastError();
    };
    if ((err = ensure_smem(k_panel_leaf<S, C, TS, DEFER>, psm)) != cudaSuccess) return err;
    if ((err = ensure_smem(k_panel_tt<S, C, TS, DEFER>, psm)) != cudaSuccess) return err;
    if ((err = ensure_smem(k_panel_tt<S, C, TS, false>, psm)) != cudaSuccess) return err;
    if (DEFER && (err = ensure_smem(k_node_tu<C, TS>, NodeTU<C, TS>::smem)) != cudaSuccess) return err;
    // per-device streams and events, created once and reused by every call
    // (the enqueue of one call holds the device's lock: calls from several
    // host threads serialise their enqueue and never share in-flight events)
    TreeCtx *tcx = nullptr;
    if ((err = tree_ctx(tcx)) != cudaSuccess) return err;
    std::lock_guard<std::mutex> enqueue_lock(tcx->mu);
    cudaStream_t caller = st, st2 = tcx->st2, st1 = nullptr;
    if (!getenv("BSVD_PANEL_NOPRIO")) {       // panel levels on a high-priority stream: the
                                              // critical path gets the next free SM slots
        st1 = tcx->st1;
        st = st1;
    }
    // BSVD_S1_TRACE=k: event timeline of sweep side k (RQ) on the three streams
    const int trace_k = getenv("BSVD_S1_TRACE") ? atoi(getenv("BSVD_S1_TRACE")) : -1;
    std::vector<std::pair<const char *, cudaEvent_t>> tl;
    int tl_side = -1;
    auto tlmark = [&](const char *what, cudaStream_t s2_) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s2_);
        tl.push_back({what, e});
    };
    // T and U of a level on a third stream as soon as the panel level exists,
    // so they overlap the previous level's trailing update; the update of
    // level j (st2) then waits only for its own factors.
    // (high priority: a level's factors must not queue behind the thousands
    // of CTAs of the previous level's update)
    cudaStream_t st3 = tcx->st3;
    // two-tile leaves (fp32 compute, ts = 128, FMA update path)
    C *ext = ws.nodes + tree_leaf2_offset<C>(N, TS);
    bool leaf2 = false;
    // full T in the leaf panel + short U kernel while the panel has many tile
    // rows (then the update chain, not the panel chain, bounds the side);
    // otherwise k_node_tu2 (less work on the panel chain)
    const int64_t ft_min = getenv("BSVD_LEAF_FT_MIN") ? atoll(getenv("BSVD_LEAF_FT_MIN")) : 32;
    bool leaf_fullt = false;
    if constexpr (Leaf2<C, TS>::ok && NodeTU2<C, TS>::smem <= 227 * 1024 && LeafU2<C, TS>::smem <= 227 * 1024)
        leaf2 = DEFER && !use_tc && !(getenv("BSVD_LEAF2") && atoi(getenv("BSVD_LEAF2")) == 0);
    if (leaf2) {
        if ((err = ensure_smem(k_panel_leaf2<S, C, TS, true>, Leaf2<C, TS>::smem)) != cudaSuccess) return err;
        if ((err = ensure_smem(k_panel_leaf2<S, C, TS, false>, Leaf2<C, TS>::smem)) != cudaSuccess) return err;
        if ((err = ensure_smem(k_leaf2_u<C, TS>, LeafU2<C, TS>::smem)) != cudaSuccess) return err;
        if ((err = ensure_smem(k_node_tu2<C, TS>, NodeTU2<C, TS>::smem)) != cudaSuccess) return err;
    }
    bool l2side = false;                                // the current side uses two-tile leaves
    int64_t mtiles = 0;                                 // its panel's tile rows
    const int Lmax0 = tree_levels(N);
    if ((err = tcx->reserve(2 * (Lmax0 + 1) + 1)) != cudaSuccess) return err;
    std::vector<cudaEvent_t> tuev(tcx->ev.begin(), tcx->ev.begin() + (Lmax0 + 1));
    std::vector<cudaEvent_t> *lvlp = nullptr;           // set below (panel level events)
    auto level_tu = [&](int j, int64_t slot0, int64_t count, bool tt) -> cudaError_t {
        cudaError_t e2;
        if (!DEFER || count <= 0) {
            cudaStreamWaitEvent(st2, (*lvlp)[j], 0);
            return cudaSuccess;
        }
        cudaStreamWaitEvent(st3, (*lvlp)[j], 0);
        if (tl_side) tlmark("  pre tu", st3);
        if (l2side && j == 0) {
            if constexpr (Leaf2<C, TS>::ok) {
                if (leaf_fullt)
                    k_leaf2_u<C, TS><<<dim3((unsigned)count, kU2Slices, (unsigned)batch), kNTP, LeafU2<C, TS>::smem, st3>>>(
                        ws.nodes, ext, ws_elems);
                else
                    k_node_tu2<C, TS><<<dim3((unsigned)count, (unsigned)batch), kNTP, NodeTU2<C, TS>::smem, st3>>>(
                        ws.nodes, ext, ws_elems);
                bsvd_host::count_launch();
                if ((e2 = cudaGetLastError()) != cudaSuccess) return e2;
            }
        } else if ((e2 = node_tu(slot0, count, tt, st3)) != cudaSuccess) {
            return e2;
        }
        cudaEventRecord(tuev[j], st3);
        if (tl_side) tlmark("  node_tu", st3);
        cudaStreamWaitEvent(st2, tuev[j], 0);
        return cudaSuccess;
    };
    auto apply_level0 = [&](bool lq, int64_t top, int64_t k, int64_t m, int j) -> cudaError_t {
        if constexpr (sizeof(C) == 4 && TS == 128) {
            if (use_tc)
                return launch_apply_level_tc<S>(a, n, batch, a_bstride, lq, top, k, m, (const float *)img,
                                                ws_elems, j, st2);
        }
        return launch_apply_level<S, C, TS>(a, n, batch, a_bstride, lq, top, k, m, ws.nodes, ws_elems, j, st2,
                                            l2side ? ext : nullptr, mtiles);
    };
    auto apply_level = [&](bool lq, int64_t top, int64_t k, int64_t m, int j) -> cudaError_t {
        if (tl_side) tlmark("    pre apply", st2);
        const cudaError_t e3 = apply_level0(lq, top, k, m, j);
        if (tl_side) tlmark("    apply", st2);
        return e3;
    };
    const int Lmax = tree_levels(N);
    std::vector<cudaEvent_t> lvl(tcx->ev.begin() + (Lmax0 + 1), tcx->ev.begin() + (Lmax0 + 1) + (Lmax + 1));
    lvlp = &lvl;
    cudaEvent_t done = tcx->ev[2 * (Lmax0 + 1)];
    cudaEventRecord(done, caller);             // both start after the caller's queued work
    std::vector<cudaEvent_t> tev;             // timing: (p0, p1) on st, (t0, t1) on st2 per side
    auto tmark = [&](cudaStream_t s) -> cudaEvent_t {
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        tev.push_back(e);
        return e;
    };
    struct Side { cudaEvent_t p0, p1, t0, t1; };
    std::vector<Side> sides;
    auto side = [&](int64_t k, bool lq) -> cudaError_t {
        View<S> V{a, lq ? n : 1, lq ? 1 : n};
        const int64_t top = lq ? k + 1 : k;
        if (top >= N) return cudaSuccess;
        const int64_t m = N - top;
        l2side = leaf2 && m >= 2;
        leaf_fullt = m >= ft_min;      // (never batch-dependent: batched == single, bit for bit)
        mtiles = m;
        const int64_t mt = l2side ? (m + 1) / 2 : m;      // tree leaves
        const int L = tree_levels(mt);
        const bool trail = (N - 1 - k) > 0;
        Side sd{};
        cudaStreamWaitEvent(st, done, 0);
        tl_side = (!lq && k == trace_k) ? 1 : 0;
        if (tl_side) tlmark("start", st);
        if (timed) sd.p0 = tmark(st);
        if (l2side) {
            if constexpr (Leaf2<C, TS>::ok)
            {
                if (leaf_fullt)
                    k_panel_leaf2<S, C, TS, true><<<dim3((unsigned)mt, (unsigned)batch), kNTP, Leaf2<C, TS>::smem, st>>>(
                        V, m, mt, top, k, ws, ext, ws_elems, a_bstride);
                else
                    k_panel_leaf2<S, C, TS, false><<<dim3((unsigned)mt, (unsigned)batch), kNTP, Leaf2<C, TS>::smem, st>>>(
                        V, m, mt, top, k, ws, ext, ws_elems, a_bstride);
            }
        } else {
            k_panel_leaf<S, C, TS, DEFER><<<dim3((unsigned)m, (unsigned)batch), kNTP, psm, st>>>(V, m, top, k, ws, ws_elems, a_bstride);
        }
        bsvd_host::count_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        cudaEventRecord(lvl[0], st);
        if (tl_side) tlmark("panel leaf", st);
        if (trail) {
            if (timed) sd.t0 = tmark(st2);
            if ((e = level_tu(0, 0, mt, false)) != cudaSuccess) return e;
            if ((e = apply_level(lq, top, k, mt, 0)) != cudaSuccess) return e;
        }
        int64_t cnt_prev = mt;
        for (int j = 1; j <= L; ++j) {
            const int64_t pairs = cnt_prev / 2;
            unsigned long long *qtrace = nullptr;
            if (tl_side && j == 1 && pairs > 0 && getenv("BSVD_TT_TRACE")) {
                cudaMalloc(&qtrace, 256 * 8);
                cudaMemsetAsync(qtrace, 0, 256 * 8, st);
                cudaMemcpyToSymbolAsync(g_panel_trace, &qtrace, sizeof(void *), 0, cudaMemcpyHostToDevice, st);
            }
            if (tl_side) tlmark("pre tt", st);
            // the root node builds its full T itself: no factor kernel between
            // the last panel node and the update the next side waits for
            const bool root_full = DEFER && !use_tc && j == L && pairs == 1;
            if (root_full) {
                k_panel_tt<S, C, TS, false><<<dim3(1u, (unsigned)batch), kNTP, psm, st>>>(V, mt, top, k, j, ws, ws_elems, a_bstride);
                bsvd_host::count_launch();
                if ((e = cudaGetLastError()) != cudaSuccess) return e;
            } else if (pairs > 0) {
                k_panel_tt<S, C, TS, DEFER><<<dim3((unsigned)pairs, (unsigned)batch), kNTP, psm, st>>>(V, mt, top, k, j, ws, ws_elems, a_bstride);
                bsvd_host::count_launch();
                if ((e = cudaGetLastError()) != cudaSuccess) return e;
            }
            cudaEventRecord(lvl[j], st);
            if (tl_side) tlmark("panel tt", st);
            if (qtrace) {
                void *null_ptr = nullptr;
                cudaMemcpyToSymbolAsync(g_panel_trace, &null_ptr, sizeof(void *), 0, cudaMemcpyHostToDevice, st);
                std::vector<unsigned long long> h(256);
                cudaMemcpyAsync(h.data(), qtrace, 256 * 8, cudaMemcpyDeviceToHost, st);
                cudaStreamSynchronize(st);
                const unsigned long long t0 = h[200];
                fprintf(stderr, "[tt node] col steps (us):");
                for (int c = 0; c < 128; c += 8) fprintf(stderr, " %d:%.1f", c, (h[c] - t0) * 1e-3);
                fprintf(stderr, "\n[tt node] subpanel end/T/update (us):");
                for (int q = 0; q < 12; ++q) fprintf(stderr, " %.1f", (h[128 + q] - t0) * 1e-3);
                fprintf(stderr, " | total %.1f raw %llu %llu %llu %llu\n", (h[201] - t0) * 1e-3, h[0], h[200], h[128], h[201]);
                cudaFree(qtrace);
            }
            if (trail && pairs > 0) {
                if ((e = level_tu(j, tree_offset(mt, j), root_full ? 0 : pairs, true)) != cudaSuccess) return e;
                if ((e = apply_level(lq, top, k, mt, j)) != cudaSuccess) return e;
            }
            cnt_prev = (mt + ((int64_t)1 << j) - 1) >> j;
        }
        if (timed) sd.p1 = tmark(st);
        if (trail) {
            if (timed) sd.t1 = tmark(st2);
            cudaEventRecord(done, st2);
        } else {
            cudaEventRecord(done, st);
        }
        if (timed) sides.push_back(sd);
        return cudaSuccess;
    };
    err = cudaSuccess;
    for (int64_t k = 0; k < N - 1 && err == cudaSuccess; ++k) {
        if ((err = side(k, false)) != cudaSuccess) break;
        err = side(k, true);
    }
    if (err == cudaSuccess) err = side(N - 1, false);
    cudaEventRecord(lvl[0], st);
    cudaStreamWaitEvent(caller, lvl[0], 0);    // stage 2 on the caller's stream sees
    cudaStreamWaitEvent(caller, done, 0);      // every panel and trailing update
    if (timed) {
        cudaStreamSynchronize(caller);
        for (const Side &sd : sides) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, sd.p0, sd.p1);
            *pms += ms;
            if (sd.t0) {
                cudaEventElapsedTime(&ms, sd.t0, sd.t1);
                *tms += ms;
            }
        }
        for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    if (!tl.empty()) {
        cudaStreamSynchronize(caller);
        for (auto &pe : tl) {
            float ms = 0.f;
            cudaError_t te = cudaEventSynchronize(pe.second);
            if (te == cudaSuccess) te = cudaEventElapsedTime(&ms, tl[0].second, pe.second);
            fprintf(stderr, "[s1 side %d] %-12s %8.1f us %s\n", trace_k, pe.first, ms * 1e3,
                    te == cudaSuccess ? "" : cudaGetErrorString(te));
        }
        for (auto &pe : tl) cudaEventDestroy(pe.second);
    }
    return err;
}

// ---------------------------------------------------------------------------
// Trailing kernel helpers.
//   acc[MR][NR] (+)= sum_k Ag[k][m] * Bs[k][c]   over the thread's microtile
// Ag: global ts x ts operand in [k][m] layout (m fastest), streamed through
// two smem chunk buffers of KC x TS.  Bs: smem [TS][CBP].
template <typename C, int TS, int CB, int MR, int NR, int KC>
__device__ __forceinline__ void gemm_acc(const C *__restrict__ Ag, const C *Bs, C *Abuf,
                                         C (&acc)[MR][NR], int tm, int tc) {
    constexpr int CBP = CB;
    constexpr int NCH = TS / KC;
    constexpr int CHUNK = KC * TS;
    constexpr int PER = (CHUNK + kNT - 1) / kNT;
    const int tid = threadIdx.x;
    C pre[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int idx = tid + q * kNT;
        pre[q] = (idx < CHUNK) ? __ldcg(Ag + idx) : C(0);
    }
#pragma unroll 1
    for (int ch = 0; ch < NCH; ++ch) {
        C *buf = Abuf + (ch & 1) * CHUNK;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = tid + q * kNT;
            if (idx < CHUNK) buf[idx] = pre[q];
        }
        __syncthreads();
        if (ch + 1 < NCH) {
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int idx = tid + q * kNT;
                pre[q] = (idx < CHUNK) ? __ldcg(Ag + (ch + 1) * CHUNK + idx) : C(0);
            }
        }
#pragma unroll 4
        for (int kk = 0; kk < KC; ++kk) {
            C a[MR], bv[NR];
#pragma unroll
            for (int i = 0; i < MR; ++i) a[i] = buf[kk * TS + tm * MR + i];
#pragma unroll
            for (int jx = 0; jx < NR; ++jx) bv[jx] = Bs[(ch * KC + kk) * CBP + tc * NR + jx];
#pragma unroll
            for (int i = 0; i < MR; ++i)
#pragma unroll
                for (int jx = 0; jx < NR; ++jx) acc[i][jx] += a[i] * bv[jx];
        }
        // the next iteration writes the other buffer; this one is rewritten
        // two chunks later, after the __syncthreads above.
    }
    __syncthreads();
}

template <typename S, typename C, int TS, int CB>
__device__ __forceinline__ void load_tile(const View<S> &V, int64_t r0, int64_t c0, int64_t cmax,
                                          C *X) {
    using CV = Conv<S, C>;
    for (int idx = threadIdx.x; idx < TS * CB; idx += kNT) {
        int r, c;
        if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % CB; r = idx / CB; }
        X[r * CB + c] = (c0 + c < cmax) ? CV::ld(*V.ptr(r0 + r, c0 + c)) : C(0);
    }
}

template <typename S, typename C, int TS, int CB>
__device__ __forceinline__ void store_tile(const View<S> &V, int64_t r0, int64_t c0, int64_t cmax,
                                           const C *X) {
    using CV = Conv<S, C>;
    for (int idx = threadIdx.x; idx < TS * CB; idx += kNT) {
        int r, c;
        if (V.rs == 1) { r = idx % TS; c = idx / TS; } else { c = idx % CB; r = idx / CB; }
        if (c0 + c < cmax) *V.ptr(r0 + r, c0 + c) = CV::st(X[r * CB + c]);
    }
}

// Trailing kernel.  Grid: ceil(ncols / CB) column blocks of the view's
// trailing columns [k+1)*TS, N*TS); rows top..top+m-1 (tile rows).
template <typename S, typename C, int TS>
__global__ void __launch_bounds__(kNT) k_trail_tree(View<S> V, int64_t m, int64_t top, int64_t k,
                                                   int64_t ncols, TreeWs<C> ws,
                                                   int64_t ws_bstride, int64_t a_bstride) {
    constexpr int CB = TileCfg<C>::elems / TS;
    constexpr int MR = 4;
    constexpr int NR = (TS * CB) / (kNT * MR);   // 4 (fp32) / 2 (fp64)
    constexpr int KC = (TS >= 16) ? 16 : TS;
    constexpr int TILE = TS * CB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C *sm = (C *)smem_raw;
    C *Abuf = sm;                   // 2 * KC * TS
    C *W = Abuf + 2 * KC * TS;      // TILE
    C *stack = W + TILE;            // depth * TILE
    __shared__ int st_lvl[24];
    __shared__ int64_t st_idx[24];

    const int64_t b = blockIdx.y;
    V.base += b * a_bstride;
    ws.nodes += b * ws_bstride;
    const int tid = threadIdx.x;
    const int tm = tid % (TS / MR), tc = tid / (TS / MR);
    const int64_t c0 = (int64_t)blockIdx.x * CB;          // relative to first trailing column
    const int64_t cbase = (k + 1) * TS;
    const int64_t cmax = cbase + ncols;
    const int L = tree_levels(m);
    int sp = 0;

    for (int64_t l = 0; l < m; ++l) {
        C *X = stack + sp * TILE;
        load_tile<S, C, TS, CB>(V, (top + l) * TS, cbase + c0, cmax, X);
        __syncthreads();
        // leaf: W = V^T X ; X -= U W
        {
            C acc[MR][NR];
#pragma unroll
            for (int i = 0; i < MR; ++i)
#pragma unroll
                for (int jx = 0; jx < NR; ++jx) acc[i][jx] = C(0);
            gemm_acc<C, TS, CB, MR, NR, KC>(ws.Vk(l), X, Abuf, acc, tm, tc);
#pragma unroll
            for (int i = 0; i < MR; ++i)
#pragma unroll
                for (int jx = 0; jx < NR; ++jx) W[(tm * MR + i) * CB + tc * NR + jx] = acc[i][jx];
            __syncthreads();
#pragma unroll
            for (int i = 0; i < MR; ++i)
#pragma unroll
                for (int jx = 0; jx < NR; ++jx) acc[i][jx] = C(0);
            gemm_acc<C, TS, CB, MR, NR, KC>(ws.Um(l), W, Abuf, acc, tm, tc);
#pragma unroll
            for (int i = 0; i < MR; ++i)
#pragma unroll
                for (int jx = 0; jx < NR; ++jx) X[(tm * MR + i) * CB + tc * NR + jx] -= acc[i][jx];
            __syncthreads();
        }
        if (tid == 0) { st_lvl[sp] = 0; st_idx[sp] = l; }
        __syncthreads();
        ++sp;
        // reduce the stack
        while (true) {
            const int j = st_lvl[sp - 1];
            const int64_t i = st_idx[sp - 1];
            if (j >= L) break;                      // root reached
            if (i & 1) {                            // right child: combine with the entry below
                C *Xt = stack + (sp - 2) * TILE, *Xb = stack + (sp - 1) * TILE;
                const int64_t slot = tree_offset(m, j + 1) + (i >> 1);
                C acc[MR][NR];
                // W = X_top + Vb^T X_bot
#pragma unroll
                for (int ii = 0; ii < MR; ++ii)
#pragma unroll
                    for (int jx = 0; jx < NR; ++jx) acc[ii][jx] = Xt[(tm * MR + ii) * CB + tc * NR + jx];
                gemm_acc<C, TS, CB, MR, NR, KC>(ws.Vk(slot), Xb, Abuf, acc, tm, tc);
#pragma unroll
                for (int ii = 0; ii < MR; ++ii)
#pragma unroll
                    for (int jx = 0; jx < NR; ++jx) W[(tm * MR + ii) * CB + tc * NR + jx] = acc[ii][jx];
                __syncthreads();
                // X_top -= T^T W
#pragma unroll
                for (int ii = 0; ii < MR; ++ii)
#pragma unroll
                    for (int jx = 0; jx < NR; ++jx) acc[ii][jx] = C(0);
                gemm_acc<C, TS, CB, MR, NR, KC>(ws.Tt(slot), W, Abuf, acc, tm, tc);
#pragma unroll
                for (int ii = 0; ii < MR; ++ii)
#pragma unroll
                    for (int jx = 0; jx < NR; ++jx) Xt[(tm * MR + ii) * CB + tc * NR + jx] -= acc[ii][jx];
                // X_bot -= U W
#pragma unroll
                for (int ii = 0; ii < MR; ++ii)
#pragma unroll
                    for (int jx = 0; jx < NR; ++jx) acc[ii][jx] = C(0);
                gemm_acc<C, TS, CB, MR, NR, KC>(ws.Um(slot), W, Abuf, acc, tm, tc);
#pragma unroll
                for (int ii = 0; ii < MR; ++ii)
#pragma unroll
                    for (int jx = 0; jx < NR; ++jx) Xb[(tm * MR + ii) * CB + tc * NR + jx] -= acc[ii][jx];
                __syncthreads();
                // X_bot is final: its leaf is the leftmost leaf of node (j, i)
                store_tile<S, C, TS, CB>(V, (top + (i << j)) * TS, cbase + c0, cmax, Xb);
                __syncthreads();
                --sp;
                if (tid == 0) { st_lvl[sp - 1] = j + 1; st_idx[sp - 1] = i >> 1; }
                __syncthreads();
            } else if (i + 1 < tree_count(m, j)) {
                break;                              // wait for the right sibling
            } else {
                if (tid == 0) { st_lvl[sp - 1] = j + 1; st_idx[sp - 1] = i >> 1; }   // pass-through
                __syncthreads();
            }
        }
    }
    // root tile = leaf 0 (top tile row)
    store_tile<S, C, TS, CB>(V, top * TS, cbase + c0, cmax, stack);
}

// ---------------------------------------------------------------------------
// host side

template <typename C, int TS>
constexpr size_t panel_smem() {
    constexpr int LD = TS + 1;
    constexpr int PK = TS * (TS + 1) / 2;
    constexpr int BIG = (TS * LD > 3 * PK) ? TS * LD : 3 * PK;
    return (size_t)(BIG + 2 * TS + 8) * sizeof(C);
}
template <typename C, int TS>
size_t trail_smem(int depth) {
    constexpr int CB = TileCfg<C>::elems / TS;
    constexpr int KC = (TS >= 16) ? 16 : TS;
    return (size_t)(2 * KC * TS + (size_t)(depth + 1) * TS * CB) * sizeof(C);
}

template <typename S, typename C>
size_t tree_workspace_bytes(int64_t n, int ts) {
    const int64_t N = n / ts;
    return tree_ws_elems<C>(N, ts) * sizeof(C) + 256;
}

template <typename S, typename C, int TS>
static cudaError_t run_tree(S *a, int64_t n, int64_t batch, int64_t a_bstride, void *wsp,
                            cudaStream_t st, cudaEvent_t *ev_p, cudaEvent_t *ev_t, double *pms,
                            double *tms) {
    if constexpr (TS >= 16) {
        if (!getenv("BSVD_NO_OVERLAP"))
            return run_levels<S, C, TS>(a, n, batch, a_bstride, wsp, st, pms, tms, ev_p != nullptr);
    }
    const int64_t N = n / TS;
    const int64_t ws_elems = (int64_t)tree_ws_elems<C>(N, TS);
    const int64_t ts2 = (int64_t)TS * TS;
    TreeWs<C> ws;
    ws.nodes = (C *)wsp;
    ws.R = ws.nodes + tree_slots(N) * 3 * ts2;
    ws.cnt = (int *)(ws.R + N * ts2);
    ws.ts2 = ts2;
    cudaError_t err;
    for (int64_t b = 0; b < batch; ++b) {
        err = cudaMemsetAsync((char *)ws.cnt + b * ws_elems * (int64_t)sizeof(C), 0,
                              (size_t)(N + 64) * sizeof(int), st);
        if (err != cudaSuccess) return err;
    }
    const int depth = tree_levels(N) + 1;
    const size_t psm = TS >= 16 ? PanelBlk<C, TS>::smem : panel_smem<C, TS>();
    const size_t tsm = trail_smem<C, TS>(depth);
    if (tsm > 220 * 1024 || psm > 220 * 1024) return cudaErrorInvalidConfiguration;
    if constexpr (TS >= 16)
        err = ensure_smem(k_panel_blk<S, C, TS>, psm);
    else
        err = ensure_smem(k_panel_tree<S, C, TS>, psm);
    if (err != cudaSuccess) return err;
    if ((err = ensure_smem(k_trail_tree<S, C, TS>, tsm)) != cudaSuccess) return err;
    constexpr int CB = TileCfg<C>::elems / TS;
    // Per-phase timing: three events per sweep side, recorded on the launch
    // stream and read once at the end (no per-side host sync).
    const bool timed = ev_p != nullptr;
    (void)ev_t;
    std::vector<cudaEvent_t> evs;
    auto ev = [&]() -> cudaEvent_t {
        cudaEvent_t e;
        cudaEventCreate(&e);
        evs.push_back(e);
        cudaEventRecord(e, st);
        return e;
    };
    struct Mark { cudaEvent_t a, b, c; };
    std::vector<Mark> marks;
    const char *trace_path = getenv("BSVD_PANEL_TRACE");
    unsigned long long *trace_buf = nullptr;
    if (trace_path) {
        cudaMalloc(&trace_buf, (64 * 9 * 8 + 256) * 8);
        cudaMemset(trace_buf, 0, (64 * 9 * 8 + 256) * 8);
    }
    auto side = [&](int64_t k, bool lq) -> cudaError_t {
        View<S> V{a, lq ? n : 1, lq ? 1 : n};
        const int64_t top = lq ? k + 1 : k;
        if (top >= N) return cudaSuccess;
        const int64_t m = N - top;
        const int64_t ntrail = N - 1 - k;
        Mark mk{};
        if (timed) mk.a = ev();
        const bool tr_this = trace_path && k == 4 && !lq;
        if (tr_this) cudaMemcpyToSymbolAsync(g_panel_trace, &trace_buf, sizeof(void *), 0, cudaMemcpyHostToDevice, st);
        if constexpr (TS >= 16)
            k_panel_blk<S, C, TS><<<dim3((unsigned)m, (unsigned)batch), kNTP, psm, st>>>(
                V, m, top, k, ws, ws_elems, a_bstride);
        else
            k_panel_tree<S, C, TS><<<dim3((unsigned)m, (unsigned)batch), kNT, psm, st>>>(
                V, m, top, k, ws, ws_elems, a_bstride);
        bsvd_host::count_launch();
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        if (tr_this) {
            void *null_ptr = nullptr;
            cudaMemcpyToSymbolAsync(g_panel_trace, &null_ptr, sizeof(void *), 0, cudaMemcpyHostToDevice, st);
            std::vector<unsigned long long> h(64 * 9 * 8 + 256);
            cudaMemcpyAsync(h.data(), trace_buf, h.size() * 8, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            FILE *f = fopen(trace_path, "wb");
            if (f) { fwrite(h.data(), 8, h.size(), f); fclose(f); }
        }
        if (timed) mk.b = ev();
        if (ntrail > 0) {
            if constexpr (TS >= 16) {
                // one launch per tree level, thousands of CTAs (stage1_apply.cu)
                e = launch_apply_levels<S, C, TS>(a, n, batch, a_bstride, lq, top, k, m, ws.nodes,
                                                  ws_elems, st);
            } else {
                const int64_t ncols = ntrail * TS;
                k_trail_tree<S, C, TS><<<dim3((unsigned)((ncols + CB - 1) / CB), (unsigned)batch), kNT, tsm, st>>>(
                    V, m, top, k, ncols, ws, ws_elems, a_bstride);
                bsvd_host::count_launch();
                e = cudaGetLastError();
            }
            if (e != cudaSuccess) return e;
        }
        if (timed) {
            mk.c = ev();
            marks.push_back(mk);
        }
        return cudaSuccess;
    };
    for (int64_t k = 0; k < N - 1 && err == cudaSuccess; ++k) {
        if ((err = side(k, false)) != cudaSuccess) break;
        err = side(k, true);
    }
    if (err == cudaSuccess) err = side(N - 1, false);
    if (timed && !evs.empty()) {
        cudaEventSynchronize(evs.back());
        for (const Mark &mk : marks) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, mk.a, mk.b);
            *pms += ms;
            cudaEventElapsedTime(&ms, mk.b, mk.c);
            *tms += ms;
        }
        for (cudaEvent_t e : evs) cudaEventDestroy(e);
    }
    return err;
}

template <typename S, typename C>
cudaError_t banddiag_tree(S *a, int64_t n, int ts, int64_t batch, int64_t a_bstride, void *ws,
                          cudaStream_t st, cudaEvent_t *ev_panel, cudaEvent_t *ev_trail,
                          double *panel_ms, double *trail_ms) {
    switch (ts) {
    case 4: return run_tree<S, C, 4>(a, n, batch, a_bstride, ws, st, ev_panel, ev_trail, panel_ms, trail_ms);
    case 8: return run_tree<S, C, 8>(a, n, batch, a_bstride, ws, st, ev_panel, ev_trail, panel_ms, trail_ms);
    case 16: return run_tree<S, C, 16>(a, n, batch, a_bstride, ws, st, ev_panel, ev_trail, panel_ms, trail_ms);
    case 32: return run_tree<S, C, 32>(a, n, batch, a_bstride, ws, st, ev_panel, ev_trail, panel_ms, trail_ms);
    case 64: return run_tree<S, C, 64>(a, n, batch, a_bstride, ws, st, ev_panel, ev_trail, panel_ms, trail_ms);
    case 128: return run_tree<S, C, 128>(a, n, batch, a_bstride, ws, st, ev_panel, ev_trail, panel_ms, trail_ms);
    default: return cudaErrorInvalidValue;
    }
}

#define INST(S, C)                                                                               \
    template size_t tree_workspace_bytes<S, C>(int64_t, int);                                     \
    template cudaError_t banddiag_tree<S, C>(S *, int64_t, int, int64_t, int64_t, void *,          \
                                             cudaStream_t, cudaEvent_t *, cudaEvent_t *, double *, \
                                             double *);
INST(double, double)
INST(float, float)
INST(__half, float)
#undef INST

}  // namespace bsvd
