// panel_qr.cuh -- on-chip Householder kernels of the stage-1 panel
// (included by stage1_tree.cu; kNT threads per CTA).
//
//  leaf_qr_la : QR of a ts x ts tile, column-major in smem (ld = ts+1).
//  tt_qr_la   : QR of [R_top; R_bot] (both upper triangular, packed).
//  build_T_rec: compact-WY T from G = V^T V by recursive merging,
//               T12 = -T11 * G12 * T22  (log2(ts) levels of parallel products
//               instead of ts dependent column steps).
//
// "la" = look-ahead: the thread group that applies reflector k to column k+1
// immediately forms reflector k+1 from it, so each column step needs ONE CTA
// barrier and no serial single-warp phase.
#pragma once

namespace bsvd {
namespace panel {

template <typename C, int TPC>
__device__ __forceinline__ C group_sum_m(C v, unsigned mask) {   // TPC consecutive lanes
#pragma unroll
    for (int o = TPC / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o);
    return v;
}

template <int NT, int TS>
struct Cols {
    static constexpr int TPC = (NT / TS) < 32 ? (NT / TS) : 32;   // threads per column
    static constexpr int NG = NT / TPC;                             // column groups
};

// ---------------------------------------------------------------------------
template <typename C, int TS, int NT, typename HS>
__device__ void leaf_qr_la(C *A, C *tau, HS house) {
    constexpr int LD = TS + 1;
    using G = Cols<NT, TS>;
    constexpr int TPC = G::TPC, NG = G::NG;
    const int tid = threadIdx.x, g = tid / TPC, q = tid % TPC;
    const int lane = tid & 31;
    const unsigned gmask = TPC == 32 ? 0xffffffffu : (((1u << TPC) - 1u) << (lane & ~(TPC - 1)));
    // reflector of column kk from its rows kk.. (group-local)
    auto pivot = [&](int kk) {
        C s0 = C(0), s1 = C(0);
        int r = kk + 1 + q;
        for (; r + TPC < TS; r += 2 * TPC) {
            const C x0 = A[kk * LD + r], x1 = A[kk * LD + r + TPC];
            s0 += x0 * x0;
            s1 += x1 * x1;
        }
        if (r < TS) s0 += A[kk * LD + r] * A[kk * LD + r];
        const C sig = group_sum_m<C, TPC>(s0 + s1, gmask);
        const C alpha = A[kk * LD + kk];
        C beta, t, scale;
        house(alpha, sig, beta, t, scale);
        for (int rr = kk + 1 + q; rr < TS; rr += TPC) A[kk * LD + rr] *= scale;
        if (q == 0) {
            A[kk * LD + kk] = beta;
            tau[kk] = t;
        }
    };
    if (g == 0) pivot(0);
    __syncthreads();
    for (int kk = 0; kk < TS - 1; ++kk) {
        const C t = tau[kk];
        const C *v = A + kk * LD;
        for (int cb = kk + 1; cb < TS; cb += NG) {          // warp-uniform trip count
            const int c = cb + g;
            const bool act = c < TS;
            C w0 = C(0), w1 = C(0);
            if (act) {
                const C *x = A + c * LD;
                int r = kk + 1 + q;
                for (; r + TPC < TS; r += 2 * TPC) {
                    w0 += v[r] * x[r];
                    w1 += v[r + TPC] * x[r + TPC];
                }
                if (r < TS) w0 += v[r] * x[r];
            }
            C w = w0 + w1;
#pragma unroll
            for (int o = TPC / 2; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            if (act) {
                C *x = A + c * LD;
                w = (w + x[kk]) * t;
                for (int r = kk + 1 + q; r < TS; r += TPC) x[r] -= w * v[r];
                if (q == 0) x[kk] -= w;
            }
            if (cb == kk + 1 && g == 0 && kk + 1 < TS - 1) {  // group 0 owns column kk+1
                __syncwarp(gmask);
                pivot(kk + 1);
            }
        }
        __syncthreads();
    }
    if (tid == 0) tau[TS - 1] = C(0);   // A8: the last tile column has no reflector
    __syncthreads();
}

// Packed upper-triangular column-major index (r <= c).
__host__ __device__ __forceinline__ int pkx(int r, int c) { return c * (c + 1) / 2 + r; }

template <typename C, int TS, int NT, typename HS>
__device__ void tt_qr_la(C *Rt, C *Rb, C *tau, HS house) {
    using G = Cols<NT, TS>;
    constexpr int TPC = G::TPC, NG = G::NG;
    const int tid = threadIdx.x, g = tid / TPC, q = tid % TPC;
    const int lane = tid & 31;
    const unsigned gmask = TPC == 32 ? 0xffffffffu : (((1u << TPC) - 1u) << (lane & ~(TPC - 1)));
    auto pivot = [&](int kk) {
        C s = C(0);
        for (int r = q; r <= kk; r += TPC) s += Rb[pkx(r, kk)] * Rb[pkx(r, kk)];
        const C sig = group_sum_m<C, TPC>(s, gmask);
        const C alpha = Rt[pkx(kk, kk)];
        C beta, t, scale;
        house(alpha, sig, beta, t, scale);
        for (int r = q; r <= kk; r += TPC) Rb[pkx(r, kk)] *= scale;
        if (q == 0) {
            Rt[pkx(kk, kk)] = beta;
            tau[kk] = t;
        }
    };
    if (g == 0) pivot(0);
    __syncthreads();
    for (int kk = 0; kk < TS; ++kk) {
        const C t = tau[kk];
        const C *v = Rb + pkx(0, kk);
        for (int cb = kk + 1; cb < TS; cb += NG) {
            const int c = cb + g;
            const bool act = c < TS;
            C w0 = C(0), w1 = C(0);
            if (act) {
                const C *x = Rb + pkx(0, c);
                int r = q;
                for (; r + TPC <= kk; r += 2 * TPC) {
                    w0 += v[r] * x[r];
                    w1 += v[r + TPC] * x[r + TPC];
                }
                if (r <= kk) w0 += v[r] * x[r];
            }
            C w = w0 + w1;
#pragma unroll
            for (int o = TPC / 2; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            if (act) {
                C *x = Rb + pkx(0, c);
                w = (w + Rt[pkx(kk, c)]) * t;
                for (int r = q; r <= kk; r += TPC) x[r] -= w * v[r];
                if (q == 0) Rt[pkx(kk, c)] -= w;
            }
            if (cb == kk + 1 && g == 0) {
                __syncwarp(gmask);
                pivot(kk + 1);
            }
        }
        __syncthreads();
    }
}

// T from G by recursive merging.  Tr(i, j) returns a reference to T(i, j)
// (i <= j), whose strict upper part holds G(i, j) on entry; tmp holds
// >= TS*TS/4 elements.  Valid for any tau (a zero tau gives a zero row and
// column, like LAPACK larft).
template <typename C, int TS, int NT, typename TR>
__device__ void build_T_rec(const C *tau, C *tmp, TR Tr) {
    const int tid = threadIdx.x;
    for (int i = tid; i < TS; i += NT) Tr(i, i) = tau[i];
    __syncthreads();
#pragma unroll 1
    for (int s = 1; s < TS; s *= 2) {
        const int nb = TS / (2 * s), ss = s * s;
        for (int idx = tid; idx < nb * ss; idx += NT) {          // X = G12 * T22
            const int qb = idx / ss, rem = idx - qb * ss, i = rem / s, j = rem - i * s;
            const int a = 2 * s * qb, b = a + s;
            C acc0 = C(0), acc1 = C(0);
            int p = 0;
            for (; p + 1 <= j; p += 2) {
                acc0 += Tr(a + i, b + p) * Tr(b + p, b + j);
                acc1 += Tr(a + i, b + p + 1) * Tr(b + p + 1, b + j);
            }
            if (p <= j) acc0 += Tr(a + i, b + p) * Tr(b + p, b + j);
            tmp[idx] = acc0 + acc1;
        }
        __syncthreads();
        for (int idx = tid; idx < nb * ss; idx += NT) {          // T12 = -T11 * X
            const int qb = idx / ss, rem = idx - qb * ss, i = rem / s, j = rem - i * s;
            const int a = 2 * s * qb, b = a + s;
            const C *X = tmp + qb * ss;
            C acc0 = C(0), acc1 = C(0);
            int p = i;
            for (; p + 1 < s; p += 2) {
                acc0 += Tr(a + i, a + p) * X[p * s + j];
                acc1 += Tr(a + i, a + p + 1) * X[(p + 1) * s + j];
            }
            if (p < s) acc0 += Tr(a + i, a + p) * X[p * s + j];
            Tr(a + i, b + j) = -(acc0 + acc1);
        }
        __syncthreads();
    }
}

}  // namespace panel
}  // namespace bsvd
