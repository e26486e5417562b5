// panel_blocked.cuh -- blocked on-chip Householder QR for the stage-1 panel
// nodes (included by stage1_tree.cu).  One CTA of NT threads factors either
//   LEAF: a ts x ts tile A (column-major in smem, ld = lda), or
//   TT  : the stack [R_top; R_bot] of two upper triangles, held unpacked as a
//         2ts x ts column-major operand (rows [0,ts) = R_top, [ts,2ts) = R_bot).
// Reflector k acts on rows  LEAF: [k, ts)   TT: {k} u [ts, ts + k]   with the
// unit entry at row k.  On exit R sits in the upper triangle of rows [0, ts),
// the reflector tails are stored in place (LEAF: strictly lower part; TT: the
// R_bot upper triangle) and T (ts x ts, upper, compact WY: Q = I - V T V^T)
// is written to Tm (column-major, ld = ldt).
//
// Algorithm (per NB = 32-column sub-panel):
//  1. factor the sub-panel in REGISTERS: warp w owns a slab of rows, lane c
//     owns column c; per column one partial-sum exchange through smem for the
//     norm and one for the 32 dot products (two CTA barriers per column, no
//     full-tile shared-memory pass);
//  2. T_sub by recursive merging (T12 = -T11 G12 T22);
//  3. apply the sub-panel's block reflector to the columns to its right:
//     W = V^T A, W = T_sub^T W, A -= V W (register-tiled smem GEMMs);
//  4. extend T block-column-wise: T[0:j0, j0:j0+NB] = -T[0:j0,0:j0] (V_0^T V_p) T_sub.
#pragma once

namespace bsvd {
namespace blk {

// Generic register-tiled product on shared-memory operands:
//   for every (m, n) in [0,M) x [0,N):  out(m, n, sum_{k in [klo(m,n), K)} a(m, k) * b(k, n))
// Each thread owns RM x RN outputs (tiles strided over the CTA).
template <typename C, int RM, int RN, int NT, typename AF, typename BF, typename OF>
__device__ __forceinline__ void sgemm(int M, int N, int K, AF a, BF b, OF out) {
    const int tmc = (M + RM - 1) / RM, tnc = (N + RN - 1) / RN;
    for (int t = threadIdx.x; t < tmc * tnc; t += NT) {
        const int m0 = (t % tmc) * RM, n0 = (t / tmc) * RN;
        C acc[RM][RN];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
            for (int j = 0; j < RN; ++j) acc[i][j] = C(0);
        for (int k = 0; k < K; ++k) {
            C av[RM], bv[RN];
#pragma unroll
            for (int i = 0; i < RM; ++i) av[i] = (m0 + i < M) ? a(m0 + i, k) : C(0);
#pragma unroll
            for (int j = 0; j < RN; ++j) bv[j] = (n0 + j < N) ? b(k, n0 + j) : C(0);
#pragma unroll
            for (int i = 0; i < RM; ++i)
#pragma unroll
                for (int j = 0; j < RN; ++j) acc[i][j] += av[i] * bv[j];
        }
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
            for (int j = 0; j < RN; ++j)
                if (m0 + i < M && n0 + j < N) out(m0 + i, n0 + j, acc[i][j]);
    }
}

template <int TS, bool TT>
struct Geom {
    static constexpr int NB = TS < 32 ? TS : 32;                  // sub-panel width
    static constexpr int ROWS = TT ? 2 * TS : TS;                 // operand rows
    // rows of sub-panel j0 (as a list): LEAF [j0, TS); TT [j0, j0+NB) u [TS, TS+j0+NB)
    __device__ static int nrows(int j0) { return TT ? (NB + j0 + NB) : (TS - j0); }
    __device__ static int row(int j0, int i) { return TT ? (i < NB ? j0 + i : TS + (i - NB)) : (j0 + i); }
    // row-list index i lies on reflector (local) kl of sub-panel j0 (excluding the unit row)?
    __device__ static bool on_ref(int j0, int kl, int i) {
        if (TT) return i >= NB && (i - NB) <= j0 + kl;
        return i > kl;
    }
    __device__ static bool unit(int kl, int i) { return i == kl; }
    static constexpr int RMAX = ((TT ? (2 * (TS < 32 ? TS : 32) + TS - (TS < 32 ? TS : 32)) : TS) + 7) / 8;
};

// V(i, a) of sub-panel j0 (row-list index i, local column a), from smem A.
template <typename C, int TS, bool TT>
__device__ __forceinline__ C vval(const C *A, int lda, int j0, int i, int a) {
    using G = Geom<TS, TT>;
    if (G::unit(a, i)) return C(1);
    if (!G::on_ref(j0, a, i)) return C(0);
    return A[(j0 + a) * lda + G::row(j0, i)];
}

// Step 1: register-resident factorisation of sub-panel j0 (NB columns).
template <typename C, int TS, bool TT, int NT, typename HS>
__device__ void subpanel(C *A, int lda, int j0, C *tau, C *red, HS house,
                         unsigned long long *st = nullptr) {
    using G = Geom<TS, TT>;
    constexpr int NB = G::NB, RMAX = G::RMAX, NW = NT / 32;
    const int R = G::nrows(j0);
    const int rpw = (R + NW - 1) / NW;                   // rows per warp
    const int warp = threadIdx.x >> 5, c = threadIdx.x & 31;
    const int i0 = warp * rpw;
    C x[RMAX];
#pragma unroll
    for (int q = 0; q < RMAX; ++q) {
        const int i = i0 + q;
        x[q] = (q < rpw && i < R && c < NB) ? A[(j0 + c) * lda + G::row(j0, i)] : C(0);
    }
    C *sig_part = red;             // [NW]
    C *alpha_s = red + NW;         // [1]
    C *dpart = red + NW + 2;       // [NW][32]
    for (int kl = 0; kl < NB; ++kl) {
        // (1) lane kl: partial ||tail||^2 of its column; the pivot row's owner posts alpha
        if (c == kl) {
            C s = C(0);
#pragma unroll
            for (int q = 0; q < RMAX; ++q) {
                const int i = i0 + q;
                if (q < rpw && i < R && G::on_ref(j0, kl, i)) s += x[q] * x[q];
                if (q < rpw && i < R && i == kl) *alpha_s = x[q];
            }
            sig_part[warp] = s;
        }
        __syncthreads();
        // (2) every thread forms the same reflector
        C sig = C(0);
#pragma unroll
        for (int w = 0; w < NW; ++w) sig += sig_part[w];
        const C alpha = *alpha_s;
        C beta, t, scale;
        house(alpha, sig, beta, t, scale);
        // (3) v for this warp's rows (from lane kl by shuffle); partial dots
        C v[RMAX];
        C d = C(0);
#pragma unroll
        for (int q = 0; q < RMAX; ++q) {
            const int i = i0 + q;
            const C xk = __shfl_sync(0xffffffffu, x[q], kl);
            const bool in = q < rpw && i < R;
            v[q] = (in && i == kl) ? C(1) : ((in && G::on_ref(j0, kl, i)) ? xk * scale : C(0));
            d += v[q] * x[q];
        }
        dpart[warp * 32 + c] = d;
        __syncthreads();
        if (c > kl && c < NB) {
            C dd = C(0);
#pragma unroll
            for (int w = 0; w < NW; ++w) dd += dpart[w * 32 + c];
            const C wc = t * dd;
#pragma unroll
            for (int q = 0; q < RMAX; ++q) x[q] -= wc * v[q];
        } else if (c == kl) {
#pragma unroll
            for (int q = 0; q < RMAX; ++q) {
                const int i = i0 + q;
                if (q < rpw && i < R) {
                    if (i == kl) x[q] = beta;
                    else if (G::on_ref(j0, kl, i)) x[q] = v[q];
                }
            }
        }
        if (threadIdx.x == 0) tau[j0 + kl] = t;
        if (st && threadIdx.x == 0) {
            unsigned long long tt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
            st[j0 + kl] = tt;
        }
    }
#pragma unroll
    for (int q = 0; q < RMAX; ++q) {
        const int i = i0 + q;
        if (q < rpw && i < R && c < NB) A[(j0 + c) * lda + G::row(j0, i)] = x[q];
    }
    __syncthreads();
}

// Full blocked QR + T.  Tm: ts x ts column-major T output (ld ldt; may alias
// nothing in A's active region).  wbuf: >= NB*TS scratch, tsub: >= NB*(NB+1),
// gbuf: >= TS*NB, red: >= NT/32*34 + 4.
template <typename C, int TS, bool TT, int NT, typename HS, typename SaveR>
__device__ void qr_blocked(C *A, int lda, C *tau, C *Tm, int ldt, C *wbuf, C *tsub, C *gbuf,
                           C *red, HS house, SaveR save_r, unsigned long long *st = nullptr) {
    using G = Geom<TS, TT>;
    constexpr int NB = G::NB;
    constexpr int LDS = NB + 1;
    for (int j0 = 0; j0 < TS; j0 += NB) {
        subpanel<C, TS, TT, NT>(A, lda, j0, tau, red, house, st);
        auto stamp = [&](int id) {
            if (st && threadIdx.x == 0) {
                unsigned long long tt;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
                st[128 + id] = tt;
            }
        };
        stamp(4 * (j0 / NB) + 0);
        save_r(j0);   // R columns [j0, j0+NB) are final; T may now overwrite them
        const int R = G::nrows(j0);
        // ---- T_sub: G_sub(a,b) = V(:,a)^T V(:,b) (a<b) then recursive merge
        sgemm<C, 2, 2, NT>(NB, NB, R,
            [&](int a, int i) { return vval<C, TS, TT>(A, lda, j0, i, a); },
            [&](int i, int b) { return vval<C, TS, TT>(A, lda, j0, i, b); },
            [&](int a, int b, C v) { if (a < b) tsub[b * LDS + a] = v; });
        __syncthreads();
        panel::build_T_rec<C, NB, NT>(tau + j0, gbuf, [&](int i, int j) -> C & { return tsub[j * LDS + i]; });
        // ---- extend the full T: T[0:j0, j0:j0+NB] = -T[0:j0,0:j0] * (V_prev^T V_p) * T_sub
        if (j0 > 0) {
            // gbuf[p][a] = sum_rows Vprev(row, p) * Vp(row, a)  (p < j0, a < NB) over global rows
            sgemm<C, 2, 2, NT>(j0, NB, G::ROWS,
                [&](int p, int r) {      // V_prev(r, p): column p's reflector at global row r
                    if (TT) {
                        if (r < TS) return r == p ? C(1) : C(0);
                        return (r - TS) <= p ? A[p * lda + r] : C(0);
                    }
                    return r == p ? C(1) : (r > p ? A[p * lda + r] : C(0));
                },
                [&](int r, int a) {
                    const int ca = j0 + a;
                    if (TT) {
                        if (r < TS) return r == ca ? C(1) : C(0);
                        return (r - TS) <= ca ? A[ca * lda + r] : C(0);
                    }
                    return r == ca ? C(1) : (r > ca ? A[ca * lda + r] : C(0));
                },
                [&](int p, int a, C v) { gbuf[a * TS + p] = v; });
            __syncthreads();
            // wbuf = gbuf * T_sub (j0 x NB), T_sub upper
            sgemm<C, 2, 2, NT>(j0, NB, NB,
                [&](int p, int q) { return gbuf[q * TS + p]; },
                [&](int q, int a) { return q <= a ? tsub[a * LDS + q] : C(0); },
                [&](int p, int a, C v) { wbuf[a * TS + p] = v; });
            __syncthreads();
            // T[0:j0, j0+a] = -T[0:j0,0:j0] * wbuf
            sgemm<C, 2, 2, NT>(j0, NB, j0,
                [&](int p, int q) { return q >= p ? Tm[q * ldt + p] : C(0); },
                [&](int q, int a) { return wbuf[a * TS + q]; },
                [&](int p, int a, C v) { Tm[(j0 + a) * ldt + p] = -v; });
        }
        // T diagonal block (upper triangle only: the strict lower part of a leaf
        // tile holds the reflector tails)
        for (int idx = threadIdx.x; idx < NB * NB; idx += NT) {
            const int a = idx % NB, b = idx / NB;
            if (a <= b) Tm[(j0 + b) * ldt + (j0 + a)] = tsub[b * LDS + a];
        }
        __syncthreads();
        stamp(4 * (j0 / NB) + 1);
        // ---- apply the sub-panel block reflector to columns [j0+NB, TS)
        const int ncol = TS - j0 - NB;
        if (ncol > 0) {
            // W = V^T A_rest   (NB x ncol, K = R)
            sgemm<C, 2, 4, NT>(NB, ncol, R,
                [&](int a, int i) { return vval<C, TS, TT>(A, lda, j0, i, a); },
                [&](int i, int cc) { return A[(j0 + NB + cc) * lda + G::row(j0, i)]; },
                [&](int a, int cc, C v) { wbuf[cc * NB + a] = v; });
            __syncthreads();
            // W2 = T_sub^T W  -> gbuf
            sgemm<C, 2, 4, NT>(NB, ncol, NB,
                [&](int a, int b) { return b <= a ? tsub[a * LDS + b] : C(0); },   // T^T(a,b) = T(b,a)
                [&](int b, int cc) { return wbuf[cc * NB + b]; },
                [&](int a, int cc, C v) { gbuf[cc * NB + a] = v; });
            __syncthreads();
            // A_rest -= V W2   (R x ncol, K = NB)
            sgemm<C, 4, 4, NT>(R, ncol, NB,
                [&](int i, int a) { return vval<C, TS, TT>(A, lda, j0, i, a); },
                [&](int a, int cc) { return gbuf[cc * NB + a]; },
                [&](int i, int cc, C v) { A[(j0 + NB + cc) * lda + G::row(j0, i)] -= v; });
            __syncthreads();
        }
        stamp(4 * (j0 / NB) + 2);
    }
}

}  // namespace blk
}  // namespace bsvd
