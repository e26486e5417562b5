// panel_blocked.cuh -- blocked on-chip Householder QR for the stage-1 panel
// nodes (included by stage1_tree.cu).  One CTA of NT threads factors either
//   LEAF: a ts x ts tile A (column-major in smem, ld = lda), or
//   TT  : the stack [R_top; R_bot] of two upper triangles, held unpacked as a
//         2ts x ts column-major operand (rows [0,ts) = R_top, [ts,2ts) = R_bot;
//         R_bot's strict lower part is explicit zeros).
// Reflector k acts on rows  LEAF: [k, ts)   TT: {k} u [ts, ts + k]   with the
// unit entry at row k.  On exit R sits in the upper triangle of rows [0, ts),
// the reflector tails are stored in place (LEAF: strictly lower part; TT: the
// R_bot upper triangle) and T (ts x ts, upper, compact WY: Q = I - V T V^T)
// is written to Tm (column-major, ld = ldt), overwriting R's upper triangle
// block column by block column after save_r(j0) has copied it out.
//
// Per NB-column sub-panel j0 (NB = 32, or 16 for fp64 ts = 128):
//  1. factor the sub-panel in REGISTERS with the rows-per-warp count a
//     compile-time constant (fully unrolled, mask-free loops): warp w owns a
//     slab of the sub-panel's rows, lane c owns column c; per column one
//     partial-sum exchange for the norm and one for the NB dot products;
//  2. an explicit dense copy Vs of the sub-panel reflectors makes every
//     following product branch-free: T_sub = merge(Vs^T Vs), the block-column
//     extension of T (earlier reflectors are read straight from the operand:
//     their zero structure is stored explicitly), and the update of the columns
//     to the right  W = Vs^T A,  W = T_sub^T W,  A -= Vs W.
#pragma once

namespace bsvd {
namespace blk {

// phase stamps (development tracing): globaltimer, or SM clock for microbenchmarks
__device__ __forceinline__ unsigned long long stamp_now() {
#ifdef BSVD_STAMP_CLOCK
    return (unsigned long long)clock64();
#else
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
#endif
}

// Register-tiled product on shared-memory operands:
//   out(m, n, sum_k a(m, k) * b(k, n))  for (m, n) in [0,M) x [0,N).
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
#pragma unroll 2
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

template <typename C, int TS>
struct NBsel {   // sub-panel width: 16 keeps fp64 ts=128 leaves inside shared memory
    static constexpr int v = TS < 32 ? TS : ((sizeof(C) == 8 && TS >= 128) ? 16 : 32);
};

// scratch elements needed by qr_blocked (Vs | wbuf | gbuf | tsub | red)
// ROWS: rows of a LEAF operand (TS for a tile, 2 TS for a two-tile leaf)
template <typename C, int TS, int ROWS = TS>
__host__ __device__ constexpr int aux_elems() {
    constexpr int NB = NBsel<C, TS>::v;
    return (ROWS + NB) * (NB + 1) + 2 * NB * TS + NB * (NB + 1) + 16 * 34 + 8 + (ROWS + 2 * NB);
}

#ifndef BSVD_NWF_LEAF2
#define BSVD_NWF_LEAF2 8
#endif
// factor warps per sub-panel: measured, 8 beat 4 (latency) and 16 (issue) on
// ts-row operands
template <bool TT, int TS, int ROWS>
__host__ __device__ constexpr int nwf() { return (!TT && ROWS == 2 * TS) ? BSVD_NWF_LEAF2 : 8; }

// Step 1: register-resident factorisation of sub-panel J0 by the first NWF
// warps (named barrier 1); the remaining warps only join the final barrier.
// Fewer, fatter warps: the per-step overheads that every warp pays (partial-
// sum reductions, reflector scalars) shrink with the warp count, and only
// the pivot lane forms v (broadcast by shuffle) -- the step is issue-bound.
template <typename C, int TS, bool TT, int NB, int J0, int NT, int ROWS, typename HS>
__device__ __forceinline__ void subpanel(C *A, int lda, C *tau, C *red, C *Vs, C *gsub, HS house,
                                         unsigned long long *st) {
    constexpr int R = TT ? (2 * NB + J0) : (ROWS - J0);  // rows in the sub-panel's row list
    constexpr int NWF = nwf<TT, TS, ROWS>();
    constexpr bool TW = NT / 32 > NWF;    // a spare warp builds T_sub alongside
    constexpr int RPW = R / NWF;
    static_assert(R % NWF == 0, "row list must split evenly over the factor warps");
    static_assert(NT / 32 >= NWF, "not enough warps");
    const int warp = threadIdx.x >> 5, c = threadIdx.x & 31;
    // T_sub is built in CHUNKS of columns by warp NWF while the factorisation
    // runs: warp 0 signals chunk q on named barrier 2 + q (warp 0 + warp NWF)
    constexpr int CHUNK = NB >= 8 ? NB / 4 : NB;
    if (warp < NWF) {
        auto fbar = []() { asm volatile("bar.sync 1, %0;" ::"n"(NWF * 32) : "memory"); };
        const int i0 = warp * RPW;
        auto row = [](int i) { return TT ? (i < NB ? J0 + i : TS + (i - NB)) : (J0 + i); };
        C x[RPW];
#pragma unroll
        for (int q = 0; q < RPW; ++q) x[q] = (c < NB) ? A[(J0 + c) * lda + row(i0 + q)] : C(0);
        // red: sig_part[NWF] | alpha | pad | dpart[NWF*32] | vbuf[R] (this warp's slab:
        // the pivot column at the start of a step, then v)
        C *sig_part = red, *alpha_s = red + NWF, *dpart = red + NWF + 2;
        C *vbuf = dpart + NWF * 32 + i0;
        static_assert(RPW <= 32, "one lane per row of the warp's slab");
        // The pivot lane of step kl (lane kl) publishes its column (vbuf), its
        // slab's partial norm (sig_part) and alpha right after its own update in
        // step kl-1, so a step needs two barriers and no separate norm phase.
        auto publish = [&](int kp) {                    // executed by lane kp
            C s0 = C(0), s1 = C(0);
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int i = i0 + q;
                const bool on = TT ? (i >= NB && i - NB <= J0 + kp) : (i > kp);
                const C xv = on ? x[q] : C(0);
                if (q & 1) s1 += xv * xv; else s0 += xv * xv;
                if (i == kp) *alpha_s = x[q];
                vbuf[q] = x[q];
            }
            sig_part[warp] = s0 + s1;
        };
        if (c == 0) publish(0);
        for (int kl = 0; kl < NB; ++kl) {
            // row-list index i is on reflector kl (excluding its unit row kl)?
            auto on_ref = [&](int i) { return TT ? (i >= NB && i - NB <= J0 + kl) : (i > kl); };
            fbar();
            C sig = C(0);
#pragma unroll
            for (int w = 0; w < NWF; ++w) sig += sig_part[w];
            C beta, t, scale;
            house(*alpha_s, sig, beta, t, scale);
            // v for this warp's rows, lane-parallel (lane q < RPW owns row i0 + q)
            const int ic = i0 + c;
            if (c < RPW) {
                const C xv = vbuf[c];
                C vq = on_ref(ic) ? xv * scale : C(0);
                vq = (ic == kl) ? C(1) : vq;
                vbuf[c] = vq;
                Vs[ic * (NB + 1) + kl] = vq;
            }
            if (warp == 0 && c == 0) tau[J0 + kl] = t;
            __syncwarp();
            C v[RPW];
            C d0 = C(0), d1 = C(0);
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int i = i0 + q;
                v[q] = vbuf[q];
                if (c == kl) x[q] = (i == kl) ? beta : (on_ref(i) ? v[q] : x[q]);
                if (q & 1) d1 += v[q] * x[q]; else d0 += v[q] * x[q];
            }
            dpart[warp * 32 + c] = d0 + d1;
            fbar();
            // one reduction for every lane (no divergent second pass): lanes
            // c > kl get their column's dot, and lanes c < kl hold v_c (zero off
            // its support) exactly where v_kl lives, so theirs is the Gram entry
            // G(c, kl) = v_c^T v_kl -- T_sub's Gram matrix for free
            C dd = C(0);
#pragma unroll
            for (int w = 0; w < NWF; ++w) dd += dpart[w * 32 + c];
            if (warp == 0) {
                if (c < kl) gsub[kl * (NB + 1) + c] = dd;
                if (TW && (kl + 1) % CHUNK == 0)         // G columns of a chunk are out
                    asm volatile("bar.arrive %0, 64;" ::"r"(2 + kl / CHUNK) : "memory");
            }
            if (c > kl && c < NB) {
                const C wc = t * dd;
#pragma unroll
                for (int q = 0; q < RPW; ++q) x[q] -= wc * v[q];
                if (c == kl + 1) publish(kl + 1);       // the next step's pivot column
            }
            if (st && threadIdx.x == 0) st[J0 + kl] = stamp_now();
        }
#pragma unroll
        for (int q = 0; q < RPW; ++q)
            if (c < NB) A[(J0 + c) * lda + row(i0 + q)] = x[q];
    } else if (TW && warp == NWF) {
        // T_sub column by column while the factorisation runs (LAPACK dlarft's
        // forward recurrence T(0:kl, kl) = -tau_kl T(0:kl, 0:kl) G(0:kl, kl)),
        // lane c holding row c of T; it sleeps on its chunk barrier, so only
        // the last chunk's columns remain once the factorisation ends.
        C trow[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j) trow[j] = C(0);
#pragma unroll 1
        for (int q = 0; q < NB / CHUNK; ++q) {
            asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");   // wait for chunk q
            for (int kl = q * CHUNK; kl < (q + 1) * CHUNK; ++kl) {
                const C t = tau[J0 + kl];
                C acc = C(0);
#pragma unroll
                for (int j = 0; j < NB; ++j)
                    if (j < kl) acc += trow[j] * gsub[kl * (NB + 1) + j];
                const C tv = c < kl ? -t * acc : (c == kl ? t : C(0));
#pragma unroll
                for (int j = 0; j < NB; ++j)
                    if (j == kl) trow[j] = tv;
            }
        }
        if (c < NB) {
#pragma unroll
            for (int j = 0; j < NB; ++j)
                if (c <= j) gsub[j * (NB + 1) + c] = trow[j];
        }
    }
    __syncthreads();
}

template <typename C, int TS, bool TT, int NB, int J0, int NT, bool FULL_T, int ROWS, typename HS, typename SaveR>
__device__ __forceinline__ void qr_step(C *A, int lda, C *tau, C *Tm, int ldt, C *aux, HS house,
                                        SaveR save_r, unsigned long long *st) {
    if constexpr (J0 < TS) {
        constexpr int R = TT ? (2 * NB + J0) : (ROWS - J0);
        constexpr int LDS = NB + 1;
        constexpr int VLD = NB + 1;   // padded: the update reads Vs down its columns
        C *Vs = aux, *wbuf = Vs + (ROWS + NB) * VLD, *gbuf = wbuf + NB * TS;
        C *tsub = gbuf + NB * TS, *red = tsub + NB * LDS;
        auto row = [](int i) { return TT ? (i < NB ? J0 + i : TS + (i - NB)) : (J0 + i); };
        auto stamp = [&](int id) {
            if (st && threadIdx.x == 0) st[128 + id] = stamp_now();
        };
        subpanel<C, TS, TT, NB, J0, NT, ROWS>(A, lda, tau, red, Vs, tsub, house, st);   // + G into tsub
        stamp(4 * (J0 / NB) + 0);
        // FULL_T: T's blocks overwrite R's rows in place, so R leaves first;
        // otherwise nothing overwrites R and qr_blocked saves it once at the end
        if constexpr (FULL_T) save_r(J0);
        stamp(4 * (J0 / NB) + 3);
        // (T_sub is in tsub: built alongside the factorisation from its Gram
        // matrix -- or here, by recursive merging, when no warp was spare)
        if constexpr (!(NT / 32 > nwf<TT, TS, ROWS>()))
            panel::build_T_rec<C, NB, NT>(tau + J0, gbuf, [&](int i, int j) -> C & { return tsub[j * LDS + i]; });
        // ---- T[0:J0, J0:J0+NB] = -T[0:J0,0:J0] (Vprev^T Vs) T_sub
        // (FULL_T = false: none -- the sub-panel updates use T_sub from tsub,
        // and k_node_tu builds T off the critical path)
        if constexpr (J0 > 0 && FULL_T) {
            // only rows where both can be nonzero: LEAF rows [J0,TS); TT bottom rows [0, J0+NB)
            constexpr int KLO = TT ? NB : 0;
            sgemm<C, 2, 2, NT>(J0, NB, R - KLO,
                [&](int p, int ii) { return A[p * lda + row(ii + KLO)]; },
                [&](int ii, int a) { return Vs[(ii + KLO) * VLD + a]; },
                [&](int p, int a, C v) { gbuf[a * TS + p] = v; });
            __syncthreads();
            sgemm<C, 2, 2, NT>(J0, NB, NB,
                [&](int p, int q) { return gbuf[q * TS + p]; },
                [&](int q, int a) { return q <= a ? tsub[a * LDS + q] : C(0); },
                [&](int p, int a, C v) { wbuf[a * TS + p] = v; });
            __syncthreads();
            sgemm<C, 2, 2, NT>(J0, NB, J0,
                [&](int p, int q) { return q >= p ? Tm[q * ldt + p] : C(0); },
                [&](int q, int a) { return wbuf[a * TS + q]; },
                [&](int p, int a, C v) { Tm[(J0 + a) * ldt + p] = -v; });
        }
        if constexpr (FULL_T) {                     // (the updates below read tsub)
            for (int idx = threadIdx.x; idx < NB * NB; idx += NT) {
                const int a = idx % NB, b = idx / NB;
                if (a <= b) Tm[(J0 + b) * ldt + (J0 + a)] = tsub[b * LDS + a];
            }
            __syncthreads();
        }
        stamp(4 * (J0 / NB) + 1);
        // ---- apply the sub-panel block reflector to columns [J0+NB, TS)
        constexpr int NCOL = TS - J0 - NB;
        if constexpr (NCOL > 0) {
            sgemm<C, 2, 4, NT>(NB, NCOL, R,
                [&](int a, int i) { return Vs[i * VLD + a]; },
                [&](int i, int cc) { return A[(J0 + NB + cc) * lda + row(i)]; },
                [&](int a, int cc, C v) { wbuf[cc * NB + a] = v; });
            __syncthreads();
            sgemm<C, 2, 4, NT>(NB, NCOL, NB,
                [&](int a, int b) { return b <= a ? tsub[a * LDS + b] : C(0); },   // T^T(a,b) = T(b,a)
                [&](int b, int cc) { return wbuf[cc * NB + b]; },
                [&](int a, int cc, C v) { gbuf[cc * NB + a] = v; });
            __syncthreads();
            sgemm<C, 4, 4, NT>(R, NCOL, NB,
                [&](int i, int a) { return Vs[i * VLD + a]; },
                [&](int a, int cc) { return gbuf[cc * NB + a]; },
                [&](int i, int cc, C v) { A[(J0 + NB + cc) * lda + row(i)] -= v; });
            __syncthreads();
        }
        stamp(4 * (J0 / NB) + 2);
        qr_step<C, TS, TT, NB, J0 + NB, NT, FULL_T, ROWS>(A, lda, tau, Tm, ldt, aux, house, save_r, st);
    }
}

template <typename C, int TS, bool TT, int NT, bool FULL_T = true, int ROWS = TS, typename HS, typename SaveR>
__device__ void qr_blocked(C *A, int lda, C *tau, C *Tm, int ldt, C *aux, HS house, SaveR save_r,
                           unsigned long long *st = nullptr) {
    qr_step<C, TS, TT, NBsel<C, TS>::v, 0, NT, FULL_T, ROWS>(A, lda, tau, Tm, ldt, aux, house, save_r, st);
    if constexpr (!FULL_T)
        for (int j0 = 0; j0 < TS; j0 += NBsel<C, TS>::v) save_r(j0);
}

}  // namespace blk
}  // namespace bsvd
