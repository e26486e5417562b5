// faithful.cu -- bit-faithful sm_100a versions of the reference tile kernels.
//
// Compiled with -fmad=false: the reference's numba bodies never contract
// a*b+c into an FMA, and sqrt / division stay IEEE (nvcc
// defaults), so every work-item reproduces the reference's bytes.  One CUDA
// thread per reference work-item, one CTA per reference work-group; the
// reference's private_mem arrays live in per-thread local memory (interleaved
// by the compiler, so same-index accesses across a warp coalesce) and its
// local_mem arrays in shared memory.  These kernels are the kernel-level
// parity path (bsvd_geqrt / bsvd_tsqrt_chain / bsvd_unmqr / bsvd_tsmqr_fused)
// and the BSVD_STAGE1_FAITHFUL stage-1 driver; the fast path is stage1_tree.cu.
#include "common.cuh"
#include "kernels.cuh"

namespace bsvd {

constexpr int kMaxTs = 128;
constexpr int kMaxSplit = 32;   // splitk <= min(ts, 1024 / ts) (kernels.py:52)

// Split-K segment updates (kernels.py:134-141 _geqrt_seg_update, :159-166
// _tsqrt_seg_update) are njit functions called from the Python-level split-K
// generator with x and rho' as Python floats, so numba specialises them for
// float64 scalars: for fp32 compute every updated element is
// float32(double(v) - double(rho') * (double(col) / double(x))) (resp.
// float32(double(v) / double(x))) -- one rounding instead of three.  For fp64
// the two forms coincide.  (The pivot-row element pivots[i] - rho' is numpy
// float32 - Python float, float32 arithmetic under NEP 50.)
template <typename C>
__device__ __forceinline__ C seg_upd(C v, C rhop, C c, C x) {
    return (C)((double)v - (double)rhop * ((double)c / (double)x));
}
template <typename C>
__device__ __forceinline__ C seg_div(C v, C x) {
    return (C)((double)v / (double)x);
}

// Split-K sums (kernels.py:233-283, :316-361): segment t of nsplit covers rows
// [t*ts/nsplit, (t+1)*ts/nsplit); each segment's partial is a serial sum from
// zero over its rows in [lo, ts) (zero when empty: _norm2_tail / _dot_seg
// :71-93), then _pairwise_sum (:191-199) combines the partials pairwise in
// ascending index, an odd tail carried to the next round.  nsplit == 1 is
// the plain serial sum of geqrt_kernel / tsqrt_kernel.
template <typename C, typename F>
__device__ __forceinline__ C split_sum(int ts, int nsplit, int lo, F term) {
    if (nsplit <= 1) {
        C s = C(0);
        for (int j = lo; j < ts; ++j) s += term(j);
        return s;
    }
    C v[kMaxSplit];
    for (int t = 0; t < nsplit; ++t) {
        const int s0 = t * ts / nsplit, s1 = (t + 1) * ts / nsplit;
        const int l = lo > s0 ? lo : s0;
        C s = C(0);
        for (int j = l; j < s1; ++j) s += term(j);
        v[t] = l < s1 ? s : C(0);
    }
    int len = nsplit;
    while (len > 1) {
        int m = 0;
        for (int j = 0; j + 1 < len; j += 2) v[m++] = v[j] + v[j + 1];
        if (len & 1) v[m++] = v[len - 1];
        len = m;
    }
    return v[0];
}

// kernels.py:205-230 geqrt_kernel (+ _geqrt_item :119-131, _norm2_tail :71-76,
// _dot_tail :79-84); nsplit > 1: geqrt_splitk_kernel :233-283, whose only
// arithmetic difference is the split-K order of the norm and dot sums
// (split_sum).  ts threads, one tile per CTA (blockIdx.y = batch).
template <typename S, typename C>
__global__ void __launch_bounds__(kMaxTs) k_geqrt_faithful(S *a, int64_t rs, int64_t cs,
                                                           int64_t a_bstride, int ts, C *tau,
                                                           int64_t tau_bstride, int nsplit) {
    using CV = Conv<S, C>;
    __shared__ C col[kMaxTs];
    __shared__ C nrm;
    a += blockIdx.y * a_bstride;
    tau += blockIdx.y * tau_bstride;
    const int i = threadIdx.x;
    const C zero = C(0), two = C(2), eps10 = C(10) * Eps<C>::v;
    C ai[kMaxTs];
    for (int j = 0; j < ts; ++j) ai[j] = CV::ld(at(a, j, i, rs, cs));
    C tau_i = zero;
    for (int k = 0; k < ts - 1; ++k) {
        if (i == k) {
            for (int j = 0; j < ts; ++j) col[j] = ai[j];
            nrm = split_sum<C>(ts, nsplit, k + 1, [&](int j) { return ai[j] * ai[j]; });
        }
        __syncthreads();
        if (i >= k) {
            const C rho = split_sum<C>(ts, nsplit, k + 1, [&](int j) { return ai[j] * col[j]; });
            C x, t, rhop;
            reflector_scalars(col[k], nrm, ai[k], rho, eps10, two, x, t, rhop);
            ai[k] = ai[k] - rhop;
            if (nsplit > 1) {
                if (i > k) {
                    for (int j = k + 1; j < ts; ++j) ai[j] = seg_upd(ai[j], rhop, col[j], x);
                } else {
                    for (int j = k + 1; j < ts; ++j) ai[j] = seg_div(ai[j], x);
                    tau_i = t;
                }
            } else if (i > k) {
                for (int j = k + 1; j < ts; ++j) ai[j] = ai[j] - rhop * (col[j] / x);
            } else {
                for (int j = k + 1; j < ts; ++j) ai[j] = ai[j] / x;
                tau_i = t;
            }
        }
        at(a, k, i, rs, cs) = CV::st(ai[k]);
        __syncthreads();
    }
    at(a, ts - 1, i, rs, cs) = CV::st(ai[ts - 1]);
    tau[i] = (i < ts - 1) ? tau_i : zero;
}

// kernels.py:286-313 tsqrt_kernel (+ _tsqrt_item :144-156): the [R; B_l]
// chain, R columns resident in the work-items across all l; nsplit > 1:
// tsqrt_splitk_kernel :316-361 (split-K norm / dot order, split_sum).
template <typename S, typename C, typename TileSeqT, typename TauSeqT>
__global__ void __launch_bounds__(kMaxTs) k_tsqrt_faithful(S *r, int64_t rs, int64_t cs,
                                                           TileSeqT bs, TauSeqT taus, int nb,
                                                           int ts, int nsplit) {
    using CV = Conv<S, C>;
    __shared__ C bcol[kMaxTs];
    __shared__ C scal[2];
    const int i = threadIdx.x;
    const C zero = C(0), two = C(2), eps10 = C(10) * Eps<C>::v;
    C ri[kMaxTs], bi[kMaxTs];
    for (int j = 0; j < ts; ++j) ri[j] = CV::ld(at(r, j, i, rs, cs));
    for (int l = 0; l < nb; ++l) {
        S *b = (S *)bs.get(l);
        C *tau = (C *)taus.get(l);
        for (int j = 0; j < ts; ++j) bi[j] = CV::ld(at(b, j, i, rs, cs));
        C tau_i = zero;
        for (int k = 0; k < ts; ++k) {
            if (i == k) {
                for (int j = 0; j < ts; ++j) bcol[j] = bi[j];
                scal[0] = split_sum<C>(ts, nsplit, 0, [&](int j) { return bi[j] * bi[j]; });
                scal[1] = ri[k];
            }
            __syncthreads();
            if (i >= k) {
                const C rho = split_sum<C>(ts, nsplit, 0, [&](int j) { return bi[j] * bcol[j]; });
                C x, t, rhop;
                reflector_scalars(scal[1], scal[0], ri[k], rho, eps10, two, x, t, rhop);
                ri[k] = ri[k] - rhop;
                if (nsplit > 1) {
                    if (i > k) {
                        for (int j = 0; j < ts; ++j) bi[j] = seg_upd(bi[j], rhop, bcol[j], x);
                    } else {
                        for (int j = 0; j < ts; ++j) bi[j] = seg_div(bi[j], x);
                        tau_i = t;
                    }
                } else if (i > k) {
                    for (int j = 0; j < ts; ++j) bi[j] = bi[j] - rhop * (bcol[j] / x);
                } else {
                    for (int j = 0; j < ts; ++j) bi[j] = bi[j] / x;
                    tau_i = t;
                }
            }
            __syncthreads();
        }
        for (int j = 0; j < ts; ++j) at(b, j, i, rs, cs) = CV::st(bi[j]);
        tau[i] = tau_i;
    }
    for (int j = 0; j < ts; ++j) at(r, j, i, rs, cs) = CV::st(ri[j]);
}

// kernels.py:364-389 unmqr_kernel (+ _unmqr_item :169-177): cpb columns per
// CTA; panel column and tau staged in shared memory.
template <typename S, typename C>
__global__ void __launch_bounds__(kMaxTs) k_unmqr_faithful(const S *panel, int64_t prs,
                                                           int64_t pcs, const C *tau, S *x,
                                                           int64_t xrs, int64_t xcs, int ts,
                                                           int cpb) {
    using CV = Conv<S, C>;
    __shared__ C ak[kMaxTs];
    __shared__ C tk[kMaxTs];
    const int i = threadIdx.x;
    const int64_t c = (int64_t)blockIdx.x * cpb + i;
    const C zero = C(0);
    C xi[kMaxTs];
    for (int j = 0; j < ts; ++j) xi[j] = CV::ld(at(x, j, c, xrs, xcs));
    for (int j = i; j < ts; j += cpb) tk[j] = tau[j];
    for (int k = 0; k < ts - 1; ++k) {
        for (int j = i; j < ts; j += cpb) ak[j] = CV::ld(at(panel, j, k, prs, pcs));
        __syncthreads();
        C s = zero;
        for (int j = k + 1; j < ts; ++j) s += xi[j] * ak[j];
        C rho = tk[k] * (xi[k] + s);
        xi[k] = xi[k] - rho;
        for (int j = k + 1; j < ts; ++j) xi[j] = xi[j] - rho * ak[j];
        __syncthreads();
    }
    for (int j = 0; j < ts; ++j) at(x, j, c, xrs, xcs) = CV::st(xi[j]);
}

// kernels.py:392-421 tsmqr_kernel (+ _tsmqr_item :180-188): Y resident in
// the work-items across all body rows, written back once.
template <typename S, typename C, typename TileSeqT, typename TauSeqT>
__global__ void __launch_bounds__(kMaxTs) k_tsmqr_faithful(S *y, int64_t rs, int64_t cs,
                                                           TileSeqT xs, TileSeqT vs, TauSeqT taus,
                                                           int nb, int ts, int cpb) {
    using CV = Conv<S, C>;
    __shared__ C ak[kMaxTs];
    __shared__ C tk[kMaxTs];
    const int i = threadIdx.x;
    const int64_t c = (int64_t)blockIdx.x * cpb + i;
    const C zero = C(0);
    C yi[kMaxTs], xi[kMaxTs];
    for (int j = 0; j < ts; ++j) yi[j] = CV::ld(at(y, j, c, rs, cs));
    for (int l = 0; l < nb; ++l) {
        S *x = (S *)xs.get(l);
        const S *v = (const S *)vs.get(l);
        const C *tau = (const C *)taus.get(l);
        for (int j = 0; j < ts; ++j) xi[j] = CV::ld(at(x, j, c, rs, cs));
        for (int j = i; j < ts; j += cpb) tk[j] = tau[j];
        for (int k = 0; k < ts; ++k) {
            for (int j = i; j < ts; j += cpb) ak[j] = CV::ld(at(v, j, k, rs, cs));
            __syncthreads();
            C s = zero;
            for (int j = 0; j < ts; ++j) s += ak[j] * xi[j];
            s = (s + yi[k]) * tk[k];
            yi[k] = yi[k] - s;
            for (int j = 0; j < ts; ++j) xi[j] = xi[j] - s * ak[j];
            __syncthreads();
        }
        for (int j = 0; j < ts; ++j) at(x, j, c, rs, cs) = CV::st(xi[j]);
    }
    for (int j = 0; j < ts; ++j) at(y, j, c, rs, cs) = CV::st(yi[j]);
}

// ------------------------------------------------------------------------
// launchers

template <typename S, typename C>
cudaError_t launch_geqrt_faithful(S *a, int64_t rs, int64_t cs, int ts, C *tau, int64_t batch,
                                  int64_t a_bstride, int64_t tau_bstride, cudaStream_t st, int nsplit) {
    k_geqrt_faithful<S, C><<<dim3(1, (unsigned)batch), ts, 0, st>>>(a, rs, cs, a_bstride, ts, tau,
                                                                    tau_bstride, nsplit);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

template <typename S, typename C, typename TS_, typename TA_>
cudaError_t launch_tsqrt_faithful(S *r, int64_t rs, int64_t cs, TS_ bs, TA_ taus, int nb, int ts,
                                  cudaStream_t st, int nsplit) {
    if (nb <= 0) return cudaSuccess;
    k_tsqrt_faithful<S, C, TS_, TA_><<<1, ts, 0, st>>>(r, rs, cs, bs, taus, nb, ts, nsplit);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

template <typename S, typename C>
cudaError_t launch_unmqr_faithful(const S *panel, int64_t prs, int64_t pcs, const C *tau, S *x,
                                  int64_t xrs, int64_t xcs, int64_t ncols, int ts, int cpb,
                                  cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    k_unmqr_faithful<S, C><<<(unsigned)(ncols / cpb), cpb, 0, st>>>(panel, prs, pcs, tau, x, xrs,
                                                                    xcs, ts, cpb);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

template <typename S, typename C, typename TS_, typename TA_>
cudaError_t launch_tsmqr_faithful(S *y, int64_t rs, int64_t cs, TS_ xs, TS_ vs, TA_ taus, int nb,
                                  int64_t ncols, int ts, int cpb, cudaStream_t st) {
    if (nb <= 0 || ncols <= 0) return cudaSuccess;
    k_tsmqr_faithful<S, C, TS_, TA_><<<(unsigned)(ncols / cpb), cpb, 0, st>>>(y, rs, cs, xs, vs,
                                                                              taus, nb, ts, cpb);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

// bandreduce.py:31-88 getsmqrt (fused) + :91-120 banddiag, faithful order.
// a: padded column-major n x n (n = N*ts); tau: ts x 2N^2 compute-dtype store.
template <typename S, typename C>
cudaError_t banddiag_faithful(S *a, int64_t n, int ts, int cpb, C *tau, cudaStream_t st, int splitk) {
    const int N = (int)(n / ts);
    auto sweep = [&](int k, bool lq) -> cudaError_t {
        const int64_t rs = lq ? n : 1, cs = lq ? 1 : n;
        const int side = lq ? 1 : 0;
        const int top = lq ? k + 1 : k;
        if (top >= N) return cudaSuccess;
        auto tile = [&](int tr, int tc) { return a + (int64_t)tr * ts * rs + (int64_t)tc * ts * cs; };
        auto tauc = [&](int kk, int ll) {
            return tau + ((int64_t)side * N * N + (int64_t)kk * N + ll) * ts;
        };
        S *diag = tile(top, k);
        cudaError_t e = launch_geqrt_faithful<S, C>(diag, rs, cs, ts, tauc(k, top), 1, 0, 0, st, splitk);
        if (e != cudaSuccess) return e;
        const int ntrail = N - 1 - k;
        S *top_slab = tile(top, k + 1);
        if (ntrail > 0) {
            e = launch_unmqr_faithful<S, C>(diag, rs, cs, tauc(k, top), top_slab, rs, cs,
                                            (int64_t)ntrail * ts, ts, cpb, st);
            if (e != cudaSuccess) return e;
        }
        const int nrows = N - (top + 1);
        if (nrows <= 0) return cudaSuccess;
        const int64_t tstep = (int64_t)ts * rs * (int64_t)sizeof(S);
        TileSeq vts{(char *)tile(top + 1, k), tstep};
        TileSeq body{(char *)tile(top + 1, k + 1), tstep};
        TileSeq tcs{(char *)tauc(k, top + 1), (int64_t)ts * (int64_t)sizeof(C)};
        e = launch_tsqrt_faithful<S, C>(diag, rs, cs, vts, tcs, nrows, ts, st, splitk);
        if (e != cudaSuccess) return e;
        if (ntrail > 0)
            e = launch_tsmqr_faithful<S, C>(top_slab, rs, cs, body, vts, tcs, nrows,
                                            (int64_t)ntrail * ts, ts, cpb, st);
        return e;
    };
    for (int k = 0; k < N - 1; ++k) {
        cudaError_t e = sweep(k, false);
        if (e != cudaSuccess) return e;
        e = sweep(k, true);
        if (e != cudaSuccess) return e;
    }
    return sweep(N - 1, false);
}

#define INST(S, C)                                                                              \
    template cudaError_t launch_geqrt_faithful<S, C>(S *, int64_t, int64_t, int, C *, int64_t,   \
                                                     int64_t, int64_t, cudaStream_t, int);       \
    template cudaError_t launch_tsqrt_faithful<S, C, TileArr, TileArr>(                          \
        S *, int64_t, int64_t, TileArr, TileArr, int, int, cudaStream_t, int);                   \
    template cudaError_t launch_unmqr_faithful<S, C>(const S *, int64_t, int64_t, const C *, S *, \
                                                     int64_t, int64_t, int64_t, int, int,         \
                                                     cudaStream_t);                              \
    template cudaError_t launch_tsmqr_faithful<S, C, TileArr, TileArr>(                          \
        S *, int64_t, int64_t, TileArr, TileArr, TileArr, int, int64_t, int, int, cudaStream_t);  \
    template cudaError_t banddiag_faithful<S, C>(S *, int64_t, int, int, C *, cudaStream_t, int);
INST(double, double)
INST(float, float)
INST(__half, float)
#undef INST

}  // namespace bsvd
