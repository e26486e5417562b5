// stage3_bisect.cu -- bidiagonal -> singular values on the GPU.
//
// Replaces the reference's host Demmel-Kahan QR iteration
// (secondstage.py:221-420, :473-507) with Sturm-count bisection on the
// Golub-Kahan tridiagonal TGK = tridiag(0; d1, e1, d2, ..., e_{n-1}, dn)
// whose eigenvalues are +-sigma_i.  Always float64 like the reference
// (secondstage.py:486-488).  Every value is independent: one thread per
// requested value, bisection on its ascending rank i with the invariant
// N(lo) < i <= N(hi), N(x) = #{sigma < x} = negcount(TGK - xI) - n, run until
// lo and hi are adjacent doubles, so sigma_i = lo exactly when the count is
// exact (diag(3,2,1) -> [3,2,1] bit-for-bit, test_secondstage.py:99-102).
// The off-diagonals are first scaled by a power of two so max|o| is in
// [1,2): power-of-two input scaling therefore commutes bit-exactly
// (test_secondstage.py:170-180), and o^2 can neither overflow nor underflow
// for representable inputs.  Only the largest n_out values are computed (the
// zero padding adds the smallest ones, matrix.py:163-181), already in the
// descending order secondstage.py:506 produces with a sort.
#include "common.cuh"
#include "kernels.cuh"

namespace bsvd {

// Per-matrix prep: o2[j] = (o_j * 2^-p)^2, scal = {2^p, gersh_scaled}.
__global__ void __launch_bounds__(256) k_bisect_prep(const double *__restrict__ d,
                                                     const double *__restrict__ e, int64_t n,
                                                     double *__restrict__ o2,
                                                     double *__restrict__ scal) {
    const int64_t b = blockIdx.x;
    d += b * n;
    e += b * (n > 1 ? n - 1 : 0);
    o2 += b * (2 * n - 1);
    scal += b * 2;
    __shared__ double red[256];
    double m = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) m = fmax(m, fabs(d[j]));
    for (int64_t j = threadIdx.x; j + 1 < n; j += blockDim.x) m = fmax(m, fabs(e[j]));
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    const double omax = red[0];
    __syncthreads();
    double sc = 1.0;
    if (omax > 0.0) {
        int ex;
        frexp(omax, &ex);          // omax = f * 2^ex, f in [0.5, 1)
        sc = ldexp(1.0, 1 - ex);   // omax * sc in [1, 2)
    }
    double g = 0.0;
    for (int64_t j = threadIdx.x; j < 2 * n - 1; j += blockDim.x) {
        const double o = ((j & 1) ? e[j >> 1] : d[j >> 1]) * sc;
        o2[j] = o * o;
        const double prev = j > 0 ? fabs(((j - 1) & 1) ? e[(j - 1) >> 1] : d[(j - 1) >> 1]) * sc : 0.0;
        g = fmax(g, fabs(o) + prev);
    }
    if (threadIdx.x == 0 && n == 1) g = fabs(d[0]) * sc;
    red[threadIdx.x] = g;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        scal[0] = 1.0 / sc;   // exact: sc is a power of two
        scal[1] = red[0];
    }
}

// #{eigenvalues of TGK < x} for the scaled problem (LAPACK dstebz-style
// negcount with a pivot floor; zero diagonal so a_j - x = -x).
__device__ __forceinline__ int negcount(const double *__restrict__ o2, int64_t m, double x,
                                        double pivmin) {
    // A vanishing pivot keeps its sign (+0 -> +pivmin): at x exactly equal to
    // an eigenvalue the count then excludes it, so exact inputs converge to
    // the exact value (LAPACK's q = -pivmin would count it).
    double q = -x;
    if (fabs(q) < pivmin) q = (q < 0.0) ? -pivmin : pivmin;
    int cnt = q < 0.0;
    for (int64_t j = 0; j < m; ++j) {
        q = -x - __ldg(o2 + j) / q;
        if (fabs(q) < pivmin) q = (q < 0.0) ? -pivmin : pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

// Two interleaved Sturm counts (independent dependency chains for ILP).
__device__ __forceinline__ void negcount2(const double *__restrict__ o2, int64_t m, double x0,
                                          double x1, double pivmin, int &c0, int &c1) {
    double q0 = -x0, q1 = -x1;
    if (fabs(q0) < pivmin) q0 = (q0 < 0.0) ? -pivmin : pivmin;
    if (fabs(q1) < pivmin) q1 = (q1 < 0.0) ? -pivmin : pivmin;
    int n0 = q0 < 0.0, n1 = q1 < 0.0;
    for (int64_t j = 0; j < m; ++j) {
        const double o = __ldg(o2 + j);
        q0 = -x0 - o / q0;
        q1 = -x1 - o / q1;
        if (fabs(q0) < pivmin) q0 = (q0 < 0.0) ? -pivmin : pivmin;
        if (fabs(q1) < pivmin) q1 = (q1 < 0.0) ? -pivmin : pivmin;
        n0 += q0 < 0.0;
        n1 += q1 < 0.0;
    }
    c0 = n0;
    c1 = n1;
}

// Multisection: a group of kLanes lanes owns one value; each round the lanes
// evaluate 2*kLanes interior points of [lo, hi] (two interleaved Sturm
// chains per lane) and keep the sub-interval where the count crosses the
// value's rank (4.1 bits per round instead of 1, and 16x the independent
// chains of one-thread-per-value bisection).  Once the points collapse (a
// few ulps) the group finishes with plain bisection.  The invariant
// N(lo) < rank <= N(hi) is the same, so the result is identical to bisection
// to adjacent doubles.
template <int kLanes, typename OutT>
__global__ void __launch_bounds__(128) k_bisect(const double *__restrict__ o2,
                                                const double *__restrict__ scal, int64_t n,
                                                int64_t n_out, OutT *__restrict__ out,
                                                int64_t out_stride) {
    const int lane = threadIdx.x & 31;
    const int sub = lane % kLanes;                       // lane within the value's group
    const unsigned gmask = ((1u << kLanes) - 1u) << (lane - sub);
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kLanes;   // output slot
    const int64_t b = blockIdx.y;
    const bool active = k < n_out;
    const double *ob = o2 + b * (2 * n - 1);
    const double unscale = scal[2 * b], gersh = scal[2 * b + 1];
    const int64_t rank = n - (active ? k : 0);           // ascending rank of the k-th largest
    double res = 0.0;
    if (gersh > 0.0) {
        const double pivmin = 0x1p-1000;
        const double floor_ = 0x1p-120 * gersh;
        double lo = 0.0, hi = 2.0 * gersh;
        constexpr int NP = 2 * kLanes;                   // points per round
        for (int round = 0; round < (kLanes > 1 ? 40 : 0); ++round) {
            if (hi <= floor_) break;
            const double h = (hi - lo) / (NP + 1);
            const double x0 = lo + h * (2 * sub + 1), x1 = lo + h * (2 * sub + 2);
            // points must be strictly increasing inside (lo, hi); else bisect
            const bool ok = h > 0.0 && (lo + h) > lo && (lo + h * NP) < hi && x0 < x1;
            if (!__all_sync(gmask, ok)) break;
            int c0, c1;
            negcount2(ob, 2 * n - 1, x0, x1, pivmin, c0, c1);
            c0 -= (int)n;
            c1 -= (int)n;
            // bit t-1 of M <=> point t has N(x) < rank; lo moves to the HIGHEST such
            // point (robust even if rounding made the computed counts non-monotone:
            // every point above it has N >= rank, so hi = the next point).
            const unsigned below = __ballot_sync(gmask, c0 < rank) >> (lane - sub);
            const unsigned below1 = __ballot_sync(gmask, c1 < rank) >> (lane - sub);
            unsigned M = 0;
#pragma unroll
            for (int s = 0; s < kLanes; ++s)
                M |= (((below >> s) & 1u) << (2 * s)) | (((below1 >> s) & 1u) << (2 * s + 1));
            const int nb = M ? 32 - __clz(M) : 0;             // highest point index below rank
            const double nlo = nb > 0 ? lo + h * nb : lo;
            const double nhi = nb < NP ? lo + h * (nb + 1) : hi;
            lo = nlo;
            hi = nhi;
        }
        for (int it = 0; it < 200; ++it) {               // finish: bisection to adjacent doubles
            const double mid = 0.5 * (lo + hi);
            if (!(mid > lo && mid < hi) || hi <= floor_) break;
            const int cnt = negcount(ob, 2 * n - 1, mid, pivmin) - (int)n;
            if (cnt < rank) lo = mid; else hi = mid;
        }
        res = lo * unscale;
    }
    if (active && sub == 0) out[b * out_stride + k] = (OutT)res;
}

size_t bisect_workspace_bytes(int64_t n, int64_t batch) {
    return (size_t)batch * ((size_t)(2 * n) * sizeof(double) + 2 * sizeof(double)) + 256;
}

template <typename OutT>
cudaError_t bidiagonal_values(const double *d, const double *e, int64_t n, int64_t batch,
                              OutT *out, int64_t n_out, int64_t out_stride, void *ws,
                              cudaStream_t st) {
    if (n < 1 || batch < 1) return cudaSuccess;
    double *o2 = (double *)ws;
    double *scal = o2 + batch * (2 * n - 1);
    k_bisect_prep<<<(unsigned)batch, 256, 0, st>>>(d, e, n, o2, scal);
    bsvd_host::count_launch();
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    // Multisection when values are scarce (one large matrix), plain bisection
    // (one lane per value, least total work) when a batch supplies the parallelism.
    if (n_out * batch >= 131072) {
        dim3 grid((unsigned)((n_out + 127) / 128), (unsigned)batch);
        k_bisect<1, OutT><<<grid, 128, 0, st>>>(o2, scal, n, n_out, out, out_stride);
    } else {
        dim3 grid((unsigned)((n_out * 8 + 127) / 128), (unsigned)batch);
        k_bisect<8, OutT><<<grid, 128, 0, st>>>(o2, scal, n, n_out, out, out_stride);
    }
    bsvd_host::count_launch();
    return cudaGetLastError();
}

template cudaError_t bidiagonal_values<double>(const double *, const double *, int64_t, int64_t,
                                               double *, int64_t, int64_t, void *, cudaStream_t);
template cudaError_t bidiagonal_values<float>(const double *, const double *, int64_t, int64_t,
                                              float *, int64_t, int64_t, void *, cudaStream_t);

}  // namespace bsvd
