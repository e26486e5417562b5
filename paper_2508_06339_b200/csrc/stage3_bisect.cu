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

template <typename OutT>
__global__ void __launch_bounds__(128) k_bisect(const double *__restrict__ o2,
                                                const double *__restrict__ scal, int64_t n,
                                                int64_t n_out, OutT *__restrict__ out,
                                                int64_t out_stride) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // output slot
    const int64_t b = blockIdx.y;
    if (k >= n_out) return;
    const double *ob = o2 + b * (2 * n - 1);
    const double unscale = scal[2 * b], gersh = scal[2 * b + 1];
    const int64_t rank = n - k;   // ascending rank of the k-th largest value
    double res = 0.0;
    if (gersh > 0.0) {
        const double pivmin = 0x1p-1000;
        const double floor_ = 0x1p-120 * gersh;
        double lo = 0.0, hi = 2.0 * gersh;
        for (int it = 0; it < 2200; ++it) {
            const double mid = 0.5 * (lo + hi);
            if (!(mid > lo && mid < hi) || hi <= floor_) break;
            const int cnt = negcount(ob, 2 * n - 1, mid, pivmin) - (int)n;   // #{sigma < mid}
            if (cnt < rank) lo = mid; else hi = mid;
        }
        res = lo * unscale;
    }
    out[b * out_stride + k] = (OutT)res;
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
    dim3 grid((unsigned)((n_out + 127) / 128), (unsigned)batch);
    k_bisect<OutT><<<grid, 128, 0, st>>>(o2, scal, n, n_out, out, out_stride);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

template cudaError_t bidiagonal_values<double>(const double *, const double *, int64_t, int64_t,
                                               double *, int64_t, int64_t, void *, cudaStream_t);
template cudaError_t bidiagonal_values<float>(const double *, const double *, int64_t, int64_t,
                                              float *, int64_t, int64_t, void *, cudaStream_t);

}  // namespace bsvd
