// stage2_chase.cu -- band -> bidiagonal on the GPU.
//
// Replaces the reference's serial Givens chase (secondstage.py:95-146,
// :452-470) with a Householder bulge chase whose sweeps run as a pipelined
// wavefront inside ONE persistent cooperative kernel:
//
//  * sweep s annihilates row s beyond the superdiagonal with a right
//    reflector on columns [s+1, s+1+b) ("op 0"), then chases the bulge:
//    task t (r0 = s+1+t*b) = left reflector on rows [r0, r0+b) (pivot column
//    r0, applied to columns [r0, r0+2b)) and right reflector on columns
//    [r0+b, r0+2b) (pivot row r0, applied to rows [r0, r0+2b));
//  * op i of sweep s may start once op i+3 of sweep s-1 has finished (the
//    largest overlapping op, derived from the op footprints -- DESIGN.md
//    "stage 2"); a per-sweep progress counter (release/acquire at gpu scope)
//    carries that dependency between CTAs;
//  * (matrix, sweep) work items are dealt round-robin in sweep-major order,
//    so a batch of small matrices fills the GPU and a single large matrix
//    pipelines its sweeps across CTAs.  The smallest unfinished item never
//    waits, and the cooperative launch guarantees co-residency: no deadlock.
//
// Arithmetic is float64 for every storage precision (the reference chases in
// the compute dtype, whose FP32 Givens chase dominates its error budget,
// SURVEY.md 4).  The band lives in packed column-major storage with room for
// the bulges (r - c in [-2b, b]), 3b+1 doubles per column: 50 MB at
// n = 16384, b = 128, i.e. L2-resident on B200 (126 MB L2).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace bsvd {

struct Band {
    double *p;
    int64_t n, ld;
    int b;
    __device__ __forceinline__ double *at(int64_t r, int64_t c) const {
        return p + c * ld + (r - c + 2 * b);
    }
};

__device__ __forceinline__ int chase_nops(int64_t s, int64_t n, int b) {
    int cnt = 1;
    for (int64_t r0 = s + 1; r0 < n; r0 += b) {
        ++cnt;                      // left op
        if (r0 + b >= n) break;
        ++cnt;                      // right op
    }
    return cnt;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Householder generation (LAPACK dlarfg convention): x -> beta e1 with
// H = I - tau v v^T, v[0] = 1.  Executed by warp 0; v (len L) into vs.
// Returns tau (0 when the tail is already zero: H = I).
__device__ double make_reflector_warp(const Band &A, int64_t r0, int64_t c0, bool column, int L,
                                      double *vs) {
    const int lane = threadIdx.x & 31;
    double alpha = __ldcg(A.at(r0, c0));
    double sig = 0.0;
    for (int j = 1 + lane; j < L; j += 32) {
        const double xj = column ? __ldcg(A.at(r0 + j, c0)) : __ldcg(A.at(r0, c0 + j));
        vs[j] = xj;
        sig += xj * xj;
    }
    sig = warp_sum(sig);
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (sig != 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sig), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
    }
    __syncwarp();
    for (int j = 1 + lane; j < L; j += 32) {
        vs[j] = vs[j] * scale;
        if (column) __stcg(A.at(r0 + j, c0), 0.0); else __stcg(A.at(r0, c0 + j), 0.0);
    }
    if (lane == 0) {
        vs[0] = 1.0;
        __stcg(A.at(r0, c0), beta);
    }
    return tau;
}

// Left op: pivot column p, rows [p, p+L), applied to columns (p, chi).
__device__ void chase_left(const Band &A, int64_t p, int L, int64_t chi, double *vs,
                           double *tau_s) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (warp == 0) {
        const double t = make_reflector_warp(A, p, p, true, L, vs);
        if (lane == 0) *tau_s = t;
    }
    __syncthreads();
    const double tau = *tau_s;
    if (tau == 0.0) return;
    constexpr int kMaxPer = 4;   // L <= 128 rows -> <= 4 per lane
    for (int64_t c = p + 1 + warp; c < chi; c += nw) {
        double xv[kMaxPer];
        double w = 0.0;
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
            const int j = lane + 32 * q;
            xv[q] = (j < L) ? __ldcg(A.at(p + j, c)) : 0.0;
            if (j < L) w += vs[j] * xv[q];
        }
        w = warp_sum(w) * tau;
#pragma unroll
        for (int q = 0; q < kMaxPer; ++q) {
            const int j = lane + 32 * q;
            if (j < L) __stcg(A.at(p + j, c), xv[q] - w * vs[j]);
        }
    }
}

// Right op: pivot row p, columns [c0, c0+L), applied to rows [rlo, rhi) \ {p}.
__device__ void chase_right(const Band &A, int64_t p, int64_t c0, int L, int64_t rlo,
                            int64_t rhi, double *vs, double *tau_s) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        const double t = make_reflector_warp(A, p, c0, false, L, vs);
        if (lane == 0) *tau_s = t;
    }
    __syncthreads();
    const double tau = *tau_s;
    if (tau == 0.0) return;
    for (int64_t r = rlo + threadIdx.x; r < rhi; r += blockDim.x) {
        if (r == p) continue;
        double w = 0.0;
        for (int j = 0; j < L; ++j) w += __ldcg(A.at(r, c0 + j)) * vs[j];
        w *= tau;
        for (int j = 0; j < L; ++j) {
            double *q = A.at(r, c0 + j);
            __stcg(q, __ldcg(q) - w * vs[j]);
        }
    }
}

__global__ void __launch_bounds__(256) k_chase(double *band, int64_t n, int b, int64_t ld,
                                               int64_t batch, int *progress, int64_t nitems) {
    __shared__ double vs[128];
    __shared__ double tau_s;
    for (int64_t w = blockIdx.x; w < nitems; w += gridDim.x) {
        const int64_t s = w / batch, m = w % batch;
        const Band A{band + m * n * ld, n, ld, b};
        int *prog = progress + m * n;
        const int nops = chase_nops(s, n, b);
        const int nprev = s > 0 ? chase_nops(s - 1, n, b) : 0;
        for (int i = 0; i < nops; ++i) {
            if (s > 0) {
                if (threadIdx.x == 0) {
                    const int need = min(i + 4, nprev);
                    while (ld_acquire(prog + s - 1) < need) __nanosleep(40);
                }
                __syncthreads();
            }
            if (i == 0) {
                const int64_t chi = min(s + 1 + b, n);
                if (chi - (s + 1) >= 2) chase_right(A, s, s + 1, (int)(chi - (s + 1)), s, chi, vs, &tau_s);
            } else {
                const int64_t t = (i - 1) / 2;
                const int64_t r0 = s + 1 + t * b;
                if (((i - 1) & 1) == 0) {
                    const int64_t rhi = min(r0 + b, n);
                    if (rhi - r0 >= 2) chase_left(A, r0, (int)(rhi - r0), min(r0 + 2 * b, n), vs, &tau_s);
                } else {
                    const int64_t c0 = r0 + b, c1 = min(r0 + 2 * b, n);
                    if (c1 - c0 >= 2) chase_right(A, r0, c0, (int)(c1 - c0), r0, c1, vs, &tau_s);
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                st_release(prog + s, i + 1);
            }
        }
    }
}

// Pack the upper band (0 <= c - r <= bw) of a column-major S matrix into the
// float64 chase layout (bulge room zeroed by a preceding memset).
template <typename S>
__global__ void k_pack_band(const S *__restrict__ a, int64_t n, int64_t lda, int64_t a_bstride,
                            int bw, double *__restrict__ band, int64_t ld, int b) {
    const int64_t m = blockIdx.y;
    a += m * a_bstride;
    band += m * n * ld;
    const int64_t total = n * (int64_t)(bw + 1);
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx / (bw + 1);
        const int64_t r = c - bw + idx % (bw + 1);
        if (r < 0) continue;
        const double v = to_f64(a[c * lda + r]);
        band[c * ld + (r - c + 2 * b)] = v;
    }
}

__global__ void k_extract_bidiag(const double *__restrict__ band, int64_t n, int64_t ld, int b,
                                 double *__restrict__ d, double *__restrict__ e) {
    const int64_t m = blockIdx.y;
    band += m * n * ld;
    d += m * n;
    e += m * (n - 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        d[i] = band[i * ld + 2 * b];
        if (i + 1 < n) e[i] = band[(i + 1) * ld + (2 * b - 1)];
    }
}

size_t chase_workspace_bytes(int64_t n, int bw, int64_t batch) {
    const int64_t ld = 3 * (int64_t)bw + 1;
    return (size_t)batch * (size_t)n * ((size_t)ld * sizeof(double) + sizeof(int)) + 512;
}

template <typename S>
cudaError_t band_to_bidiagonal(const S *a, int64_t n, int64_t lda, int bw, int64_t batch,
                               int64_t a_bstride, double *d, double *e, void *ws,
                               cudaStream_t st) {
    if (n < 1 || batch < 1) return cudaSuccess;
    const int b = bw;
    const int64_t ld = 3 * (int64_t)b + 1;
    double *band = (double *)ws;
    int *progress = (int *)(band + batch * n * ld);
    cudaError_t err = cudaMemsetAsync(band, 0, (size_t)batch * n * ld * sizeof(double), st);
    if (err != cudaSuccess) return err;
    err = cudaMemsetAsync(progress, 0, (size_t)batch * n * sizeof(int), st);
    if (err != cudaSuccess) return err;
    {
        const int64_t total = n * (int64_t)(bw + 1);
        dim3 grid((unsigned)std::min<int64_t>((total + 255) / 256, 4096), (unsigned)batch);
        k_pack_band<S><<<grid, 256, 0, st>>>(a, n, lda, a_bstride, bw, band, ld, b);
        bsvd_host::count_launch();
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
    }
    if (n > 2) {
        int dev = 0, nsm = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chase, 256, 0);
        int64_t nitems = (n - 2) * batch;   // sweeps 0..n-3 do work (reference loop bound)
        int64_t grid = std::min<int64_t>(nitems, (int64_t)nsm * std::max(per_sm, 1));
        int64_t n_ = n, ld_ = ld, batch_ = batch;
        int b_ = b;
        void *args[] = {&band, &n_, &b_, &ld_, &batch_, &progress, &nitems};
        err = cudaLaunchCooperativeKernel((void *)k_chase, dim3((unsigned)grid), dim3(256), args, 0, st);
        bsvd_host::count_launch();
        if (err != cudaSuccess) return err;
    }
    dim3 g2((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)batch);
    k_extract_bidiag<<<g2, 256, 0, st>>>(band, n, ld, b, d, e);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

template cudaError_t band_to_bidiagonal<double>(const double *, int64_t, int64_t, int, int64_t,
                                                int64_t, double *, double *, void *, cudaStream_t);
template cudaError_t band_to_bidiagonal<float>(const float *, int64_t, int64_t, int, int64_t,
                                               int64_t, double *, double *, void *, cudaStream_t);
template cudaError_t band_to_bidiagonal<__half>(const __half *, int64_t, int64_t, int, int64_t,
                                                int64_t, double *, double *, void *, cudaStream_t);

}  // namespace bsvd
