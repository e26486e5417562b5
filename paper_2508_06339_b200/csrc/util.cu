// util.cu -- copy-in / padding / validation and band clean-up kernels.
#include "common.cuh"
#include "kernels.cuh"

namespace bsvd {

__device__ __forceinline__ bool is_finite_v(double v) { return isfinite(v); }
__device__ __forceinline__ bool is_finite_v(float v) { return isfinite(v); }
__device__ __forceinline__ bool is_finite_v(__half v) { return isfinite(__half2float(v)); }

// matrix.py:163-181 pad_to_tiles + secondstage.py:518-519 finite check,
// fused: the padded working copy is written column-major (ld = np) and any
// NaN/Inf raises a flag the host reads before launching stage 1.
template <typename S>
__global__ void k_copy_in_pad(const S *__restrict__ src, int64_t n, int64_t lda, int64_t sbs,
                              S *__restrict__ dst, int64_t np, int *__restrict__ flag) {
    const int64_t m = blockIdx.y;
    src += m * sbs;
    dst += m * np * np;
    const int64_t total = np * np;
    bool bad = false;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx / np, r = idx % np;
        S v = S(0.0f);
        if (r < n && c < n) {
            v = src[c * lda + r];
            bad |= !is_finite_v(v);
        }
        dst[idx] = v;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, 1);
}

template <typename S>
cudaError_t copy_in_pad(const S *src, int64_t n, int64_t lda, int64_t src_bstride, S *dst,
                        int64_t np, int64_t batch, int *nonfinite_flag, cudaStream_t st) {
    const int64_t total = np * np;
    dim3 grid((unsigned)std::min<int64_t>((total + 255) / 256, 8192), (unsigned)batch);
    k_copy_in_pad<S><<<grid, 256, 0, st>>>(src, n, lda, src_bstride, dst, np, nonfinite_flag);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

// bandreduce.py:113-120 _clear_outside_band.
template <typename S>
__global__ void k_clear_outside_band(S *a, int64_t n, int bw) {
    const int64_t m = blockIdx.y;
    a += m * n * n;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n * n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx / n, r = idx % n;
        if (r > c || c > r + bw) a[idx] = S(0.0f);
    }
}

template <typename S>
cudaError_t clear_outside_band(S *a, int64_t n, int bw, int64_t batch, cudaStream_t st) {
    dim3 grid((unsigned)std::min<int64_t>((n * n + 255) / 256, 8192), (unsigned)batch);
    k_clear_outside_band<S><<<grid, 256, 0, st>>>(a, n, bw);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

#define INST(S)                                                                                  \
    template cudaError_t copy_in_pad<S>(const S *, int64_t, int64_t, int64_t, S *, int64_t,       \
                                        int64_t, int *, cudaStream_t);                           \
    template cudaError_t clear_outside_band<S>(S *, int64_t, int, int64_t, cudaStream_t);
INST(double)
INST(float)
INST(__half)
#undef INST

}  // namespace bsvd
