// util.cu -- copy-in / padding / validation and band clean-up kernels.
#include "common.cuh"
#include "kernels.cuh"

namespace bsvd {

__device__ __forceinline__ bool is_finite_v(double v) { return isfinite(v); }
__device__ __forceinline__ bool is_finite_v(float v) { return isfinite(v); }
__device__ __forceinline__ bool is_finite_v(__half v) { return isfinite(__half2float(v)); }
// v * 2^k, exact (sc a power of two; the product stays in range by construction)
__device__ __forceinline__ double scale_pow2(double v, double sc) { return v * sc; }
__device__ __forceinline__ float scale_pow2(float v, double sc) { return v * (float)sc; }
__device__ __forceinline__ __half scale_pow2(__half v, double sc) {
    return __float2half_rn(__half2float(v) * (float)sc);
}

// matrix.py:163-181 pad_to_tiles + secondstage.py:518-519 finite check,
// fused: the padded working copy is written column-major (ld = np) and any
// NaN/Inf raises a flag the host reads before launching stage 1.  The fast
// path also normalises each matrix by a power of two (max |a| into [1, 2))
// when it lies outside the ordinary range (always for fp16 storage; see
// input_scale): floating-point arithmetic commutes exactly with power-of-two
// scaling, so ordinary inputs give the same bits either way, and inputs near
// the range ends (1e-30, 1e30 in fp32) no longer under/overflow the squared
// norms of the panel and chase reflectors; the values are multiplied back
// exactly at the end.  max |a| comes out of the copy-in pass itself.
// scale = 2^(1 - e) with max|a| = f 2^e, f in [0.5, 1): max|a| * scale in [1, 2)
__device__ __forceinline__ double pow2_scale(unsigned long long bits) {
    const double mx = __longlong_as_double((long long)bits);
    if (!(mx > 0.0) || !isfinite(mx)) return 1.0;
    int ex;
    frexp(mx, &ex);
    return ldexp(1.0, 1 - ex);
}

// fp32 / fp64 working copies: ordinary inputs (max |a| in [2^-24, 2^24]) need
// no normalisation (their squared norms stay far inside the range), so the
// copy-in computes max |a| on the fly and a rescale pass runs only outside
// that range.  fp16 storage always normalises (its intermediate column norms
// would otherwise leave the half range).
template <typename S>
__device__ __forceinline__ double input_scale(unsigned long long bits) {
    if constexpr (sizeof(S) != 2) {
        const double mx = __longlong_as_double((long long)bits);
        if (mx >= 0x1p-24 && mx <= 0x1p24) return 1.0;
    }
    return pow2_scale(bits);
}

// amax_acc: accumulate max |a| of the copied elements (unscaled copy) instead
// of scaling by a precomputed amax.
template <typename S>
__global__ void k_copy_in_pad(const S *__restrict__ src, int64_t n, int64_t lda, int64_t sbs,
                              S *__restrict__ dst, int64_t np, int *__restrict__ flag,
                              const unsigned long long *__restrict__ amax, double *__restrict__ unscale,
                              unsigned long long *__restrict__ amax_acc) {
    const int64_t m = blockIdx.y;
    src += m * sbs;
    dst += m * np * np;
    const double sc = amax ? pow2_scale(amax[m]) : 1.0;   // exact: a power of two
    if (unscale && blockIdx.x == 0 && threadIdx.x == 0) unscale[m] = 1.0 / sc;
    bool bad = false, vdone = false;
    float mxf = 0.f;      // max |a| of this thread's elements (fp32 sweep)
    double mxd = 0.0;
    if constexpr (sizeof(S) == 4) {
        if ((n & 3) == 0 && (np & 3) == 0 && (lda & 3) == 0 && ((uintptr_t)src & 15) == 0 &&
            ((uintptr_t)dst & 15) == 0) {                  // float4 sweep
            vdone = true;
            for (int64_t c = blockIdx.x; c < np; c += gridDim.x) {
                const float4 *col = reinterpret_cast<const float4 *>(src + c * lda);
                float4 *out = reinterpret_cast<float4 *>(dst + c * np);
#pragma unroll 4
                for (int64_t r = threadIdx.x; r < np / 4; r += blockDim.x) {
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (4 * r < n && c < n) {
                        v = col[r];
                        bad |= !(isfinite(v.x) && isfinite(v.y) && isfinite(v.z) && isfinite(v.w));
                        mxf = fmaxf(mxf, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
                        if (amax) {
                            const float f = (float)sc;
                            v.x *= f; v.y *= f; v.z *= f; v.w *= f;
                        }
                    }
                    out[r] = v;
                }
            }
        }
    }
    for (int64_t c = vdone ? np : blockIdx.x; c < np; c += gridDim.x) {   // column-wise, coalesced
        const S *col = src + c * lda;
        S *out = dst + c * np;
#pragma unroll 4
        for (int64_t r = threadIdx.x; r < np; r += blockDim.x) {
            S v = S(0.0f);
            if (r < n && c < n) {
                v = col[r];
                bad |= !is_finite_v(v);
                const double av = fabs(to_f64(v));
                mxd = av > mxd ? av : mxd;     // NaN never wins (the finite check reports it)
                if (amax) v = scale_pow2(v, sc);
            }
            out[r] = v;
        }
    }
    if (amax_acc) {
        __shared__ double red[32];
        double mx = fmax((double)mxf, mxd);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
            atomicMax(amax_acc + m, (unsigned long long)__double_as_longlong(mx));
        }
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, 1);
}

// After an unscaled copy-in: unscale[m] = 1 / scale and, only when the input
// is outside the ordinary range, the padded copy *= scale (exact).
template <typename S>
__global__ void __launch_bounds__(256) k_rescale(S *__restrict__ dst, int64_t np,
                                                 const unsigned long long *__restrict__ amax,
                                                 double *__restrict__ unscale) {
    const int64_t m = blockIdx.y;
    const double sc = input_scale<S>(amax[m]);
    if (blockIdx.x == 0 && threadIdx.x == 0) unscale[m] = 1.0 / sc;
    if (sc == 1.0) return;
    dst += m * np * np;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np * np; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = scale_pow2(dst[i], sc);
}

template <typename S>
cudaError_t copy_in_pad(const S *src, int64_t n, int64_t lda, int64_t src_bstride, S *dst,
                        int64_t np, int64_t batch, int *nonfinite_flag, cudaStream_t st,
                        unsigned long long *amax, double *unscale) {
    dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(np, 2368 / batch)), (unsigned)batch);
    if (amax) {
        // one pass: unscaled copy + max |a|; then the (usually empty) rescale
        cudaError_t e = cudaMemsetAsync(amax, 0, (size_t)batch * sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
        k_copy_in_pad<S><<<grid, 256, 0, st>>>(src, n, lda, src_bstride, dst, np, nonfinite_flag, nullptr,
                                               nullptr, amax);
        bsvd_host::count_launch();
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        k_rescale<S><<<grid, 256, 0, st>>>(dst, np, amax, unscale);
        bsvd_host::count_launch();
        return cudaGetLastError();
    }
    k_copy_in_pad<S><<<grid, 256, 0, st>>>(src, n, lda, src_bstride, dst, np, nonfinite_flag, nullptr, unscale,
                                           nullptr);
    bsvd_host::count_launch();
    return cudaGetLastError();
}

// values *= unscale[matrix] (exact powers of two): undo the input normalisation
template <typename C>
__global__ void k_unscale_values(C *__restrict__ v, int64_t n, int64_t stride, const double *__restrict__ unscale) {
    const int64_t m = blockIdx.y;
    const double u = unscale[m];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[m * stride + i] = (C)((double)v[m * stride + i] * u);
}
template <typename C>
cudaError_t unscale_values(C *v, int64_t n, int64_t stride, int64_t batch, const double *unscale, cudaStream_t st) {
    dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)batch);
    k_unscale_values<C><<<grid, 256, 0, st>>>(v, n, stride, unscale);
    bsvd_host::count_launch();
    return cudaGetLastError();
}
template cudaError_t unscale_values<double>(double *, int64_t, int64_t, int64_t, const double *, cudaStream_t);
template cudaError_t unscale_values<float>(float *, int64_t, int64_t, int64_t, const double *, cudaStream_t);

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
                                        int64_t, int *, cudaStream_t, unsigned long long *,      \
                                        double *);                                               \
    template cudaError_t clear_outside_band<S>(S *, int64_t, int, int64_t, cudaStream_t);
INST(double)
INST(float)
INST(__half)
#undef INST

}  // namespace bsvd
