// common.cuh -- shared device/host helpers for libbsvd (sm_100a only).
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <utility>

#include "../../include/bsvd.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libbsvd is built for sm_100a (B200) only"
#endif

namespace bsvd {

// Raise a kernel's dynamic shared-memory limit on the CURRENT device.  Function
// attributes are per device (context), so the largest size set is remembered
// per (kernel, device); thread-safe.
inline cudaError_t ensure_smem_fn(const void *fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, size_t> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t &have = done[{fn, dev}];
    if (bytes <= have) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}
template <typename F>
inline cudaError_t ensure_smem(F *fn, size_t bytes) {
    return ensure_smem_fn(reinterpret_cast<const void *>(fn), bytes);
}

// Storage <-> compute conversion.  FP16 is storage-only (precision.py:16-37):
// loads widen exactly, stores round to nearest even like numpy's cast.
template <typename S, typename C> struct Conv;
template <> struct Conv<double, double> {
    __device__ __forceinline__ static double ld(double v) { return v; }
    __device__ __forceinline__ static double st(double v) { return v; }
};
template <> struct Conv<float, float> {
    __device__ __forceinline__ static float ld(float v) { return v; }
    __device__ __forceinline__ static float st(float v) { return v; }
};
template <> struct Conv<__half, float> {
    __device__ __forceinline__ static float ld(__half v) { return __half2float(v); }
    __device__ __forceinline__ static __half st(float v) { return __float2half_rn(v); }
};

__device__ __forceinline__ double to_f64(double v) { return v; }
__device__ __forceinline__ double to_f64(float v) { return (double)v; }
__device__ __forceinline__ double to_f64(__half v) { return (double)__half2float(v); }

template <typename C> struct Eps;
template <> struct Eps<double> { static constexpr double v = 2.220446049250313e-16; };
template <> struct Eps<float> { static constexpr float v = 1.1920928955078125e-07f; };

// Strided view element (matrix.py:93-154): (i, j) -> p[i*rs + j*cs].
template <typename T>
__device__ __forceinline__ T &at(T *p, int64_t i, int64_t j, int64_t rs, int64_t cs) {
    return p[i * rs + j * cs];
}

__device__ __forceinline__ double dsqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float dsqrt(float x) { return sqrtf(x); }

// Reference reflector scalars (kernels.py:96-116): x, tau-hat, rho'.  The
// absolute |x| < 10 eps guard is reproduced verbatim.
template <typename C>
__device__ __forceinline__ void reflector_scalars(C piv, C sigma, C aik, C rho, C eps10, C two,
                                                  C &x, C &tau, C &rhop) {
    const C zero = eps10 - eps10;
    if (piv < zero)
        x = piv - dsqrt(piv * piv + sigma);
    else
        x = piv + dsqrt(piv * piv + sigma);
    if ((x < zero ? -x : x) < eps10) {
        x = eps10;
        tau = two;
        rhop = two * (aik + rho / x);
    } else {
        tau = two * x * x / (x * x + sigma);
        rhop = (tau / x) * (aik * x + rho);
    }
}

}  // namespace bsvd

// Host-side error plumbing (capi.cu owns the thread-local message) and the
// process-wide count of kernels this library has launched (bench evidence).
namespace bsvd_host {
void count_launch(unsigned n = 1);
bsvd_status set_error(bsvd_status st, const char *fmt, ...);
bsvd_status cuda_error(cudaError_t e, const char *where);
}  // namespace bsvd_host

#define BSVD_CUDA_TRY(expr)                                                  \
    do {                                                                     \
        cudaError_t e__ = (expr);                                            \
        if (e__ != cudaSuccess) return bsvd_host::cuda_error(e__, #expr);    \
    } while (0)

#define BSVD_LAUNCH_CHECK(where)                                             \
    do {                                                                     \
        cudaError_t e__ = cudaGetLastError();                                \
        if (e__ != cudaSuccess) return bsvd_host::cuda_error(e__, where);    \
    } while (0)
