// Microbenchmark of the on-chip blocked node QR (panel_blocked.cuh): cycles
// per leaf / TT factorisation of a 128 x 128 fp32 tile, FULL_T off (the
// panel's critical path).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdlib>
#include <vector>
#define BSVD_STAMP_CLOCK 1
#define BSVD_QR_PROBE 1
#include "../paper_2508_06339_b200/csrc/common.cuh"
namespace bsvd {
constexpr int kNT = 256;
template <typename C>
__device__ __forceinline__ void house_scalars(C alpha, C sig, C &beta, C &tau, C &scale) {
    if (sig == C(0)) { beta = alpha; tau = C(0); scale = C(1); }
    else { beta = -copysign(dsqrt(alpha * alpha + sig), alpha); tau = (beta - alpha) / beta; scale = C(1) / (alpha - beta); }
}
// fp32: one correctly rounded sqrt and two correctly rounded reciprocals in
// place of two IEEE divisions (shorter dependent chain in the panel's column
// step; tau and scale stay within an ulp or two).
__device__ __forceinline__ void house_scalars(float alpha, float sig, float &beta, float &tau, float &scale) {
    if (sig == 0.f) {
        beta = alpha;
        tau = 0.f;
        scale = 1.f;
    } else {
        beta = -copysignf(__fsqrt_rn(fmaf(alpha, alpha, sig)), alpha);
        const float d = alpha - beta;
        scale = __frcp_rn(d);
        tau = -d * __frcp_rn(beta);
    }
}

}
#include "../paper_2508_06339_b200/csrc/panel_qr.cuh"
#include "../paper_2508_06339_b200/csrc/panel_blocked.cuh"
using namespace bsvd;

constexpr int TS = 128, NTP = 512;
constexpr int LDL = TS + 1, LDT = 2 * TS + 1;
constexpr int AUX = blk::aux_elems<float, TS>();

template <bool TT>
__global__ void __launch_bounds__(NTP, 1) k_bench(const float *src, float *dst, long long *cyc, int reps, unsigned long long *st) {
    extern __shared__ float sm[];
    constexpr int lda = TT ? LDT : LDL;
    float *A = sm, *aux = A + TS * lda, *tau = aux + AUX;
    auto house = [](float a, float s, float &b, float &t, float &sc) { house_scalars(a, s, b, t, sc); };
    long long tot = 0;
    for (int rep = 0; rep < reps; ++rep) {
        for (int idx = threadIdx.x; idx < TS * TS; idx += NTP) {
            const int c = idx / TS, r = idx % TS;
            if (TT) {
                A[c * lda + r] = r <= c ? src[idx] : 0.f;
                A[c * lda + TS + r] = r <= c ? src[TS * TS + idx] : 0.f;
            } else {
                A[c * lda + r] = src[idx];
            }
        }
        __syncthreads();
        long long t0 = clock64();
        blk::qr_blocked<float, TS, TT, NTP, false>(A, lda, tau, A, lda, aux, house, [&](int) {}, rep == reps - 1 ? st : nullptr);
        if (rep == reps - 1 && threadIdx.x == 0) st[255] = t0;
        __syncthreads();
        tot += clock64() - t0;
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = tot / reps;
    for (int idx = threadIdx.x; idx < TS * TS; idx += NTP) dst[idx] = A[(idx / TS) * lda + idx % TS];
}

int main() {
    std::vector<float> h(2 * TS * TS);
    srand(3);
    for (auto &x : h) x = (float)rand() / RAND_MAX - 0.5f;
    float *src, *dst;
    long long *cyc;
    cudaMalloc(&src, h.size() * 4); cudaMalloc(&dst, TS * TS * 4); cudaMalloc(&cyc, 8 * 64);
    cudaMemcpy(src, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    unsigned long long *st;
    cudaMalloc(&st, 256 * 8);
    for (int tt = 0; tt < 2; ++tt) {
        const size_t smem = ((tt ? TS * LDT : TS * LDL) + AUX + TS + 8) * 4;
        auto kern = tt ? k_bench<true> : k_bench<false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaMemset(st, 0, 256 * 8);
        kern<<<1, NTP, smem>>>(src, dst, cyc, 5, st);
        cudaError_t e = cudaDeviceSynchronize();
        long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%s: %s  %lld cycles = %.1f us @1.965GHz\n", tt ? "TT  " : "leaf", cudaGetErrorString(e), c, c / 1965.0);
        unsigned long long hs[256];
        cudaMemcpy(hs, st, 256 * 8, cudaMemcpyDeviceToHost);
        unsigned long long prev = hs[255];
        for (int sp = 0; sp < 4; ++sp) {
            const unsigned long long f = hs[128 + 4 * sp], t = hs[128 + 4 * sp + 1], u = hs[128 + 4 * sp + 2];
            printf("  subpanel %d: factor %llu (%.0f/col)  T %llu  update %llu\n", sp, f - prev, (f - prev) / 32.0, t - f, u - t);
            prev = u;
        }
        printf("  step probe (thread 64, kl=5):");
        for (int k = 1; k < 7; ++k) printf(" %llu", hs[200 + k] - hs[200 + k - 1]);
        printf("  | next step start +%llu\n", hs[6] - hs[200]);
    }
    return 0;
}
