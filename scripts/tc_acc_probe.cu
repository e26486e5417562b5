// Probe of the kind::tf32 accumulation rounding on sm_100a (development aid).
// D[128 x 64] = C0 + A[128 x K] * B[64 x K]^T with tf32-exact inputs, K = 8
// (one MMA) or K = 128 (16 MMAs); compared with fp64 on the host.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2508_06339_b200/csrc/tc_sm100.cuh"  // build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 scripts/tc_acc_probe.cu
using namespace bsvd;
constexpr int M = 128, N = 64, KMAX = 128;

__global__ void __launch_bounds__(128) k_probe(const float *A, const float *B, const float *C0, float *D, int K, int three, int R) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    float *sm = (float *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    float *As = sm, *Bs = As + M * KMAX, *Al = Bs + N * KMAX, *Bl = Al + M * KMAX;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tc::tmem_alloc<64>(&tslot);
    if (tid == 0) tc::mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tb = tslot;
    for (int idx = tid; idx < M * KMAX; idx += 128) {
        const int m = idx / KMAX, k = idx % KMAX;
        float h = 0.f, l = 0.f;
        if (k < K) { if (three) tc::split3(A[m * KMAX + k], h, l); else h = A[m * KMAX + k]; }
        As[tc::img_off(m, k, M * 32)] = h;
        Al[tc::img_off(m, k, M * 32)] = l;
    }
    for (int idx = tid; idx < N * KMAX; idx += 128) {
        const int nn = idx / KMAX, k = idx % KMAX;
        float h = 0.f, l = 0.f;
        if (k < K) { if (three) tc::split3(B[nn * KMAX + k], h, l); else h = B[nn * KMAX + k]; }
        Bs[tc::img_off(nn, k, N * 32)] = h;
        Bl[tc::img_off(nn, k, N * 32)] = l;
    }
    const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        for (int j = 0; j < 16; ++j) v[j] = C0[tid * N + c0 + j];
        tc::tmem_st16(tb + lane_base + c0, v);
    }
    tc::tmem_st_wait();
    tc::fence_async_smem();
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
        tc::fence_after();
        constexpr uint32_t id = tc::idesc_tf32<M, N, false>();
        for (int rep = 0; rep < R; ++rep)
        for (int k8 = 0; k8 < K / 8; ++k8) {
            const int kb = k8 / 4, kk = k8 % 4;
            tc::mma_tf32(tb, tc::sdesc(tc::smem_u32(As + kb * M * 32) + 32u * kk),
                         tc::sdesc(tc::smem_u32(Bs + kb * N * 32) + 32u * kk), id, true);
            if (three) {
                tc::mma_tf32(tb, tc::sdesc(tc::smem_u32(As + kb * M * 32) + 32u * kk),
                             tc::sdesc(tc::smem_u32(Bl + kb * N * 32) + 32u * kk), id, true);
                tc::mma_tf32(tb, tc::sdesc(tc::smem_u32(Al + kb * M * 32) + 32u * kk),
                             tc::sdesc(tc::smem_u32(Bs + kb * N * 32) + 32u * kk), id, true);
            }
        }
        tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tc::tmem_ld16(tb + lane_base + c0, v);
        for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = v[j];
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_free<64>(tb);
}

static float tf32_trunc(float x) { unsigned u; memcpy(&u, &x, 4); u &= 0xffffe000u; float r; memcpy(&r, &u, 4); return r; }
static float rz(double x) {   // round toward zero to fp32
    float f = (float)x;
    if (fabs((double)f) > fabs(x)) f = nextafterf(f, 0.f);
    return f;
}
int main() {
    srand(1);
    auto rnd = [] { return (float)((rand() / (double)RAND_MAX) * 2 - 1); };
    std::vector<float> A(M * KMAX), B(N * KMAX), C0(M * N), D(M * N);
    float *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C0.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * (M + N) * KMAX * 4 + 1024);
    for (int R : {1, 4, 16, 64})
    for (int three : {1})
    for (int K : {128}) {
        for (int withc : {0}) {
            for (auto &x : A) x = three ? rnd() : tf32_trunc(rnd());
            for (auto &x : B) x = three ? rnd() : tf32_trunc(rnd());
            for (auto &x : C0) x = withc ? rnd() * 4 : 0.f;
            cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(dC, C0.data(), C0.size() * 4, cudaMemcpyHostToDevice);
            k_probe<<<1, 128, 2 * (M + N) * KMAX * 4 + 1024>>>(dA, dB, dC, dD, K, three, R);
            cudaError_t e = cudaDeviceSynchronize();
            if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
            int n_rn = 0, n_rz = 0, n_other = 0;
            double bias = 0, rms = 0, maxe = 0;
            // also a serial fp32 RN reference (k order) for comparison
            double bias_ser = 0, rms_ser = 0;
            for (int m = 0; m < M; ++m)
                for (int nn = 0; nn < N; ++nn) {
                    double ex = C0[m * N + nn];
                    float ser = C0[m * N + nn];
                    double mag = fabs(ex);
                    for (int k = 0; k < K; ++k) {
                        ex += (double)A[m * KMAX + k] * B[nn * KMAX + k];
                        ser = fmaf(A[m * KMAX + k], B[nn * KMAX + k], ser);
                        mag += fabs((double)A[m * KMAX + k] * B[nn * KMAX + k]);
                    }
                    ex *= R; mag *= R;
                    const float g = D[m * N + nn];
                    if (g == (float)ex) ++n_rn;
                    else if (g == rz(ex)) ++n_rz;
                    else ++n_other;
                    const double err = (g - ex) / mag, es = (ser - ex) / mag;
                    bias += err; rms += err * err; maxe = fmax(maxe, fabs(err));
                    bias_ser += es; rms_ser += es * es;
                }
            const double cnt = M * N;
            printf("R=%d 3x=%d K=%3d C0=%d: RN %5d RZ %5d other %5d | err/sum|ab|: mean %+.3e rms %.3e max %.3e | serial fp32 fma: mean %+.3e rms %.3e\n",
                   R, three, K, withc, n_rn, n_rz, n_other, bias / cnt, sqrt(rms / cnt), maxe, bias_ser / cnt, sqrt(rms_ser / cnt));
        }
    }
    return 0;
}
