// Standalone check of the tcgen05 tf32 toolkit: D = C0 - A * B^T (3xTF32),
// M = 128, N = 128, K = 128.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2508_06339_b200/csrc/tc_sm100.cuh"
using namespace bsvd;

constexpr int M = 128, N = 64, K = 128;

__global__ void __launch_bounds__(128) k_test(const float *A, const float *B, const float *C0, float *D) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    float *sm = (float *)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
    float *Ahi = sm, *Alo = Ahi + M * K, *Bhi = Alo + M * K, *Blo = Bhi + N * K;
    __shared__ uint64_t mbar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tc::tmem_alloc<128>(&tslot);
    if (tid == 0) tc::mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tb = tslot;
    // images: K-block stride = rows * 32 floats
    for (int idx = tid; idx < M * K; idx += 128) {
        const int m = idx / K, k = idx % K;
        float h, l;
        tc::split3(A[m * K + k], h, l);
        Ahi[tc::img_off(m, k, M * 32)] = h;
        Alo[tc::img_off(m, k, M * 32)] = l;
    }
    for (int idx = tid; idx < N * K; idx += 128) {
        const int nn = idx / K, k = idx % K;
        float h, l;
        tc::split3(B[nn * K + k], h, l);
        Bhi[tc::img_off(nn, k, N * 32)] = h;
        Blo[tc::img_off(nn, k, N * 32)] = l;
    }
    // accumulator init: D row m = thread m, columns 0..N-1
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
        for (int kb = 0; kb < K / 32; ++kb)
            tc::mma3_kblock<M, N, true>(tb, tc::smem_u32(Ahi + kb * M * 32), tc::smem_u32(Alo + kb * M * 32),
                                        tc::smem_u32(Bhi + kb * N * 32), tc::smem_u32(Blo + kb * N * 32), true);
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
    if (warp == 0) tc::tmem_free<128>(tb);
}

int main() {
    std::vector<float> A(M * K), B(N * K), C0(M * N), D(M * N);
    srand(1);
    for (auto &x : A) x = (float)rand() / RAND_MAX - 0.5f;
    for (auto &x : B) x = (float)rand() / RAND_MAX - 0.5f;
    for (auto &x : C0) x = (float)rand() / RAND_MAX - 0.5f;
    float *dA, *dB, *dC, *dD;
    cudaMalloc(&dA, 4 * M * K); cudaMalloc(&dB, 4 * N * K); cudaMalloc(&dC, 4 * M * N); cudaMalloc(&dD, 4 * M * N);
    cudaMemcpy(dA, A.data(), 4 * M * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), 4 * N * K, cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C0.data(), 4 * M * N, cudaMemcpyHostToDevice);
    const int smem = (2 * M * K + 2 * N * K) * 4 + 1024;
    cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_test<<<1, 128, smem>>>(dA, dB, dC, dD);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    cudaMemcpy(D.data(), dD, 4 * M * N, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int nn = 0; nn < N; ++nn) {
            double s = C0[m * N + nn];
            for (int k = 0; k < K; ++k) s -= (double)A[m * K + k] * B[nn * K + k];
            double err = fabs(s - D[m * N + nn]);
            if (err > maxerr) maxerr = err;
            if (fabs(s) > maxref) maxref = fabs(s);
            if (err > 1e-3 && bad++ < 5) printf("  m=%d n=%d ref=%g got=%g\n", m, nn, s, D[m * N + nn]);
        }
    printf("max abs err %.3e (max |ref| %.3e) bad=%d\n", maxerr, maxref, bad);
    return 0;
}
