// Latency per Sturm step of count-recurrence variants (development aid):
// one warp, m steps, cycles per step from clock64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double sdiv(double o, double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    r = r * fma(-q, r, 2.0);
    const double y = o * r;
    return fma(fma(-q, y, o), r, y);
}
__device__ __forceinline__ double nz_fix(double pn, double p) {
    return pn == 0.0 ? copysign(fmax(fabs(p) * 0x1p-100, 0x1p-1074), p) : pn;
}
__device__ __forceinline__ double pow2_norm(double v) {
    return __hiloint2double(0x7fe00000 - (__double2hiint(v) & 0x7ff00000), 0);
}

template <int V>
__global__ void k(const double* o2, int m, double x0, long long* cyc, int* out) {
    const double x = x0 + threadIdx.x * 1e-3;
    int cnt = 0;
    long long t0 = clock64();
    if (V == 0) {   // ratio
        double q = -x;
        for (int j = 0; j < m; ++j) {
            q = -x - sdiv(__ldg(o2 + j), q);
            if (fabs(q) < 0x1p-1000) q = (q < 0.0) ? -0x1p-1000 : 0x1p-1000;
            cnt += q < 0.0;
        }
    } else {
        double pm = 1.0, p = -x;
        int j = 0;
        for (; j + 8 <= m; j += 8) {
            double o[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) o[u] = __ldg(o2 + j + u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                double pn = fma(-x, p, -o[u] * pm);
                if (V == 1) pn = nz_fix(pn, p);
                if (V == 3) pn = fma(p, 0x1p-300, pn);
                cnt += (pn < 0.0) != (p < 0.0);
                pm = p; p = pn;
            }
            if (V != 4) {
                const double s = pow2_norm(fmax(fabs(pm), fabs(p)));
                pm *= s; p *= s;
            }
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = cnt;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    const int m = 16383;
    double* h = new double[m];
    for (int i = 0; i < m; ++i) h[i] = 0.5 + (i % 7) * 0.3;
    double* o2; long long* cyc; int* out;
    cudaMalloc(&o2, m * 8); cudaMalloc(&cyc, 8); cudaMalloc(&out, 4 * 148 * 1024);
    cudaMemcpy(o2, h, m * 8, cudaMemcpyHostToDevice);
    const char* names[] = {"ratio", "cont+nzfix", "cont raw", "cont+fmafix", "cont no-rescale"};
    for (int blocks : {1, 148, 296, 592}) for (int thr : {32, 128}) for (int v = 0; v < 5; ++v) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        auto launch = [&] {
            switch (v) { case 0: k<0><<<blocks, thr>>>(o2, m, 0.7, cyc, out); break;
                         case 1: k<1><<<blocks, thr>>>(o2, m, 0.7, cyc, out); break;
                         case 2: k<2><<<blocks, thr>>>(o2, m, 0.7, cyc, out); break;
                         case 3: k<3><<<blocks, thr>>>(o2, m, 0.7, cyc, out); break;
                         default: k<4><<<blocks, thr>>>(o2, m, 0.7, cyc, out); }
        };
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("blocks %4d thr %4d %-16s %7.1f cyc/step  %8.3f ms  (%.1f ns/step)\n", blocks, thr, names[v],
               double(c) / m, ms, ms * 1e6 / m);
    }
    return 0;
}
