// Cycles per step of one Sturm pass with a Laguerre triple (p, p', p'') at x
// plus K extra count chains, continuant form (development aid).  256 warps
// over the GPU like k_values at n = 8192.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ double cstep(double x, double p, double o, double pm) {
    return fma(p, 0x1p-300, fma(-x, p, -o * pm));
}
__device__ __forceinline__ double pow2_norm(double v) {
    return __hiloint2double(0x7fe00000 - (__double2hiint(v) & 0x7ff00000), 0);
}

template <int K, bool LAG>
__global__ void k(const double* o2, int m, double x0, long long* cyc, int* out, double* gout) {
    const double x = x0 + threadIdx.x * 1e-3;
    double xs[K > 0 ? K : 1], qm[K > 0 ? K : 1], q[K > 0 ? K : 1];
    int c[K > 0 ? K : 1];
#pragma unroll
    for (int i = 0; i < K; ++i) { xs[i] = x + (i + 1) * 1e-9; qm[i] = 1.0; q[i] = -xs[i]; c[i] = 0; }
    double pm = 1.0, p = -x, dpm = 0.0, dp = -1.0, ddpm = 0.0, ddp = 0.0;
    int cnt = 0;
    long long t0 = clock64();
    for (int j = 0; j + 8 <= m; j += 8) {
        double o[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) o[u] = __ldg(o2 + j + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (LAG) {
                const double pn = cstep(x, p, o[u], pm);
                const double dpn = fma(-x, dp, fma(-o[u], dpm, -p));
                const double ddpn = fma(-x, ddp, fma(-o[u], ddpm, -2.0 * dp));
                cnt += (pn < 0.0) != (p < 0.0);
                pm = p; p = pn; dpm = dp; dp = dpn; ddpm = ddp; ddp = ddpn;
            }
#pragma unroll
            for (int i = 0; i < K; ++i) {
                const double qn = cstep(xs[i], q[i], o[u], qm[i]);
                c[i] += (qn < 0.0) != (q[i] < 0.0);
                qm[i] = q[i]; q[i] = qn;
            }
        }
        if (LAG) {
            const double s = pow2_norm(fmax(fabs(pm), fabs(p)));
            pm *= s; p *= s; dpm *= s; dp *= s; ddpm *= s; ddp *= s;
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const double s = pow2_norm(fmax(fabs(qm[i]), fabs(q[i])));
            qm[i] *= s; q[i] *= s;
        }
    }
    long long t1 = clock64();
    int tot = cnt;
#pragma unroll
    for (int i = 0; i < K; ++i) tot += c[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
    gout[blockIdx.x * blockDim.x + threadIdx.x] = dp / p + ddp;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int K, bool LAG>
void run(const double* o2, int m, long long* cyc, int* out, double* g, int blocks, int thr) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<K, LAG><<<blocks, thr>>>(o2, m, 0.7, cyc, out, g); cudaDeviceSynchronize();
    cudaEventRecord(e0); k<K, LAG><<<blocks, thr>>>(o2, m, 0.7, cyc, out, g); cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("blocks %4d thr %3d  lag %d  K %2d   %7.1f cyc/step  %7.3f ms/pass\n", blocks, thr, (int)LAG, K,
           double(c) / m, ms);
}

int main() {
    const int m = 16383;
    double* h = new double[m];
    for (int i = 0; i < m; ++i) h[i] = 0.5 + (i % 7) * 0.3;
    double* o2; long long* cyc; int* out; double* g;
    cudaMalloc(&o2, m * 8); cudaMalloc(&cyc, 8); cudaMalloc(&out, 4 * 65536); cudaMalloc(&g, 8 * 65536);
    cudaMemcpy(o2, h, m * 8, cudaMemcpyHostToDevice);
    for (int cfg = 0; cfg < 3; ++cfg) {
        const int blocks = cfg == 0 ? 256 : (cfg == 1 ? 128 : 512), thr = cfg == 1 ? 64 : 32;
        run<1, false>(o2, m, cyc, out, g, blocks, thr);
        run<2, false>(o2, m, cyc, out, g, blocks, thr);
        run<4, false>(o2, m, cyc, out, g, blocks, thr);
        run<8, false>(o2, m, cyc, out, g, blocks, thr);
        run<0, true>(o2, m, cyc, out, g, blocks, thr);
        run<2, true>(o2, m, cyc, out, g, blocks, thr);
        run<4, true>(o2, m, cyc, out, g, blocks, thr);
        run<6, true>(o2, m, cyc, out, g, blocks, thr);
    }
    return 0;
}
