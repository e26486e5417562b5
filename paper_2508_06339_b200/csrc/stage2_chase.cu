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
#include <stdio.h>
#include <stdlib.h>

#include <vector>

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

// Cluster helpers (CS CTAs of one thread-block cluster cooperate on an op).
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
template <int CS>
__device__ __forceinline__ void cluster_sync() {
    if constexpr (CS > 1) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                     "barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
        __syncthreads();
    }
}

// Householder generation (LAPACK dlarfg convention): x -> beta e1 with
// H = I - tau v v^T, v[0] = 1.  Executed by warp 0 of every CTA of the
// cluster (identical arithmetic -> identical v); v (len L) into vs.
__device__ __forceinline__ void pivot_load(const Band &A, int64_t r0, int64_t c0, bool column, int L,
                                           double (&x4)[4], double &alpha) {
    const int lane = threadIdx.x & 31;
    alpha = __ldcg(A.at(r0, c0));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = 1 + lane + 32 * q;
        x4[q] = j < L ? (column ? __ldcg(A.at(r0 + j, c0)) : __ldcg(A.at(r0, c0 + j))) : 0.0;
    }
}

__device__ __forceinline__ void pivot_finish(const double (&x4)[4], double alpha, int L, double *vs,
                                             double *tau_s, double *beta_s) {
    const int lane = threadIdx.x & 31;
    double sig = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = 1 + lane + 32 * q;
        if (j < L) vs[j] = x4[q];
        sig += x4[q] * x4[q];
    }
    sig = warp_sum(sig);
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (sig != 0.0) {
        beta = -copysign(sqrt(alpha * alpha + sig), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
    }
    __syncwarp();
    for (int j = 1 + lane; j < L; j += 32) vs[j] *= scale;
    if (lane == 0) {
        vs[0] = 1.0;
        *tau_s = tau;
        *beta_s = beta;
    }
}

__device__ void write_pivot(const Band &A, int64_t r0, int64_t c0, bool column, int L, double beta) {
    const int lane = threadIdx.x & 31;
    for (int j = 1 + lane; j < L; j += 32) {
        if (column) __stcg(A.at(r0 + j, c0), 0.0); else __stcg(A.at(r0, c0 + j), 0.0);
    }
    if (lane == 0) __stcg(A.at(r0, c0), beta);
}

// Left op slice: pivot column p (rows [p, p+L), L <= 128), this CTA's
// columns [ca, cb) (<= 64).  Register tile: warp w owns columns w, w+8, ...;
// lane l holds rows l, l+32, l+64, l+96 of each.  The slice's loads are
// issued BEFORE mid() (reflector formation + cluster barrier) so the two L2
// round trips overlap; mid() must be reached by every thread.
template <int CPW, int NW, typename Mid>
__device__ __forceinline__ void left_slice(const Band &A, int64_t p, int L, int64_t ca, int64_t cb,
                                           const double *vs, const double *tau_s, Mid mid) {
    const int ncol = cb > ca ? (int)(cb - ca) : 0;      // <= NW * CPW
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double x[CPW][4];
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
        const int c = warp + NW * k;
        const double *col = (c < ncol) ? A.at(p, ca + c) : nullptr;   // rows contiguous
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = lane + 32 * q;
            x[k][q] = (col && r < L) ? __ldcg(col + r) : 0.0;
        }
    }
    mid();
    const double tau = *tau_s;
    if (tau == 0.0 || ncol == 0) return;
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = (lane + 32 * q < L) ? vs[lane + 32 * q] : 0.0;
    double w[CPW];
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
        w[k] = 0.0;
#pragma unroll
        for (int q = 0; q < 4; ++q) w[k] += v[q] * x[k][q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < CPW; ++k) w[k] += __shfl_xor_sync(0xffffffffu, w[k], o);
#pragma unroll
    for (int k = 0; k < CPW; ++k) {
        const int c = warp + NW * k;
        if (c >= ncol) continue;
        double *col = A.at(p, ca + c);
        const double tw = tau * w[k];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = lane + 32 * q;
            if (r < L) __stcg(col + r, x[k][q] - tw * v[q]);
        }
    }
}

// Right op slice: pivot row p, columns [c0, c0+L) (L <= 128), this CTA's
// rows [ra, rb) (<= 64).  Register tile: lanes <-> 32 consecutive rows
// (coalesced column segments), warp w = (row half, column phase q of 4);
// each thread holds columns q, q+4, ... of its row (<= 32 values); the four
// column-phase partial dots are combined through shared memory.
template <int NH, int NW, typename Mid>
__device__ __forceinline__ void right_slice(const Band &A, int64_t p, int64_t c0, int L, int64_t ra,
                                            int64_t rb, const double *vs, const double *tau_s,
                                            double *part, Mid mid) {
    const int nrow = rb > ra ? (int)(rb - ra) : 0;      // <= 32 * NH
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int PH = NW / NH;                         // column phases
    const int half = warp % NH, q = warp / NH;
    const int r = half * 32 + lane;
    const bool act = r < nrow;
    constexpr int JPT = 128 / PH;                       // columns per thread
    double x[JPT];
    const int64_t cstride = A.ld - 1;                   // (r, c+1) - (r, c)
    const double *base = act ? A.at(ra + r, c0) : nullptr;
#pragma unroll
    for (int k = 0; k < JPT; ++k) {
        const int j = q + PH * k;
        x[k] = (act && j < L) ? __ldcg(base + (int64_t)j * cstride) : 0.0;
    }
    mid();
    const double tau = *tau_s;
    if (tau == 0.0 || nrow == 0) return;                // uniform within the CTA
    double w = 0.0;
#pragma unroll
    for (int k = 0; k < JPT; ++k) {
        const int j = q + PH * k;
        if (j < L) w += x[k] * vs[j];
    }
    part[q * (32 * NH) + r] = w;
    __syncthreads();
    double ws = 0.0;
#pragma unroll
    for (int g = 0; g < PH; ++g) ws += part[g * (32 * NH) + r];
    const double tw = tau * ws;
    if (act && ra + r != p) {
        double *rowp = A.at(ra + r, c0);
#pragma unroll
        for (int k = 0; k < JPT; ++k) {
            const int j = q + PH * k;
            if (j < L) __stcg(rowp + (int64_t)j * cstride, x[k] - tw * vs[j]);
        }
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// One op (index i) of sweep s.  All CTAs of the cluster call this with the
// same arguments; rank `rk` of CS owns a contiguous slice of the op.
template <int CS, int NW = 8>
__device__ void chase_op(const Band &A, int64_t s, int i, int64_t n, int b, unsigned rk,
                         double *vs, double *tau_s, double *beta_s, double *part,
                         unsigned long long *tr) {
    bool column;
    int64_t p, c0, lo, hi;   // pivot row/col, first column, apply range [lo, hi)
    int L;
    if (i == 0) {                       // right op: annihilate row s
        column = false; p = s; c0 = s + 1;
        L = (int)(min(s + 1 + b, n) - c0);
        lo = s; hi = min(s + 1 + b, n);
    } else {
        const int64_t t = (i - 1) / 2;
        const int64_t r0 = s + 1 + t * b;
        if (((i - 1) & 1) == 0) {       // left op: annihilate column r0
            column = true; p = r0; c0 = r0;
            L = (int)(min(r0 + b, n) - r0);
            lo = r0 + 1; hi = min(r0 + 2 * b, n);
        } else {                        // right op: annihilate row r0's fill
            column = false; p = r0; c0 = r0 + b;
            L = (int)(min(r0 + 2 * b, n) - c0);
            lo = r0; hi = min(r0 + 2 * b, n);
        }
    }
    if (L < 2) return;                  // uniform across the cluster
    const int64_t tot = hi - lo;
    const int64_t chunk = (tot + CS - 1) / CS;
    const int64_t a = lo + (int64_t)rk * chunk, e = min(a + chunk, hi);
    double x4[4], alpha = 0.0;
    if ((threadIdx.x >> 5) == 0) pivot_load(A, p, c0, column, L, x4, alpha);   // first in the LSU queue
    auto mid = [&]() {
        if ((threadIdx.x >> 5) == 0) pivot_finish(x4, alpha, L, vs, tau_s, beta_s);
        __syncthreads();
        if (tr && threadIdx.x == 0) tr[2] = gtimer();
        cluster_sync<CS>();             // every CTA has read the pivot
        if (tr && threadIdx.x == 0) tr[3] = gtimer();
        if (rk == 0 && (threadIdx.x >> 5) == 0) write_pivot(A, p, c0, column, L, *beta_s);
    };
    // left slice <= NW*CPW columns, right slice <= 32*NH rows
    constexpr int CPW = NW == 16 ? 8 : (CS >= 8 ? 4 : 8);
    constexpr int NH = NW == 16 ? 4 : (CS >= 8 ? 1 : 2);
    if (column) left_slice<CPW, NW>(A, p, L, a, e, vs, tau_s, mid);
    else right_slice<NH, NW>(A, p, c0, L, a, e, vs, tau_s, part, mid);
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[4] = gtimer();
    if (threadIdx.x == 0) __threadfence();   // publish this CTA's slice gpu-wide
}

template <int CS>
__global__ void __launch_bounds__(256) k_chase(double *band, int64_t n, int b, int64_t ld,
                                               int64_t batch, int *progress, int64_t nitems,
                                               unsigned long long *trace) {
    __shared__ double vs[128];
    __shared__ double part[512];
    __shared__ double tau_s, beta_s;
    const unsigned rk = CS > 1 ? cluster_rank() : 0;
    const int64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
    for (int64_t w = cid; w < nitems; w += ncl) {
        const int64_t s = w / batch, m = w % batch;
        const Band A{band + m * n * ld, n, ld, b};
        int *prog = progress + m * n;
        const int nops = chase_nops(s, n, b);
        const int nprev = s > 0 ? chase_nops(s - 1, n, b) : 0;
        for (int i = 0; i < nops; ++i) {
            unsigned long long *tr =
                (trace && rk == 0 && m == 0 && s < 256 && i < 32) ? trace + (s * 32 + i) * 8 : nullptr;
            if (tr && threadIdx.x == 0) tr[0] = gtimer();
            if (s > 0) {
                if (threadIdx.x == 0) {
                    const int need = min(i + 4, nprev);
                    for (int spin = 0; ld_acquire(prog + s - 1) < need; ++spin)
                        if (spin > 64) __nanosleep(20);
                    __threadfence();
                }
                __syncthreads();
            }
            if (tr && threadIdx.x == 0) tr[1] = gtimer();
            chase_op<CS>(A, s, i, n, b, rk, vs, &tau_s, &beta_s, part, tr);
            cluster_sync<CS>();         // all slices of op i are written
            if (rk == 0 && threadIdx.x == 0) st_release(prog + s, i + 1);
            if (tr && threadIdx.x == 0) tr[5] = gtimer();
        }
    }
}

// Batched chase for narrow bands (b <= 64): one 16-warp CTA owns whole
// matrices and runs their sweeps back to back -- no inter-CTA progress
// flags; with thousands of matrices the GPU is full without pipelining.
__global__ void __launch_bounds__(512) k_chase_seq(double *band, int64_t n, int b, int64_t ld,
                                                   int64_t batch) {
    __shared__ double vs[128];
    __shared__ double part[512];
    __shared__ double tau_s, beta_s;
    for (int64_t m = blockIdx.x; m < batch; m += gridDim.x) {
        const Band A{band + m * n * ld, n, ld, b};
        for (int64_t s = 0; s + 2 < n; ++s) {
            const int nops = chase_nops(s, n, b);
            for (int i = 0; i < nops; ++i) {
                chase_op<1, 16>(A, s, i, n, b, 0, vs, &tau_s, &beta_s, part, nullptr);
                __syncthreads();
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
    if (n > 2 && b <= 64 && batch >= 512 && !getenv("BSVD_CHASE_PIPELINED")) {
        int dev = 0, nsm = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chase_seq, 512, 0);
        const int64_t grid = std::min<int64_t>(batch, (int64_t)nsm * std::max(per_sm, 1));
        k_chase_seq<<<(unsigned)grid, 512, 0, st>>>(band, n, b, ld, batch);
        bsvd_host::count_launch();
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
    } else if (n > 2) {
        // Cluster size: a single large band splits every op over 4 CTAs (4x
        // the L2 bandwidth per op); batches get their parallelism from the
        // matrices.  Shared slice: b x ceil(2b/CS) doubles.
        // Cluster size: every op is split over CS CTAs so each CTA's slice is
        // <= 64 columns (left op) or <= 64 rows (right op) of a register tile.
        int CS = b > 64 ? 8 : (b > 32 ? 2 : 1);
        if (const char *cs_env = getenv("BSVD_CHASE_CS")) CS = atoi(cs_env);
        if (CS < 8 && b > 64) CS = 4;               // slices must fit the register tiles
        const size_t smem = 0;
        int64_t nitems = (n - 2) * batch;   // sweeps 0..n-3 do work (reference loop bound)
        // useful concurrency: a sweep trails its predecessor by 4 ops
        int64_t nops0 = 1 + 2 * ((n - 2 + b) / b);
        int64_t want = std::min<int64_t>(nitems, batch * (nops0 / 4 + 2));
        cudaLaunchConfig_t lc{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CS;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        lc.blockDim = dim3(256);
        lc.dynamicSmemBytes = smem;
        lc.stream = st;
        lc.attrs = attr;
        lc.numAttrs = 1;
        void (*kern)(double *, int64_t, int, int64_t, int64_t, int *, int64_t, unsigned long long *) =
            CS == 8 ? k_chase<8> : (CS == 4 ? k_chase<4> : (CS == 2 ? k_chase<2> : k_chase<1>));
        if (CS > 1) {
            int max_clusters = 0;
            lc.gridDim = dim3((unsigned)(want * CS));
            err = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &lc);
            if (err != cudaSuccess) return err;
            want = std::min<int64_t>(want, std::max(max_clusters, 1));
        } else {
            int dev = 0, nsm = 0, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
            want = std::min<int64_t>(want, (int64_t)nsm * std::max(per_sm, 1));
        }
        lc.gridDim = dim3((unsigned)(want * CS));
        int64_t n_ = n, ld_ = ld, batch_ = batch;
        int b_ = b;
        // BSVD_CHASE_TRACE=<file>: per-op phase timestamps of the first
        // 256 sweeps (development instrumentation, off by default).
        const char *trace_path = getenv("BSVD_CHASE_TRACE");
        unsigned long long *trace = nullptr;
        const size_t trace_bytes = 256 * 32 * 8 * sizeof(unsigned long long);
        if (trace_path) {
            cudaMallocAsync((void **)&trace, trace_bytes, st);
            cudaMemsetAsync(trace, 0, trace_bytes, st);
        }
        err = cudaLaunchKernelEx(&lc, kern, band, n_, b_, ld_, batch_, progress, nitems, trace);
        bsvd_host::count_launch();
        if (err != cudaSuccess) return err;
        if (trace) {
            std::vector<unsigned long long> h(trace_bytes / 8);
            cudaMemcpyAsync(h.data(), trace, trace_bytes, cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            FILE *f = fopen(trace_path, "wb");
            if (f) { fwrite(h.data(), 1, trace_bytes, f); fclose(f); }
            cudaFreeAsync(trace, st);
        }
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
