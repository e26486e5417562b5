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
__device__ __forceinline__ void st_relaxed(int *p, int v) {   // after an explicit fence
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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
template <typename S, typename TB>
__global__ void k_pack_band(const S *__restrict__ a, int64_t n, int64_t lda, int64_t a_bstride,
                            int bw, TB *__restrict__ band, int64_t ld, int b) {
    const int64_t m = blockIdx.y;
    a += m * a_bstride;
    band += m * n * ld;
    const int64_t total = n * (int64_t)(bw + 1);
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = idx / (bw + 1);
        const int64_t r = c - bw + idx % (bw + 1);
        if (r < 0) continue;
        const TB v = (TB)to_f64(a[c * lda + r]);
        band[c * ld + (r - c + 2 * b)] = v;
    }
}

template <typename TB>
__global__ void k_extract_bidiag(const TB *__restrict__ band, int64_t n, int64_t ld, int b,
                                 double *__restrict__ d, double *__restrict__ e) {
    const int64_t m = blockIdx.y;
    band += m * n * ld;
    d += m * n;
    e += m * (n - 1);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        d[i] = (double)band[i * ld + 2 * b];
        if (i + 1 < n) e[i] = (double)band[(i + 1) * ld + (2 * b - 1)];
    }
}

// ---------------------------------------------------------------------------
// Chase v2 (64 < b <= 128): carried-block pipeline on a thread-block cluster.
//
// The footprint of every op is two b x b blocks, and consecutive ops of a
// sweep share one of them:
//   left op t  (r0 = s+1+t b):  D_t = [r0, r0+b) x [r0, r0+b)      (carried)
//                               E_t = [r0, r0+b) x [r0+b, r0+2b)   (loaded)
//   right op t:                 P_t = E_t                          (carried)
//                               Q_t = [r0+b, r0+2b) x [r0+b, r0+2b) (loaded)
//   and D_{t+1} = Q_t; op 0 (row s) loads Q_{-1} = [s+1, s+1+b)^2.
// Block k of a sweep (the block op k loads) lives in the REGISTERS of CTA
// k mod NC of the cluster for exactly two ops: op k (as the new block) and
// op k+1 (as the carried block, whose first column / row is op k+1's pivot),
// then it is stored.  Each op therefore needs one global block load (after
// the inter-sweep dependency) and no global pivot round trip: the carrier
// forms op k+1's pivot from its registers and ships the raw vector (1 KB)
// to the next block's CTA through distributed shared memory, signalled on
// an mbarrier; both CTAs form the identical reflector.  Dependency (checked
// by exhaustive footprint enumeration, scripts/chase_dep_check.py): block k
// of sweep s may be loaded once sweep s-1 has STORED blocks 0..k+2; stores
// are published in block order with a release counter per sweep.
namespace ch2 {
constexpr int NW = 16, NTH = 512, BK = 128;
// Tile shapes: a BKT x BKT block over BKT/8 warps, thread (w, l) holding rows
// l + 32a (a < BKT/32) and columns w + (BKT/8) q (q < 8).  BKT = 128 serves
// 64 < b <= 128; narrow bands use BKT = 64 / 32 (8 / 4 warps), so the
// reductions, barriers and loads of an op scale with the band, not with 128.
template <int BKT>
struct Shape {
    static constexpr int NW = BKT / 8, NTH = NW * 32, RA = BKT / 32;
};

__device__ __forceinline__ uint32_t saddr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}

__device__ __forceinline__ void arrive_remote(uint32_t a) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void wait_local(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W_%=;\n\t}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

// Edge mailbox (4-byte band elements): every published edge element is also
// written as one 64-bit word (tag << 32 | bits) with a relaxed gpu-scope store;
// the next sweep polls the words it needs until the tag matches -- the word is
// single-copy atomic, so the tag validates the value with no fence and no flag
// (the edge's old store -> fence -> flag -> poll -> load hand-off).
__device__ __forceinline__ void mbox_put(unsigned long long *p, uint32_t tag, float v) {
    const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long mbox_ld(const unsigned long long *p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}
__device__ __forceinline__ float mbox_get(const unsigned long long *p, uint32_t tag) {
    unsigned long long w;
    for (int spin = 0;; ++spin) {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
        if ((uint32_t)(w >> 32) == tag) break;
        if (spin > 64) __nanosleep(32);
    }
    return __uint_as_float((uint32_t)w);
}
constexpr int MBX_STRIDE = 128;   // words per (sweep parity, block) edge slot

template <typename T>
struct BandT {
    T *p;
    int64_t n, ld;
    int b;
    __device__ __forceinline__ T *at(int64_t r, int64_t c) const { return p + c * ld + (r - c + 2 * b); }
};

struct Blk {
    int64_t R0, C0;
    int nr, nc;
};
__device__ __forceinline__ Blk geom(int64_t s, int k, int64_t n, int b) {
    Blk g;
    if (k & 1) {
        g.R0 = s + 1 + (int64_t)((k - 1) >> 1) * b;
        g.C0 = g.R0 + b;
    } else {
        g.R0 = g.C0 = s + 1 + (int64_t)(k >> 1) * b;
    }
    g.nr = (int)max((int64_t)0, min((int64_t)b, n - g.R0));
    g.nc = (int)max((int64_t)0, min((int64_t)b, n - g.C0));
    return g;
}

// Householder scalars from the raw pivot vector p[0..L) (LAPACK dlarfg
// convention, v = (1, p[1:] * scale)).  Every warp of every CTA computes them
// from the same bytes in the same order (xor butterfly: identical in all
// lanes), so the reflector is bit-identical everywhere.
template <typename T>
__device__ __forceinline__ void reflector(const T *p, int L, T &tau, T &scale,
                                          T &beta) {
    const int lane = threadIdx.x & 31;
    T sg = T(0);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int j = lane + 32 * a;
        const T t = (j >= 1 && j < L) ? p[j] : T(0);
        sg = fma(t, t, sg);
    }
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) sg += __shfl_xor_sync(0xffffffffu, sg, o);
    const T alpha = p[0];
    tau = T(0);
    scale = T(0);
    beta = alpha;
    if (sg != T(0)) {
        // norm = sqrt(alpha^2 + sg) via one reciprocal square root (two Newton
        // steps on the hardware seed) instead of sqrt + two divisions:
        // beta = -sign(alpha) norm, tau = 1 + |alpha|/norm,
        // scale = 1/(alpha - beta) = sign(alpha)/(|alpha| + norm).
        const T s2 = fma(alpha, alpha, sg);
        const T aa = fabs(alpha);
        if constexpr (sizeof(T) == 8) {
            const T r = rsqrt(s2);
            const T nrm = s2 * r;
            beta = -copysign(nrm, alpha);
            tau = fma(aa, r, T(1));
            scale = copysign(T(1) / (aa + nrm), alpha);
        } else {
            // fp32: correctly rounded sqrt and divisions -- an inexact tau
            // (rsqrtf is 2 ulp) leaves H = I - tau v v^T slightly non-orthogonal,
            // and ~2 n^2 / b reflectors accumulate that drift
            const T nrm = sqrtf(s2);
            beta = -copysign(nrm, alpha);
            tau = (beta - alpha) / beta;
            scale = T(1) / (alpha - beta);
        }
    }
}

// Register tile: thread (warp w, lane l) holds rows l + 32a (a < 4) and
// columns w + 16q (q < 8) of the 128 x 128 block -- one coalesced 256-byte
// column segment per (a, q).
template <typename T, int BKT>
__device__ __forceinline__ void load_blk(const BandT<T> &A, const Blk &g, T (&x)[Shape<BKT>::RA][8]) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int c = w + Shape<BKT>::NW * q;
#pragma unroll
        for (int a = 0; a < Shape<BKT>::RA; ++a) {
            const int r = l + 32 * a;
            x[a][q] = (r < g.nr && c < g.nc) ? __ldcg(A.at(g.R0 + r, g.C0 + c)) : T(0);
        }
    }
}
// part: 0 all, 1 row 0 only, 2 column 0 only, 3 all but row 0, 4 all but column 0
template <typename T, int BKT>
__device__ __forceinline__ void store_blk(const BandT<T> &A, const Blk &g, const T (&x)[Shape<BKT>::RA][8],
                                          int part) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int c = w + Shape<BKT>::NW * q;
#pragma unroll
        for (int a = 0; a < Shape<BKT>::RA; ++a) {
            const int r = l + 32 * a;
            const bool sel = part == 0 || (part == 1 && r == 0) || (part == 2 && c == 0) ||
                             (part == 3 && r != 0) || (part == 4 && c != 0);
            if (sel && r < g.nr && c < g.nc) __stcg(A.at(g.R0 + r, g.C0 + c), x[a][q]);
        }
    }
}

// Pivot hand-off for the next op: the emitting CTA writes the raw vector to
// its own piv_self and to the receiving CTA's buffer (DSMEM).
template <typename T>
struct Emit {
    T *self;      // nullptr: nothing to emit
    uint32_t remote;   // cluster address of the receiver's buffer
    uint32_t rbar;     // cluster address of the receiver's mbarrier for it
};
// The remote half is an st.async whose completion is counted in bytes on the
// receiver's mbarrier (complete_tx): no fence, barrier or arrive on the
// sender's side -- the receiver's phase completes when all 1 KB has landed.
template <typename T>
__device__ __forceinline__ void emit_put(const Emit<T> &e, int j, T v) {
    e.self[j] = v;
    if constexpr (sizeof(T) == 8)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                         e.remote + 8u * (uint32_t)j),
                     "l"(__double_as_longlong(v)), "r"(e.rbar)
                     : "memory");
    else
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                         e.remote + 4u * (uint32_t)j),
                     "r"(__float_as_uint(v)), "r"(e.rbar)
                     : "memory");
}

// Sum of part[0..7] over the 32 lanes by recursive halving (9 shuffles, not
// 40); every lane returns all eight totals (8 broadcast shuffles).  Lane l
// owns total q = 4*bit4(l) + 2*bit3(l) + bit2(l) after the halving steps.
template <typename T>
__device__ __forceinline__ void lane_allreduce8(T (&part)[8]) {
    const int l = threadIdx.x & 31;
    T h4[4], h2[2], h1;
    const bool b4 = l & 16, b3 = l & 8, b2 = l & 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const T mine = b4 ? part[i + 4] : part[i], other = b4 ? part[i] : part[i + 4];
        h4[i] = mine + __shfl_xor_sync(0xffffffffu, other, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const T mine = b3 ? h4[i + 2] : h4[i], other = b3 ? h4[i] : h4[i + 2];
        h2[i] = mine + __shfl_xor_sync(0xffffffffu, other, 8);
    }
    {
        const T mine = b2 ? h2[1] : h2[0], other = b2 ? h2[0] : h2[1];
        h1 = mine + __shfl_xor_sync(0xffffffffu, other, 4);
    }
    h1 += __shfl_xor_sync(0xffffffffu, h1, 2);
    h1 += __shfl_xor_sync(0xffffffffu, h1, 1);
#pragma unroll
    for (int q = 0; q < 8; ++q) part[q] = __shfl_sync(0xffffffffu, h1, ((q >> 2) << 4) | (((q >> 1) & 1) << 3) | ((q & 1) << 2));
}

// Left reflector (rows of the block, pivot relative row 0) on every column:
// column dots reduce over the lanes.  carrier: column 0 is the pivot column.
// emit: row 0 after the update (the next right op's pivot) is shipped before
// the rest of the block is updated.
template <typename T, int BKT>
__device__ __forceinline__ void left_apply(T (&x)[Shape<BKT>::RA][8], const T *p, int L, T tau,
                                           T scale, T beta, bool carrier, const Emit<T> &em) {
    constexpr int RA = Shape<BKT>::RA, NWT = Shape<BKT>::NW;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    T va[RA], part[8];
#pragma unroll
    for (int a = 0; a < RA; ++a) {
        const int j = l + 32 * a;
        va[a] = j == 0 ? T(1) : (j < L ? p[j] * scale : T(0));
    }
    if (tau != T(0)) {                        // uniform across the CTA
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            T t = va[0] * x[0][q];
#pragma unroll
            for (int a = 1; a < RA; ++a) t = fma(va[a], x[a][q], t);
            part[q] = t;
        }
        lane_allreduce8<T>(part);
#pragma unroll
        for (int q = 0; q < 8; ++q) part[q] *= tau;
    } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) part[q] = T(0);
    }
    if (em.self && l == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) emit_put(em, w + NWT * q, fma(-part[q], va[0], x[0][q]));
    }
    if (tau != T(0)) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
            for (int a = 0; a < RA; ++a) x[a][q] = fma(-part[q], va[a], x[a][q]);
    }
    if (carrier && w == 0) {
#pragma unroll
        for (int a = 0; a < RA; ++a) x[a][0] = (l + 32 * a == 0) ? beta : T(0);
    }
}

// Right reflector (columns of the block, pivot relative column 0) on every
// row: row dots reduce over the 16 warps through shared memory.
// carrier: row 0 is the pivot row.  emit: column 0 after the update (the
// next left op's pivot).
template <typename T, int BKT>
__device__ __forceinline__ void right_apply(T (&x)[Shape<BKT>::RA][8], const T *p, int L, T tau,
                                            T scale, T beta, bool carrier,
                                            T (*red)[BKT], T (*red2)[BKT], const Emit<T> &em) {
    constexpr int RA = Shape<BKT>::RA, NWT = Shape<BKT>::NW;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, tid = threadIdx.x;
    T vq[8], td[RA];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int c = w + NWT * q;
        vq[q] = c == 0 ? T(1) : (c < L ? p[c] * scale : T(0));
    }
    if (tau != T(0)) {                        // uniform across the CTA
#pragma unroll
        for (int a = 0; a < RA; ++a) {
            T t = x[a][0] * vq[0];
#pragma unroll
            for (int q = 1; q < 8; ++q) t = fma(x[a][q], vq[q], t);
            red[w][l + 32 * a] = t;
        }
        __syncthreads();
        if constexpr (NWT == 16) {
            {
                const int row = tid & (BKT - 1), g = tid >> 7;
                red2[g][row] = (red[4 * g][row] + red[4 * g + 1][row]) + (red[4 * g + 2][row] + red[4 * g + 3][row]);
            }
            __syncthreads();
#pragma unroll
            for (int a = 0; a < RA; ++a) {
                const int r = l + 32 * a;
                td[a] = tau * ((red2[0][r] + red2[1][r]) + (red2[2][r] + red2[3][r]));
            }
        } else {
            // <= 8 warps: every thread sums its rows' NWT partials (fixed
            // pairwise tree: every warp gets the same bits)
#pragma unroll
            for (int a = 0; a < RA; ++a) {
                const int r = l + 32 * a;
                T v[NWT];
#pragma unroll
                for (int u = 0; u < NWT; ++u) v[u] = red[u][r];
#pragma unroll
                for (int h = NWT / 2; h > 0; h >>= 1)
#pragma unroll
                    for (int u = 0; u < h; ++u) v[u] += v[u + h];
                td[a] = tau * v[0];
            }
        }
    } else {
#pragma unroll
        for (int a = 0; a < RA; ++a) td[a] = T(0);
    }
    if (em.self && w == 0) {
#pragma unroll
        for (int a = 0; a < RA; ++a) emit_put(em, l + 32 * a, fma(-td[a], vq[0], x[a][0]));
    }
    if (tau != T(0)) {
#pragma unroll
        for (int a = 0; a < RA; ++a)
#pragma unroll
            for (int q = 0; q < 8; ++q) x[a][q] = fma(-td[a], vq[q], x[a][q]);
    }
    if (carrier && l == 0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[0][q] = (w + NWT * q == 0) ? beta : T(0);
    }
}

template <int NC>
__device__ __forceinline__ int msg_index(const int (&mc)[NC], int k) {
    const int dr = k % NC;
    int base = 0;
#pragma unroll
    for (int r = 0; r < NC; ++r)
        if (r == dr) base = mc[r];
    return base + k / NC - (dr == 0 ? 1 : 0);
}

// DEV: the development variants (BSVD_CHASE_TRACE timestamps, the
// BSVD_CHASE_EARLY edge reload); compiled out of the default kernel, whose
// register budget (128 at 512 threads) they would otherwise share.
template <int NC, typename T, bool DEV, int BKT>
__global__ void __launch_bounds__(Shape<BKT>::NTH, 1) k_chase2(T *band, int64_t n, int b, int64_t ld,
                                                              int64_t batch, int *flags, int fstride,
                                                              int64_t nitems, unsigned long long *trace,
                                                              int strict, unsigned long long *mbox) {
    static_assert(!DEV || BKT == 128, "the development variants assume 128 x 128 tiles");
    constexpr int RA = Shape<BKT>::RA, NTH = Shape<BKT>::NTH, BK = BKT, NWT = Shape<BKT>::NW;
    // the edge mailbox serves 4-byte bands (fp32 compute); fp64 keeps edge flags
    constexpr bool MBX = !DEV && sizeof(T) == 4;
    const bool mbx = MBX && mbox && !(strict & 1);
    __shared__ T piv_self[BK];
    __shared__ T piv0[BK];
    __shared__ T piv_in[2][BK];
    __shared__ T red[Shape<BKT>::NW][BK];
    __shared__ T red2[BKT == 128 ? 4 : 1][BK];
    __shared__ __align__(8) uint64_t mbar[2];
    const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
    const unsigned rank = cluster_rank();
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&mbar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&mbar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync<2>();
    int mc[NC];
#pragma unroll
    for (int r = 0; r < NC; ++r) mc[r] = 0;
    const int64_t cid = blockIdx.x / NC, ncl = gridDim.x / NC;
    for (int64_t item = cid; item < nitems; item += ncl) {
        const int64_t s = item / batch, m = item % batch;
        const BandT<T> A{band + m * n * ld, n, ld, b};
        int *fl = flags + (m * n + s) * (int64_t)fstride;     // fl[j]: block j stored
        const int nops = chase_nops(s, n, b);
        const int nprev = s > 0 ? chase_nops(s - 1, n, b) : 0;
        for (int k = (int)rank; k < nops; k += NC) {
            const Blk g = geom(s, k, n, b);
            unsigned long long *tr =
                (DEV && trace && m == 0 && s < 256 && k < 32 && tid == 0) ? trace + (s * 32 + k) * 16 : nullptr;
            if (tr) tr[0] = gtimer();
            T x[RA][8];
            if (s > 0 && (!DEV || !(strict & 2))) {
                // sweep s-1 must have stored blocks 0..k (flag 2) and the
                // edges of blocks k+1, k+2 (flag >= 1): the rows/columns of
                // this block that lie in them (scripts/chase_dep_check.py);
                // blocks below k-NC+1 were checked for this CTA's previous block
                const int lo = k >= NC ? k - NC + 1 : 0;
                // mailbox mode: only full flags of blocks <= k, polled by every
                // warp itself (lane j: flag lo + j), which then loads its part
                // of the block -- no CTA barrier between the flags and the load
                const int j = lo + (mbx ? l : tid);
                if (j < min(mbx ? k + 1 : k + 3, nprev) && !(strict & 16)) {
                    const int want = (j <= k || (strict & 1)) ? 2 : 1;
                    const int *f = fl - fstride + j;
                    for (int spin = 0; ld_acquire(f) < want; ++spin)
                        if (spin > 64) __nanosleep(32);
                }
                if (mbx) __syncwarp();
                else __syncthreads();
                load_blk<T, BKT>(A, g, x);
                if constexpr (MBX) {
                    if (mbx) {
                        // the last column (even k) / last row (odd k) of this block
                        // lies on the edges of the previous sweep's blocks k+1
                        // (all but its last element, at index +1) and k+2 (the
                        // last element, at index 0); everything else is in
                        // blocks <= k (scripts/chase_dep_check.py)
                        const int bl = b - 1;
                        const unsigned long long *mp =
                            mbox + ((m * 2 + ((s - 1) & 1)) * (int64_t)fstride) * MBX_STRIDE;
                        const uint32_t tag = (uint32_t)s;
                        // all of a thread's words are loaded at once (one round
                        // trip), then only the ones whose tag is stale re-polled
                        if (!(k & 1)) {
                            if (bl < g.nc && (bl % NWT) == w) {
                                const int q = bl / NWT;
                                const unsigned long long *pa[RA];
                                unsigned long long wv[RA];
#pragma unroll
                                for (int a = 0; a < RA; ++a) {
                                    const int r = l + 32 * a;
                                    const int ke = r < bl ? k + 1 : k + 2, je = r < bl ? r + 1 : 0;
                                    pa[a] = (r < g.nr && ke < nprev) ? mp + ke * MBX_STRIDE + je : nullptr;
                                    wv[a] = pa[a] ? mbox_ld(pa[a]) : 0ull;
                                }
#pragma unroll
                                for (int a = 0; a < RA; ++a) {
                                    if (!pa[a]) continue;
                                    for (int spin = 0; (uint32_t)(wv[a] >> 32) != tag && !(strict & 32); ++spin) {
                                        if (spin > 64) __nanosleep(32);
                                        wv[a] = mbox_ld(pa[a]);
                                    }
#pragma unroll
                                    for (int qq = 0; qq < 8; ++qq)
                                        if (qq == q) x[a][qq] = (T)__uint_as_float((uint32_t)wv[a]);
                                }
                            }
                        } else if (bl < g.nr && (bl & 31) == l) {
                            const int a0 = bl >> 5;
                            const unsigned long long *pq[8];
                            unsigned long long wv[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const int c = w + NWT * q;
                                const int ke = c < bl ? k + 1 : k + 2, je = c < bl ? c + 1 : 0;
                                pq[q] = (c < g.nc && ke < nprev) ? mp + ke * MBX_STRIDE + je : nullptr;
                                wv[q] = pq[q] ? mbox_ld(pq[q]) : 0ull;
                            }
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                if (!pq[q]) continue;
                                for (int spin = 0; (uint32_t)(wv[q] >> 32) != tag && !(strict & 32); ++spin) {
                                    if (spin > 64) __nanosleep(32);
                                    wv[q] = mbox_ld(pq[q]);
                                }
#pragma unroll
                                for (int a = 0; a < RA; ++a)
                                    if (a == a0) x[a][q] = (T)__uint_as_float((uint32_t)wv[q]);
                            }
                        }
                    }
                }
            } else if (DEV && s > 0) {
              if constexpr (DEV) {
                // sweep s-1 must have stored blocks 0..k (flag 2) and the
                // edges of blocks k+1, k+2 (flag >= 1): the rows/columns of
                // this block that lie in them (scripts/chase_dep_check.py);
                // blocks below k-NC+1 were checked for this CTA's previous block.
                // The block is loaded once blocks <= k are stored; the elements
                // on those two edges (a bit mask over the thread's slots, from
                // the geometry alone) are reloaded after the edge flags.
                const int lo = k >= NC ? k - NC + 1 : 0;
                const int j = lo + tid;
                if (j <= k && j < nprev) {
                    const int *f = fl - fstride + j;
                    for (int spin = 0; ld_acquire(f) < 2; ++spin)
                        if (spin > 64) __nanosleep(32);
                }
                __syncthreads();
                load_blk<T, BKT>(A, g, x);
                uint32_t mask = 0;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int ke = k + 1 + e;
                    const Blk ge = geom(s - 1, ke, n, b);
                    const int dr = (int)(ge.R0 - g.R0), dc = (int)(ge.C0 - g.C0);
                    if (ke < nprev && !(ke & 1)) {             // row 0 of an even block
                        if (dr >= 0 && dr < g.nr && (dr & 31) == l) {
                            const int clo = max(0, dc), chi = min(g.nc, dc + ge.nc);
                            uint32_t qb = 0;
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const int c = w + 16 * q;
                                qb |= (c >= clo && c < chi) ? (1u << q) : 0u;
                            }
                            mask |= qb << (8 * (dr >> 5));
                        }
                    } else if (ke < nprev) {                   // column 0 of an odd block
                        if (dc >= 0 && dc < g.nc && (dc & 15) == w) {
                            const int rlo = max(0, dr), rhi = min(g.nr, dr + ge.nr);
#pragma unroll
                            for (int aa = 0; aa < 4; ++aa) {
                                const int r = l + 32 * aa;
                                mask |= (r >= rlo && r < rhi) ? (1u << (8 * aa + (dc >> 4))) : 0u;
                            }
                        }
                    }
                }
                if (j > k && j < min(k + 3, nprev)) {
                    const int *f = fl - fstride + j;
                    for (int spin = 0; ld_acquire(f) < ((strict & 1) ? 2 : 1); ++spin)
                        if (spin > 64) __nanosleep(32);
                }
                __syncthreads();
                if (mask) {
#pragma unroll
                    for (int aa = 0; aa < 4; ++aa)
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if ((mask >> (8 * aa + q)) & 1u)
                                x[aa][q] = __ldcg(A.at(g.R0 + l + 32 * aa, g.C0 + w + 16 * q));
                }
              }
            } else {
                load_blk<T, BKT>(A, g, x);
            }
            if (tr) tr[1] = gtimer();
            const T *pv;
            int L;
            if (k == 0) {
                L = (int)min((int64_t)b, n - s - 1);
                for (int j = tid; j < BK; j += NTH) {
                    T v = T(0);
                    if (j < L) {
                        // (s, s+b) is column 0 (the edge) of the previous sweep's
                        // block 1, index 0: from the mailbox in that mode
                        if (MBX && mbx && s > 0 && j == b - 1 && 1 < nprev)
                            v = (T)mbox_get(mbox + ((m * 2 + ((s - 1) & 1)) * (int64_t)fstride + 1) * MBX_STRIDE,
                                            (uint32_t)s);
                        else
                            v = __ldcg(A.at(s, s + 1 + j));
                    }
                    piv0[j] = v;
                }
                __syncthreads();
                pv = piv0;
            } else {
                const int idx = msg_index<NC>(mc, k);
                if (tid == 0)       // this phase completes when the 1 KB pivot has landed
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                                     saddr(&mbar[idx & 1])),
                                 "n"(BK * (int)sizeof(T))
                                 : "memory");
                wait_local(saddr(&mbar[idx & 1]), (uint32_t)((idx >> 1) & 1));
                if (tr) tr[2] = gtimer();
                pv = piv_in[idx & 1];
                const Blk gp = geom(s, k - 1, n, b);
                L = (k & 1) ? gp.nr : gp.nc;
            }
            if (tr) {
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int q = 0; q < 8; ++q) { if constexpr (sizeof(T) == 8) asm volatile("" ::"d"(x[a][q])); else asm volatile("" ::"f"(x[a][q])); }
                tr[8] = gtimer();
            }
            T tau, scale, beta;
            reflector<T>(pv, L, tau, scale, beta);
            if (tr) tr[9] = gtimer();
            if (k == 0 && tid == 0) __stcg(A.at(s, s + 1), beta);
            if constexpr (MBX) {
                // block k-1's (0, 0) after its carrier op (= op k) is this op's
                // beta: publish that edge word now, ~2 us before the carrier
                // CTA publishes the whole edge -- it is the element the next
                // sweep's block k-3 waits for last (its (b-1, b-1))
                if (mbx && k >= 1 && tid == 0)
                    mbox_put(mbox + ((m * 2 + (s & 1)) * (int64_t)fstride + (k - 1)) * MBX_STRIDE, (uint32_t)(s + 1),
                             (float)beta);
            }
            // op k on the new block; its update yields op k+1's pivot, which is
            // shipped to the CTA holding block k+1 before the bulk update
            Emit<T> em{nullptr, 0u, 0u};
            if (k + 1 < nops) {
                const int dr = (k + 1) % NC;
                const int idx1 = msg_index<NC>(mc, k + 1);
                em.self = piv_self;
                em.remote = mapa(saddr(&piv_in[idx1 & 1][0]), (uint32_t)dr);
                em.rbar = mapa(saddr(&mbar[idx1 & 1]), (uint32_t)dr);
            }
            if (k & 1) left_apply<T, BKT>(x, pv, L, tau, scale, beta, false, em);
            else right_apply<T, BKT>(x, pv, L, tau, scale, beta, false, red, red2, em);
            if (tr) tr[3] = gtimer();
            if (k + 1 < nops) {
                __syncthreads();                        // piv_self complete
                if (tr) tr[4] = gtimer();
                const int L1 = (k & 1) ? g.nc : g.nr;
                reflector<T>(piv_self, L1, tau, scale, beta);
                const Emit<T> none{nullptr, 0u, 0u};
                if (k & 1) right_apply<T, BKT>(x, piv_self, L1, tau, scale, beta, true, red, red2, none);
                else left_apply<T, BKT>(x, piv_self, L1, tau, scale, beta, true, none);
            }
            if (tr) tr[5] = gtimer();
            // publish block k: its edge (row 0 of an even / Q-type block,
            // column 0 of an odd / E-type block -- the part the next sweep's
            // block k-2 / k-1 reads) first, then the rest
            bool edge_done = false;
            if constexpr (MBX) {
                if (mbox) {
                    // the edge goes to the mailbox first (no fence); the band
                    // copy of it is published with the rest of the block
                    unsigned long long *mp =
                        mbox + ((m * 2 + (s & 1)) * (int64_t)fstride + k) * MBX_STRIDE;
                    const uint32_t tag = (uint32_t)(s + 1);
                    if (!(k & 1)) {
                        if (l == 0 && g.nr > 0) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const int c = w + NWT * q;
                                if (c < g.nc) mbox_put(mp + c, tag, (float)x[0][q]);
                            }
                        }
                    } else if (w == 0 && g.nc > 0) {
#pragma unroll
                        for (int a = 0; a < RA; ++a) {
                            const int r = l + 32 * a;
                            if (r < g.nr) mbox_put(mp + r, tag, (float)x[a][0]);
                        }
                    }
                    edge_done = true;
                }
            }
            if (edge_done) {
                store_blk<T, BKT>(A, g, x, 0);
                __syncthreads();
                if (tid == 0) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    st_relaxed(fl + k, 2);
                }
            } else {
                const bool row_edge = !(k & 1);
                store_blk<T, BKT>(A, g, x, row_edge ? 1 : 2);
                __syncthreads();
                if (tid == 0) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    if (tr) tr[6] = gtimer();
                    st_relaxed(fl + k, 1);
                }
                store_blk<T, BKT>(A, g, x, row_edge ? 3 : 4);
                __syncthreads();
                if (tid == 0) {
                    asm volatile("fence.acq_rel.gpu;" ::: "memory");
                    st_relaxed(fl + k, 2);
                    if (tr) tr[7] = gtimer();
                }
            }
        }
        // messages each rank received in this sweep (blocks k >= 1, k = rank mod NC)
#pragma unroll
        for (int r = 0; r < NC; ++r) mc[r] += (r < nops ? (nops - r + NC - 1) / NC : 0) - (r == 0 ? 1 : 0);
    }
    cluster_sync<2>();
}
}  // namespace ch2

// ---------------------------------------------------------------------------
// Batched narrow-band chase (b <= 64, many matrices): one CTA per matrix runs
// its sweeps back to back with the carried-block scheme of ch2 inside the CTA
// -- the carried block, the new block and the prefetch of the next block all
// sit in registers (BK x BK tiles, thread (w, l) holds rows l + 32a and
// columns w + NW q), the pivot passes through shared memory, and because the
// previous sweep is complete, the next block's load is issued one op ahead.
namespace ch3 {
template <typename T, int BK, int NW>
struct Tile {
    static constexpr int RA = BK / 32, CQ = BK / NW;
    T v[RA][CQ];
};

template <typename T, int BK, int NW>
__device__ __forceinline__ void load_t(const ch2::BandT<T> &A, const ch2::Blk &g, Tile<T, BK, NW> &x) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < Tile<T, BK, NW>::CQ; ++q) {
        const int c = w + NW * q;
#pragma unroll
        for (int a = 0; a < Tile<T, BK, NW>::RA; ++a) {
            const int r = l + 32 * a;
            x.v[a][q] = (r < g.nr && c < g.nc) ? __ldcg(A.at(g.R0 + r, g.C0 + c)) : T(0);
        }
    }
}
template <typename T, int BK, int NW>
__device__ __forceinline__ void store_t(const ch2::BandT<T> &A, const ch2::Blk &g, const Tile<T, BK, NW> &x) {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int q = 0; q < Tile<T, BK, NW>::CQ; ++q) {
        const int c = w + NW * q;
#pragma unroll
        for (int a = 0; a < Tile<T, BK, NW>::RA; ++a) {
            const int r = l + 32 * a;
            if (r < g.nr && c < g.nc) __stcg(A.at(g.R0 + r, g.C0 + c), x.v[a][q]);
        }
    }
}
template <typename T>
__device__ __forceinline__ void refl(const T *p, int L, T &tau, T &scale, T &beta) {
    const int lane = threadIdx.x & 31;
    T sg = T(0);
    for (int j = 1 + lane; j < L; j += 32) sg = fma(p[j], p[j], sg);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sg += __shfl_xor_sync(0xffffffffu, sg, o);
    const T alpha = p[0];
    tau = T(0);
    scale = T(0);
    beta = alpha;
    if (sg != T(0)) {
        const T nrm = sqrt(fma(alpha, alpha, sg));
        beta = -copysign(nrm, alpha);
        tau = (beta - alpha) / beta;
        scale = T(1) / (alpha - beta);
    }
}
// Left reflector (block rows) on every column; carrier: column 0 is the pivot.
template <typename T, int BK, int NW>
__device__ __forceinline__ void left_t(Tile<T, BK, NW> &x, const T *p, int L, T tau, T scale, T beta,
                                       bool carrier) {
    constexpr int RA = Tile<T, BK, NW>::RA, CQ = Tile<T, BK, NW>::CQ;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (tau != T(0)) {
        T va[RA], part[CQ];
#pragma unroll
        for (int a = 0; a < RA; ++a) {
            const int j = l + 32 * a;
            va[a] = j == 0 ? T(1) : (j < L ? p[j] * scale : T(0));
        }
#pragma unroll
        for (int q = 0; q < CQ; ++q) {
            T t = va[0] * x.v[0][q];
#pragma unroll
            for (int a = 1; a < RA; ++a) t = fma(va[a], x.v[a][q], t);
            part[q] = t;
        }
        if constexpr (CQ == 8) {
            // reduce-scatter (lane bits 4,3,2 pick q; bits 1,0 finish the sum)
            // then broadcast: 17 shuffles instead of a 40-shuffle butterfly
            const unsigned F = 0xffffffffu;
            const bool hb = l & 16, mb = l & 8, lb = l & 4;
            T e1[4], e2[2];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const T mine = hb ? part[4 + t] : part[t], oth = hb ? part[t] : part[4 + t];
                e1[t] = mine + __shfl_xor_sync(F, oth, 16);
            }
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const T mine = mb ? e1[2 + t] : e1[t], oth = mb ? e1[t] : e1[2 + t];
                e2[t] = mine + __shfl_xor_sync(F, oth, 8);
            }
            T e3 = (lb ? e2[1] : e2[0]) + __shfl_xor_sync(F, lb ? e2[0] : e2[1], 4);
            e3 += __shfl_xor_sync(F, e3, 2);
            e3 += __shfl_xor_sync(F, e3, 1);
            // lane with bits (h, m, l) holds q = 4h + 2m + l
#pragma unroll
            for (int q = 0; q < 8; ++q) part[q] = __shfl_sync(F, e3, ((q >> 2) << 4) | (((q >> 1) & 1) << 3) | ((q & 1) << 2));
        } else {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int q = 0; q < CQ; ++q) part[q] += __shfl_xor_sync(0xffffffffu, part[q], o);
        }
#pragma unroll
        for (int q = 0; q < CQ; ++q) {
            const T tw = tau * part[q];
#pragma unroll
            for (int a = 0; a < RA; ++a) x.v[a][q] = fma(-tw, va[a], x.v[a][q]);
        }
    }
    if (carrier && w == 0) {
#pragma unroll
        for (int a = 0; a < RA; ++a) x.v[a][0] = (l + 32 * a == 0) ? beta : T(0);
    }
}
// Right reflector (block columns) on every row (dots over the NW warps
// through shared memory red[NW][BK]); carrier: row 0 is the pivot.
template <typename T, int BK, int NW>
__device__ __forceinline__ void right_t(Tile<T, BK, NW> &x, const T *p, int L, T tau, T scale, T beta,
                                        bool carrier, T *red) {
    constexpr int RA = Tile<T, BK, NW>::RA, CQ = Tile<T, BK, NW>::CQ;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (tau != T(0)) {                     // uniform across the CTA
        T vq[CQ];
#pragma unroll
        for (int q = 0; q < CQ; ++q) {
            const int c = w + NW * q;
            vq[q] = c == 0 ? T(1) : (c < L ? p[c] * scale : T(0));
        }
#pragma unroll
        for (int a = 0; a < RA; ++a) {
            T t = x.v[a][0] * vq[0];
#pragma unroll
            for (int q = 1; q < CQ; ++q) t = fma(x.v[a][q], vq[q], t);
            red[w * BK + l + 32 * a] = t;
        }
        __syncthreads();
        // reduce-scatter: thread r sums row r's NW partials once (the same
        // order as a per-thread sum), then every thread reads its RA row sums:
        // RA (+ NW for BK threads) shared loads per thread instead of RA * NW
        T *rsum = red + 2 * NW * BK;
        if ((int)threadIdx.x < BK) {
            T d = T(0);
#pragma unroll
            for (int g = 0; g < NW; ++g) d += red[g * BK + threadIdx.x];
            rsum[threadIdx.x] = d;
        }
        __syncthreads();                   // also orders these reads of red before the next op's writes
#pragma unroll
        for (int a = 0; a < RA; ++a) {
            const T td = tau * rsum[l + 32 * a];
#pragma unroll
            for (int q = 0; q < CQ; ++q) x.v[a][q] = fma(-td, vq[q], x.v[a][q]);
        }
    }
    if (carrier && l == 0) {
#pragma unroll
        for (int q = 0; q < CQ; ++q) x.v[0][q] = (w + NW * q == 0) ? beta : T(0);
    }
}

// right_t on the new block (x0) and the carried block (x1, carrier) with one
// shared-memory reduction round (red[2][NW][BK]) for both.
template <typename T, int BK, int NW>
__device__ __forceinline__ void right_t2(Tile<T, BK, NW> &x0, Tile<T, BK, NW> &x1, const T *p, int L, T tau,
                                         T scale, T beta, T *red) {
    constexpr int RA = Tile<T, BK, NW>::RA, CQ = Tile<T, BK, NW>::CQ;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (tau != T(0)) {                     // uniform across the CTA
        T vq[CQ];
#pragma unroll
        for (int q = 0; q < CQ; ++q) {
            const int c = w + NW * q;
            vq[q] = c == 0 ? T(1) : (c < L ? p[c] * scale : T(0));
        }
#pragma unroll
        for (int a = 0; a < RA; ++a) {
            T t0 = x0.v[a][0] * vq[0], t1 = x1.v[a][0] * vq[0];
#pragma unroll
            for (int q = 1; q < CQ; ++q) {
                t0 = fma(x0.v[a][q], vq[q], t0);
                t1 = fma(x1.v[a][q], vq[q], t1);
            }
            red[w * BK + l + 32 * a] = t0;
            red[(NW + w) * BK + l + 32 * a] = t1;
        }
        __syncthreads();
        // reduce-scatter over the 2 BK rows (thread t: block t / BK, row t % BK),
        // then each thread reads its 2 RA row sums
        static_assert(2 * BK <= NW * 32, "one thread per row sum");
        T *rsum = red + 2 * NW * BK;
        if ((int)threadIdx.x < 2 * BK) {
            const int blk = threadIdx.x / BK, r = threadIdx.x % BK;
            T d = T(0);
#pragma unroll
            for (int g = 0; g < NW; ++g) d += red[(blk * NW + g) * BK + r];
            rsum[threadIdx.x] = d;
        }
        __syncthreads();                   // also orders these reads of red before the next op's writes
#pragma unroll
        for (int a = 0; a < RA; ++a) {
            const int r = l + 32 * a;
            const T td0 = tau * rsum[r], td1 = tau * rsum[BK + r];
#pragma unroll
            for (int q = 0; q < CQ; ++q) {
                x0.v[a][q] = fma(-td0, vq[q], x0.v[a][q]);
                x1.v[a][q] = fma(-td1, vq[q], x1.v[a][q]);
            }
        }
    }
    if (l == 0) {
#pragma unroll
        for (int q = 0; q < CQ; ++q) x1.v[0][q] = (w + NW * q == 0) ? beta : T(0);
    }
}

template <typename T, int BK, int NW>
__global__ void __launch_bounds__(NW * 32) k_chase_cta(T *band, int64_t n, int b, int64_t ld,
                                                      int64_t batch) {
    using TL = Tile<T, BK, NW>;
    constexpr int RA = TL::RA, CQ = TL::CQ;
    __shared__ T piv[BK];
    __shared__ T red[2 * NW * BK + 2 * BK];   // partial row dots | row sums
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    for (int64_t m = blockIdx.x; m < batch; m += gridDim.x) {
        const ch2::BandT<T> A{band + m * n * ld, n, ld, b};
        for (int64_t s = 0; s + 2 < n; ++s) {
            const int nops = chase_nops(s, n, b);
            TL xc, xn, xp;
            __syncthreads();               // the previous sweep's stores are visible
            ch2::Blk g = ch2::geom(s, 0, n, b), gc = g;
            load_t<T, BK, NW>(A, g, xn);
            int L = (int)min((int64_t)b, n - s - 1);
            for (int j = threadIdx.x; j < BK; j += NW * 32) piv[j] = j < L ? __ldcg(A.at(s, s + 1 + j)) : T(0);
            __syncthreads();
            for (int k = 0; k < nops; ++k) {
                const ch2::Blk gn = k + 1 < nops ? ch2::geom(s, k + 1, n, b) : g;
                if (k + 1 < nops) load_t<T, BK, NW>(A, gn, xp);      // prefetch block k+1
                T tau, scale, beta;
                refl<T>(piv, L, tau, scale, beta);
                if (k == 0 && threadIdx.x == 0) __stcg(A.at(s, s + 1), beta);
                if (k & 1) {
                    left_t<T, BK, NW>(xn, piv, L, tau, scale, beta, false);
                    left_t<T, BK, NW>(xc, piv, L, tau, scale, beta, true);
                } else if (k > 0) {
                    right_t2<T, BK, NW>(xn, xc, piv, L, tau, scale, beta, red);
                } else {
                    right_t<T, BK, NW>(xn, piv, L, tau, scale, beta, false, red);
                }
                if (k > 0) store_t<T, BK, NW>(A, gc, xc);               // block k-1 is final
                __syncthreads();                                        // piv fully consumed
                if (k + 1 < nops) {
                    // op k+1's pivot: column 0 (left op next) or row 0 (right op next) of block k
                    if (!(k & 1)) {
                        if (w == 0) {
#pragma unroll
                            for (int a = 0; a < RA; ++a) piv[l + 32 * a] = xn.v[a][0];
                        }
                        L = g.nr;
                    } else {
                        if (l == 0) {
#pragma unroll
                            for (int q = 0; q < CQ; ++q) piv[w + NW * q] = xn.v[0][q];
                        }
                        L = g.nc;
                    }
                    __syncthreads();
                    xc = xn;
                    xn = xp;
                    gc = g;
                    g = gn;
                } else {
                    store_t<T, BK, NW>(A, g, xn);                        // the sweep's last block
                }
            }
        }
    }
}
}  // namespace ch3

// ops (= blocks) of sweep 0, the longest sweep: the per-sweep flag stride of
// the carried-block chase
static int chase_max_ops(int64_t n, int b) { return 3 + (int)(2 * ((n + b - 1) / b)); }

// k_chase2 serves every band width of single matrices and small batches
// (narrow bands too: measured 2-2.7x faster than the first-generation
// pipelined k_chase at b = 32 / 64, n = 300..2048); batches of >= 512 narrow
// bands keep one CTA per matrix (k_chase_cta).  BSVD_CHASE2_MIN=b restricts
// it to wider bands (development knob).
static bool chase2_used(int b, int64_t batch) {
    static const int lo = getenv("BSVD_CHASE2_MIN") ? atoi(getenv("BSVD_CHASE2_MIN")) : 0;
    return b > lo && b <= ch2::BK && (b > 64 || batch < 512);
}

size_t chase_workspace_bytes(int64_t n, int bw, int64_t batch) {
    const int64_t ld = 3 * (int64_t)bw + 1;
    size_t flags = chase2_used(bw, batch) ? (size_t)batch * n * chase_max_ops(n, bw) * sizeof(int) : 0;
    // + the edge mailbox of the fp32 cluster chase (2 sweep parities x blocks x 128 words)
    if (flags) flags += (size_t)batch * 2 * chase_max_ops(n, bw) * ch2::MBX_STRIDE * sizeof(unsigned long long) + 16;
    return (size_t)batch * (size_t)n * ((size_t)ld * sizeof(double) + sizeof(int)) + flags + 512;
}

// Carried-block cluster chase on a packed band of element type T (k_chase2).
template <typename T>
static cudaError_t launch_chase2(T *band, int64_t n, int b, int64_t ld, int64_t batch, int *progress,
                                 cudaStream_t st) {
    cudaError_t err;
        // carried-block cluster pipeline (NC CTAs per sweep, 1 CTA per SM)
        int NC = 4;
        if (const char *e = getenv("BSVD_CHASE_NC")) NC = atoi(e);
        if (NC < 2 || NC > 4) NC = 4;
        const int64_t nitems = (n - 2) * batch;
        const int64_t nops0 = 1 + 2 * ((n - 2 + b) / b);
        int64_t want = std::min<int64_t>(nitems, batch * (nops0 / 4 + 2));
        cudaLaunchConfig_t lc{};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = NC;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        lc.dynamicSmemBytes = 0;
        lc.stream = st;
        lc.attrs = attr;
        lc.numAttrs = 1;
        // tile: the narrowest of 32 / 64 / 128 that holds the band
        // (BSVD_CHASE_BK=128 forces the wide tile: development A/B)
        int bkt = b <= 32 ? 32 : (b <= 64 ? 64 : 128);
        if (const char *e = getenv("BSVD_CHASE_BK")) bkt = std::max(bkt, atoi(e) >= 128 ? 128 : (atoi(e) >= 64 ? 64 : 32));
        const bool dev = getenv("BSVD_CHASE_TRACE") || (getenv("BSVD_CHASE_EARLY") && atoi(getenv("BSVD_CHASE_EARLY")));
        if (dev) bkt = 128;
        void (*kern)(T *, int64_t, int, int64_t, int64_t, int *, int, int64_t, unsigned long long *, int,
                     unsigned long long *) =
            dev ? (NC == 2 ? ch2::k_chase2<2, T, true, 128>
                           : (NC == 3 ? ch2::k_chase2<3, T, true, 128> : ch2::k_chase2<4, T, true, 128>))
            : bkt == 32 ? (NC == 2 ? ch2::k_chase2<2, T, false, 32>
                                   : (NC == 3 ? ch2::k_chase2<3, T, false, 32> : ch2::k_chase2<4, T, false, 32>))
            : bkt == 64 ? (NC == 2 ? ch2::k_chase2<2, T, false, 64>
                                   : (NC == 3 ? ch2::k_chase2<3, T, false, 64> : ch2::k_chase2<4, T, false, 64>))
                        : (NC == 2 ? ch2::k_chase2<2, T, false, 128>
                                   : (NC == 3 ? ch2::k_chase2<3, T, false, 128> : ch2::k_chase2<4, T, false, 128>));
        lc.blockDim = dim3((unsigned)(bkt / 8 * 32));
        int max_clusters = 0;
        lc.gridDim = dim3((unsigned)(want * NC));
        err = cudaOccupancyMaxActiveClusters(&max_clusters, kern, &lc);
        if (err != cudaSuccess) return err;
        want = std::min<int64_t>(want, std::max(max_clusters, 1));
        lc.gridDim = dim3((unsigned)(want * NC));
        int64_t n_ = n, ld_ = ld, batch_ = batch;
        int b_ = b;
        const char *trace_path = getenv("BSVD_CHASE_TRACE");
        unsigned long long *trace = nullptr;
        const size_t trace_bytes = 256 * 32 * 16 * sizeof(unsigned long long);
        if (trace_path) {
            cudaMallocAsync((void **)&trace, trace_bytes, st);
            cudaMemsetAsync(trace, 0, trace_bytes, st);
        }
        int *flags = progress + batch * n;
        const int fstride = chase_max_ops(n, b);
        err = cudaMemsetAsync(flags, 0, (size_t)batch * n * fstride * sizeof(int), st);
        if (err != cudaSuccess) return err;
        // bit 1 (BSVD_CHASE_EARLY=1): load a block before its neighbours' edges
        // land and reload just those edges after their flags.  Measured: 59.9
        // vs 58.6 ms at 8192 and 145.7 vs 136.0 ms at 16384 (the extra CTA time
        // per block costs more than the earlier load saves) -- off by default.
        int early = 0;
        if (const char *e = getenv("BSVD_CHASE_EARLY")) early = atoi(e) ? 2 : 0;
        // BSVD_CHASE_DIAG=16 / 32 / 48: skip the block-flag / mailbox waits
        // (wrong values -- a timing diagnostic of which dependency binds)
        const int diag = getenv("BSVD_CHASE_DIAG") ? (atoi(getenv("BSVD_CHASE_DIAG")) & 48) : 0;
        if (diag) {
            static bool warned = false;
            if (!warned) {
                warned = true;
                fprintf(stderr, "bsvd: BSVD_CHASE_DIAG=%d skips chase dependencies -- the values are WRONG "
                                "(timing diagnostic only)\n", diag);
            }
        }
        const int strict = (getenv("BSVD_CHASE_STRICT") ? 1 : 0) | early | diag;
        // edge mailbox after the flags (fp32 bands; BSVD_CHASE_MBOX=0: edge flags)
        unsigned long long *mbox = nullptr;
        if (sizeof(T) == 4 && !dev && !(getenv("BSVD_CHASE_MBOX") && !atoi(getenv("BSVD_CHASE_MBOX")))) {
            mbox = (unsigned long long *)(((uintptr_t)(flags + (size_t)batch * n * fstride) + 15) & ~(uintptr_t)15);
            const size_t mbytes = (size_t)batch * 2 * fstride * ch2::MBX_STRIDE * sizeof(unsigned long long);
            err = cudaMemsetAsync(mbox, 0, mbytes, st);
            if (err != cudaSuccess) return err;
        }
        err = cudaLaunchKernelEx(&lc, kern, band, n_, b_, ld_, batch_, flags, fstride, nitems, trace, strict, mbox);
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
    return cudaSuccess;
}

template <typename S>
cudaError_t band_to_bidiagonal(const S *a, int64_t n, int64_t lda, int bw, int64_t batch,
                               int64_t a_bstride, double *d, double *e, void *ws,
                               cudaStream_t st) {
    if (n < 1 || batch < 1) return cudaSuccess;
    const int b = bw;
    const int64_t ld = 3 * (int64_t)b + 1;
    if (n > 2 && chase2_used(b, batch) && !getenv("BSVD_CHASE_V1")) {
        // carried-block cluster chase, in the compute precision of the input
        // (fp32 for FP32 / FP16 storage like the reference's chase,
        // secondstage.py:456-457; BSVD_CHASE_F64=1 keeps fp64)
        const bool f32 = sizeof(S) < 8 && !getenv("BSVD_CHASE_F64");
        const size_t es = f32 ? sizeof(float) : sizeof(double);
        char *bandp = (char *)ws;
        int *progress = (int *)(bandp + (size_t)batch * n * ld * es);
        cudaError_t err = cudaMemsetAsync(bandp, 0, (size_t)batch * n * ld * es, st);
        if (err != cudaSuccess) return err;
        const int64_t total = n * (int64_t)(bw + 1);
        dim3 grid((unsigned)std::min<int64_t>((total + 255) / 256, 4096), (unsigned)batch);
        dim3 g2((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)batch);
        if (f32) {
            k_pack_band<S, float><<<grid, 256, 0, st>>>(a, n, lda, a_bstride, bw, (float *)bandp, ld, b);
            bsvd_host::count_launch();
            if ((err = cudaGetLastError()) != cudaSuccess) return err;
            if ((err = launch_chase2<float>((float *)bandp, n, b, ld, batch, progress, st)) != cudaSuccess) return err;
            k_extract_bidiag<float><<<g2, 256, 0, st>>>((const float *)bandp, n, ld, b, d, e);
        } else {
            k_pack_band<S, double><<<grid, 256, 0, st>>>(a, n, lda, a_bstride, bw, (double *)bandp, ld, b);
            bsvd_host::count_launch();
            if ((err = cudaGetLastError()) != cudaSuccess) return err;
            if ((err = launch_chase2<double>((double *)bandp, n, b, ld, batch, progress, st)) != cudaSuccess) return err;
            k_extract_bidiag<double><<<g2, 256, 0, st>>>((const double *)bandp, n, ld, b, d, e);
        }
        bsvd_host::count_launch();
        return cudaGetLastError();
    }
    if (n > 2 && b <= 64 && batch >= 512 && !getenv("BSVD_CHASE_PIPELINED") && !getenv("BSVD_CHASE_SEQ")) {
        // many matrices, narrow band: one CTA per matrix (ch3), compute precision
        const bool f32 = sizeof(S) < 8 && !getenv("BSVD_CHASE_F64");
        const size_t es = f32 ? sizeof(float) : sizeof(double);
        char *bandp = (char *)ws;
        cudaError_t err = cudaMemsetAsync(bandp, 0, (size_t)batch * n * ld * es, st);
        if (err != cudaSuccess) return err;
        const int64_t total = n * (int64_t)(bw + 1);
        dim3 grid((unsigned)std::min<int64_t>((total + 255) / 256, 4096), (unsigned)batch);
        dim3 g2((unsigned)std::min<int64_t>((n + 255) / 256, 1024), (unsigned)batch);
        int dev = 0, nsm = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (f32) {
            k_pack_band<S, float><<<grid, 256, 0, st>>>(a, n, lda, a_bstride, bw, (float *)bandp, ld, b);
            bsvd_host::count_launch();
            auto kern = ch3::k_chase_cta<float, 64, 8>;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
            if (const char *e = getenv("BSVD_CTA_PER_SM")) per_sm = std::max(1, std::min(per_sm, atoi(e)));
            kern<<<(unsigned)std::min<int64_t>(batch, (int64_t)nsm * std::max(per_sm, 1)), 256, 0, st>>>(
                (float *)bandp, n, b, ld, batch);
            bsvd_host::count_launch();
            k_extract_bidiag<float><<<g2, 256, 0, st>>>((const float *)bandp, n, ld, b, d, e);
        } else {
            k_pack_band<S, double><<<grid, 256, 0, st>>>(a, n, lda, a_bstride, bw, (double *)bandp, ld, b);
            bsvd_host::count_launch();
            auto kern = ch3::k_chase_cta<double, 64, 8>;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
            kern<<<(unsigned)std::min<int64_t>(batch, (int64_t)nsm * std::max(per_sm, 1)), 256, 0, st>>>(
                (double *)bandp, n, b, ld, batch);
            bsvd_host::count_launch();
            k_extract_bidiag<double><<<g2, 256, 0, st>>>((const double *)bandp, n, ld, b, d, e);
        }
        bsvd_host::count_launch();
        return cudaGetLastError();
    }
    double *band = (double *)ws;
    int *progress = (int *)(band + batch * n * ld);
    cudaError_t err = cudaMemsetAsync(band, 0, (size_t)batch * n * ld * sizeof(double), st);
    if (err != cudaSuccess) return err;
    err = cudaMemsetAsync(progress, 0, (size_t)batch * n * sizeof(int), st);
    if (err != cudaSuccess) return err;
    {
        const int64_t total = n * (int64_t)(bw + 1);
        dim3 grid((unsigned)std::min<int64_t>((total + 255) / 256, 4096), (unsigned)batch);
        k_pack_band<S, double><<<grid, 256, 0, st>>>(a, n, lda, a_bstride, bw, band, ld, b);
        bsvd_host::count_launch();
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
    }
    if (false) {
    } else if (n > 2 && b <= 64 && batch >= 512 && !getenv("BSVD_CHASE_PIPELINED")) {
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
    k_extract_bidiag<double><<<g2, 256, 0, st>>>(band, n, ld, b, d, e);
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
