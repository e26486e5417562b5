// stage3_bisect.cu -- bidiagonal -> singular values on the GPU.
//
// Replaces the reference's host Demmel-Kahan QR iteration
// (secondstage.py:221-420, :473-507) with Sturm-count bisection on the
// Golub-Kahan tridiagonal TGK = tridiag(0; d1, e1, d2, ..., e_{n-1}, dn)
// whose eigenvalues are +-sigma_i.  Always float64 like the reference
// (secondstage.py:486-488).  Every value is independent: one thread per
// requested value, bisection on its ascending rank i with the invariant
// N(lo) < i <= N(hi), N(x) = #{sigma < x} = negcount(TGK - xI) - n, run until
// lo and hi are adjacent doubles, so sigma_i = lo exactly when the count is
// exact (diag(3,2,1) -> [3,2,1] bit-for-bit, test_secondstage.py:99-102).
// The off-diagonals are first scaled by a power of two so max|o| is in
// [1,2): power-of-two input scaling therefore commutes bit-exactly
// (test_secondstage.py:170-180), and o^2 can neither overflow nor underflow
// for representable inputs.  Only the largest n_out values are computed (the
// zero padding adds the smallest ones, matrix.py:163-181), already in the
// descending order secondstage.py:506 produces with a sort.
#include <stdlib.h>
#include <stdio.h>

#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace bsvd {

#ifndef BSVD_PROBE_ULPS
#define BSVD_PROBE_ULPS 4.0
#endif
constexpr double kProbeUlps = BSVD_PROBE_ULPS;   // first probe offset around Laguerre's iterate
#ifndef BSVD_STENCIL_SIDED
#define BSVD_STENCIL_SIDED 0
#endif
#ifndef BSVD_STENCIL_TRIG
#define BSVD_STENCIL_TRIG 0x1p-24
#endif
constexpr double kStencilTrig = BSVD_STENCIL_TRIG;   // relative Laguerre step that predicts convergence

// development instrumentation (BSVD_S3_STATS=file): per value the number of
// isolation / Laguerre / probe / final-bisection Sturm passes
__device__ int *g_s3stats = nullptr;
__device__ int64_t g_s3trace = -1;   // BSVD_S3_TRACE=k: printf the passes of value k (build -DBSVD_S3_DEBUG)

// Per-matrix prep: o2[j] = (o_j * 2^-p)^2, scal = {2^p, gersh_scaled}.
__global__ void __launch_bounds__(256) k_bisect_prep(const double *__restrict__ d,
                                                     const double *__restrict__ e, int64_t n,
                                                     double *__restrict__ o2,
                                                     double *__restrict__ scal) {
    const int64_t b = blockIdx.x;
    d += b * n;
    e += b * (n > 1 ? n - 1 : 0);
    o2 += b * (2 * n - 1);
    scal += b * 2;
    __shared__ double red[256];
    double m = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) m = fmax(m, fabs(d[j]));
    for (int64_t j = threadIdx.x; j + 1 < n; j += blockDim.x) m = fmax(m, fabs(e[j]));
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    const double omax = red[0];
    __syncthreads();
    double sc = 1.0;
    if (omax > 0.0) {
        int ex;
        frexp(omax, &ex);          // omax = f * 2^ex, f in [0.5, 1)
        sc = ldexp(1.0, 1 - ex);   // omax * sc in [1, 2)
    }
    double g = 0.0;
    for (int64_t j = threadIdx.x; j < 2 * n - 1; j += blockDim.x) {
        const double o = ((j & 1) ? e[j >> 1] : d[j >> 1]) * sc;
        o2[j] = o * o;
        const double prev = j > 0 ? fabs(((j - 1) & 1) ? e[(j - 1) >> 1] : d[(j - 1) >> 1]) * sc : 0.0;
        g = fmax(g, fabs(o) + prev);
    }
    if (threadIdx.x == 0 && n == 1) g = fabs(d[0]) * sc;
    red[threadIdx.x] = g;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        scal[0] = 1.0 / sc;   // exact: sc is a power of two
        scal[1] = red[0];
    }
}

// o / q for the Sturm recurrences: reciprocal seed, one Newton step (~2^-46)
// and one residual correction y + r (o - q y), which squares that error again:
// correctly rounded but for rare near-ties -- branch-free, because the
// recurrence's operands never reach the IEEE division's slow-path ranges
// (|q| >= pivmin = 2^-1000, o <= 4 after prescaling).  A second Newton step
// changed no value of 3 x 8192 tested and cost 14% of stage 3.
__device__ __forceinline__ double sdiv(double o, double q) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
    r = r * fma(-q, r, 2.0);
    const double y = o * r;
    return fma(fma(-q, y, o), r, y);
}

#ifdef BSVD_S3_RATIO
// #{eigenvalues of TGK < x} for the scaled problem (LAPACK dstebz-style
// negcount with a pivot floor; zero diagonal so a_j - x = -x).
__device__ __forceinline__ int negcount(const double *__restrict__ o2, int64_t m, double x,
                                        double pivmin) {
    // A vanishing pivot keeps its sign (+0 -> +pivmin): at x exactly equal to
    // an eigenvalue the count then excludes it, so exact inputs converge to
    // the exact value (LAPACK's q = -pivmin would count it).
    double q = -x;
    if (fabs(q) < pivmin) q = (q < 0.0) ? -pivmin : pivmin;
    int cnt = q < 0.0;
    for (int64_t j = 0; j < m; ++j) {
        q = -x - sdiv(__ldg(o2 + j), q);
        if (fabs(q) < pivmin) q = (q < 0.0) ? -pivmin : pivmin;
        cnt += q < 0.0;
    }
    return cnt;
}

// Two interleaved Sturm counts (independent dependency chains for ILP).
__device__ __forceinline__ void negcount2(const double *__restrict__ o2, int64_t m, double x0,
                                          double x1, double pivmin, int &c0, int &c1) {
    double q0 = -x0, q1 = -x1;
    if (fabs(q0) < pivmin) q0 = (q0 < 0.0) ? -pivmin : pivmin;
    if (fabs(q1) < pivmin) q1 = (q1 < 0.0) ? -pivmin : pivmin;
    int n0 = q0 < 0.0, n1 = q1 < 0.0;
    for (int64_t j = 0; j < m; ++j) {
        const double o = __ldg(o2 + j);
        q0 = -x0 - sdiv(o, q0);
        q1 = -x1 - sdiv(o, q1);
        if (fabs(q0) < pivmin) q0 = (q0 < 0.0) ? -pivmin : pivmin;
        if (fabs(q1) < pivmin) q1 = (q1 < 0.0) ? -pivmin : pivmin;
        n0 += q0 < 0.0;
        n1 += q1 < 0.0;
    }
    c0 = n0;
    c1 = n1;
}

// K interleaved Sturm counts (identical arithmetic to negcount per chain).
template <int K>
__device__ __forceinline__ void negcountK(const double *__restrict__ o2, int64_t m, const double (&x)[K],
                                          double pivmin, int (&c)[K]) {
    double q[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        q[i] = -x[i];
        if (fabs(q[i]) < pivmin) q[i] = (q[i] < 0.0) ? -pivmin : pivmin;
        c[i] = q[i] < 0.0;
    }
    for (int64_t j = 0; j < m; ++j) {
        const double o = __ldg(o2 + j);
#pragma unroll
        for (int i = 0; i < K; ++i) {
            q[i] = -x[i] - sdiv(o, q[i]);
            if (fabs(q[i]) < pivmin) q[i] = (q[i] < 0.0) ? -pivmin : pivmin;
            c[i] += q[i] < 0.0;
        }
    }
}

#else
// Continuant form (default): the leading principal minors
//   p_0 = 1, p_1 = -x, p_{j+1} = -x p_j - o2_j p_{j-1}
// of TGK - xI, whose sign changes are the same count as the negative pivots
// q_j = p_j / p_{j-1} of the ratio form above -- but the dependency chain per
// step is one FMA instead of a reciprocal, a Newton step and a correction
// (about 1/6 of the latency; the stage is latency-bound with one value per
// thread).  Every 8 steps the pair (p_{j-1}, p_j) is rescaled by the power of
// two that brings its larger magnitude into [1, 2): exact, so signs and the
// count are unaffected; between rescales |p| grows by at most 12^8 (|x| <= 8,
// o2 <= 4 after the prep's scaling) and shrinks by at most (2^-120)^8 (x >=
// floor_), both inside the double range.  Each minor is computed as
// fma(p_j, 2^-300, -x p_j - o2_j p_{j-1}): the recurrence at x - 2^-300
// (x >= floor_ = 2^-120 gersh, so far below an ulp of x) -- an exact zero
// minor becomes 2^-300 p_j, taking its predecessor's sign (the ratio form's
// q = +pivmin): at x exactly equal to an eigenvalue the count excludes it, so
// exact inputs still converge to the exact value, and a split (o2_j = 0)
// after a zero minor cannot stall the recurrence at zero.  Every nonzero
// minor is unchanged by the second rounding, and the fix costs one dependent
// FMA instead of a compare and select (61 against 90 cycles per step on
// B200, scripts/s3_lat.cu).
__device__ __forceinline__ double cstep(double x, double p, double o, double pm) {
    return fma(p, 0x1p-300, fma(-x, p, -o * pm));
}
// 2^(1023 - e) for the biased exponent e of v: v * pow2_norm(v) in [1, 2)
__device__ __forceinline__ double pow2_norm(double v) {
    return __hiloint2double(0x7fe00000 - (__double2hiint(v) & 0x7ff00000), 0);
}

// The o2 stream of the step loops: block j of 8 values.  Each block's loads
// are issued one iteration ahead (o2_load8 of j + 8 into `on`), so their
// latency never lands on the recurrence's dependency chain however the
// compiler schedules the iteration (a build that interleaved them with the
// chain ran stage 3 1.5x slower).
__device__ __forceinline__ void o2_load8(const double *__restrict__ o2, int64_t j, int64_t m, double (&o)[8]) {
    const bool ok = j + 8 <= m;
#pragma unroll
    for (int u = 0; u < 8; ++u) o[u] = ok ? __ldg(o2 + j + u) : 0.0;
}

template <int K>
__device__ __forceinline__ void negcountK(const double *__restrict__ o2, int64_t m, const double (&x)[K],
                                          double pivmin, int (&c)[K]) {
    (void)pivmin;
    double pm[K], p[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        pm[i] = 1.0;
        p[i] = fma(1.0, 0x1p-300, -x[i]);
        c[i] = p[i] < 0.0;
    }
    int64_t j = 0;
    double o[8];
    o2_load8(o2, 0, m, o);
    for (; j + 8 <= m; j += 8) {
        double on[8];
        o2_load8(o2, j + 8, m, on);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < K; ++i) {
                const double pn = cstep(x[i], p[i], o[u], pm[i]);
                c[i] += (pn < 0.0) != (p[i] < 0.0);
                pm[i] = p[i];
                p[i] = pn;
            }
        }
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const double s = pow2_norm(fmax(fabs(pm[i]), fabs(p[i])));
            pm[i] *= s;
            p[i] *= s;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) o[u] = on[u];
    }
    for (; j < m; ++j) {
        const double ot = __ldg(o2 + j);
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const double pn = cstep(x[i], p[i], ot, pm[i]);
            c[i] += (pn < 0.0) != (p[i] < 0.0);
            pm[i] = p[i];
            p[i] = pn;
        }
    }
}

__device__ __forceinline__ int negcount(const double *__restrict__ o2, int64_t m, double x, double pivmin) {
    const double xs[1] = {x};
    int c[1];
    negcountK<1>(o2, m, xs, pivmin, c);
    return c[0];
}

__device__ __forceinline__ void negcount2(const double *__restrict__ o2, int64_t m, double x0,
                                          double x1, double pivmin, int &c0, int &c1) {
    const double xs[2] = {x0, x1};
    int c[2];
    negcountK<2>(o2, m, xs, pivmin, c);
    c0 = c[0];
    c1 = c[1];
}
#endif

// Multisection of the bracket N(lo) < rank <= N(hi) with K points per pass
// (K interleaved chains in one thread: when values are scarce the stage is
// latency-bound and K chains cost about one pass of one chain): lo moves to
// the highest point with N < rank, hi to the next point, so the result is the
// pair of adjacent doubles plain bisection converges to.  Stops when no
// double lies strictly inside, hi <= floor_, or (isolate) the bracket holds
// one value.
template <int K>
__device__ __forceinline__ int multisect(const double *__restrict__ ob, int64_t n, int64_t rank, double &lo,
                                          double &hi, int64_t &clo, int64_t &chi, double pivmin, double floor_,
                                          bool isolate) {
    const int64_t m = 2 * n - 1;
    int pass = 0;
    for (; pass < 200; ++pass) {
        if (hi <= floor_ || (isolate && chi - clo == 1)) break;
        const double w = hi - lo;
        double x[K];
        bool ok[K];
        double prev = lo;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            double t = lo + w * ((double)(i + 1) / (double)(K + 1));
            ok[i] = t > prev && t < hi;
            if (ok[i]) prev = t;
            x[i] = ok[i] ? t : prev;
        }
        if (!ok[0] && !(0.5 * (lo + hi) > lo && 0.5 * (lo + hi) < hi)) break;   // adjacent
        if (!ok[0]) {                       // too narrow for K points: the midpoint alone
#pragma unroll
            for (int i = 0; i < K; ++i) { x[i] = 0.5 * (lo + hi); ok[i] = i == 0; }
        }
        int c[K];
        negcountK<K>(ob, m, x, pivmin, c);
        double nlo = lo, nhi = hi;
        int64_t nclo = clo, nchi = chi;
        int top = -1;
#pragma unroll
        for (int i = 0; i < K; ++i)
            if (ok[i] && c[i] - n < rank) top = i;
        if (top >= 0) { nlo = x[top]; nclo = c[top] - n; }
#pragma unroll
        for (int i = K - 1; i >= 0; --i)
            if (ok[i] && i > top && c[i] - n >= rank) { nhi = x[i]; nchi = c[i] - n; }
        lo = nlo; hi = nhi; clo = nclo; chi = nchi;
    }
    return pass;
}

#ifdef BSVD_S3_RATIO
// Sturm count (identical arithmetic to negcount) plus the Laguerre sums at x:
// G = sum 1/(x - lambda) = (log|f|)', S2 = (log|f|)'' = -sum 1/(x - lambda)^2
// for f(x) = det(TGK - x I), from the derivative recurrences of
// q_j = -x - o2_j / q_{j-1}:  a_j = q_j'/q_j = (t_j a_{j-1} - 1)/q_j,
// b_j = q_j''/q_j = t_j (b_{j-1} - 2 a_{j-1}^2)/q_j,  t_j = o2_j / q_{j-1}.
__device__ __forceinline__ double rcp_fast(double v) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
    return r * fma(-v, r, 2.0);          // one Newton step: ample for a derivative
}
__device__ __forceinline__ int sturm_laguerre(const double *__restrict__ o2, int64_t m, double x,
                                              double pivmin, double &G, double &S2) {
    double q = -x;
    if (fabs(q) < pivmin) q = (q < 0.0) ? -pivmin : pivmin;
    int cnt = q < 0.0;
    double a = -rcp_fast(q), bb = 0.0;
    double g = a, h = -a * a;
    for (int64_t j = 0; j < m; ++j) {
        const double t = sdiv(__ldg(o2 + j), q);
        double qn = -x - t;
        if (fabs(qn) < pivmin) qn = (qn < 0.0) ? -pivmin : pivmin;
        cnt += qn < 0.0;
        const double rn = rcp_fast(qn);
        const double an = fma(t, a, -1.0) * rn;
        const double bn = t * fma(-2.0 * a, a, bb) * rn;
        g += an;
        h = fma(-an, an, h + bn);
        q = qn;
        a = an;
        bb = bn;
    }
    G = g;
    S2 = h;
    return cnt;
}

#else
// Count plus the Laguerre sums from the continuant and its derivatives
// (p' and p'' obey the same recurrence with the extra terms -p, -2p'):
// G = p'/p and S2 = p''/p - G^2 at the end; the 8-step power-of-two rescale
// multiplies all six carried values alike.
__device__ __forceinline__ int sturm_laguerre(const double *__restrict__ o2, int64_t m, double x,
                                              double pivmin, double &G, double &S2) {
    (void)pivmin;
    double pm = 1.0, p = fma(1.0, 0x1p-300, -x);
    double dpm = 0.0, dp = -1.0, ddpm = 0.0, ddp = 0.0;
    int cnt = p < 0.0;
    int64_t j = 0;
    auto step = [&](double o) {
        const double pn = cstep(x, p, o, pm);
        const double dpn = fma(-x, dp, fma(-o, dpm, -p));
        const double ddpn = fma(-x, ddp, fma(-o, ddpm, -2.0 * dp));
        cnt += (pn < 0.0) != (p < 0.0);
        pm = p; p = pn;
        dpm = dp; dp = dpn;
        ddpm = ddp; ddp = ddpn;
    };
    double o[8];
    o2_load8(o2, 0, m, o);
    for (; j + 8 <= m; j += 8) {
        double on[8];
        o2_load8(o2, j + 8, m, on);
#pragma unroll
        for (int u = 0; u < 8; ++u) step(o[u]);
        const double s = pow2_norm(fmax(fabs(pm), fabs(p)));
        pm *= s; p *= s; dpm *= s; dp *= s; ddpm *= s; ddp *= s;
#pragma unroll
        for (int u = 0; u < 8; ++u) o[u] = on[u];
    }
    for (; j < m; ++j) step(__ldg(o2 + j));
    const double r = 1.0 / p;
    G = dp * r;
    S2 = fma(ddp, r, -G * G);
    return cnt;
}

// One pass: the Laguerre sums and the count at x (as sturm_laguerre) plus
// Sturm counts at E more points, all chains sharing the o2 stream (with E = 2
// a pass costs 106 cycles per step against 100 for sturm_laguerre alone and
// 66 for one count, scripts/s3_lat2.cu).
template <int E>
__device__ __forceinline__ int sturm_laguerre_pts(const double *__restrict__ o2, int64_t m, double x,
                                                  const double (&xs)[E], double &G, double &S2, int (&c)[E]) {
    double qm[E], q[E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
        qm[i] = 1.0;
        q[i] = fma(1.0, 0x1p-300, -xs[i]);
        c[i] = q[i] < 0.0;
    }
    double pm = 1.0, p = fma(1.0, 0x1p-300, -x);
    double dpm = 0.0, dp = -1.0, ddpm = 0.0, ddp = 0.0;
    int cnt = p < 0.0;
    auto step = [&](double o) {
        const double pn = cstep(x, p, o, pm);
        const double dpn = fma(-x, dp, fma(-o, dpm, -p));
        const double ddpn = fma(-x, ddp, fma(-o, ddpm, -2.0 * dp));
        cnt += (pn < 0.0) != (p < 0.0);
        pm = p; p = pn;
        dpm = dp; dp = dpn;
        ddpm = ddp; ddp = ddpn;
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const double qn = cstep(xs[i], q[i], o, qm[i]);
            c[i] += (qn < 0.0) != (q[i] < 0.0);
            qm[i] = q[i];
            q[i] = qn;
        }
    };
    int64_t j = 0;
    double o[8];
    o2_load8(o2, 0, m, o);
    for (; j + 8 <= m; j += 8) {
        double on[8];
        o2_load8(o2, j + 8, m, on);
#pragma unroll
        for (int u8 = 0; u8 < 8; ++u8) step(o[u8]);
        const double s = pow2_norm(fmax(fabs(pm), fabs(p)));
        pm *= s; p *= s; dpm *= s; dp *= s; ddpm *= s; ddp *= s;
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const double si = pow2_norm(fmax(fabs(qm[i]), fabs(q[i])));
            qm[i] *= si;
            q[i] *= si;
        }
#pragma unroll
        for (int u8 = 0; u8 < 8; ++u8) o[u8] = on[u8];
    }
    for (; j < m; ++j) step(__ldg(o2 + j));
    const double r = 1.0 / p;
    G = dp * r;
    S2 = fma(ddp, r, -G * G);
    return cnt;
}
#endif

// One value, bracket N(lo) < rank <= N(hi) with counts clo, chi known.  If
// the bracket isolates the value (chi - clo == 1), Laguerre's iteration for
// the real-rooted det(TGK - xI) (degree 2n) converges cubically and
// monotonically toward it from inside; every iterate's Sturm count keeps the
// bracket invariant, so a bad step only costs a bisection.  Then two probes
// a few ulps either side of the converged iterate and a short bisection to
// adjacent doubles give exactly the value plain bisection would return.
template <int K = 1>
__device__ __forceinline__ double finish_value(const double *__restrict__ ob, int64_t n, int64_t rank,
                                               double lo, double hi, int64_t clo, int64_t chi,
                                               double pivmin, double floor_) {
    const int64_t m = 2 * n - 1;
    int n_lag = 0, n_probe = 0, n_bis = 0;
    if (chi - clo == 1 && hi > floor_) {
        const double Nd = 2.0 * (double)n;
        double x = 0.5 * (lo + hi);
        bool conv = false;
        for (int it = 0; it < 40; ++it) {
            double G, S2;
            ++n_lag;
            const int64_t c = sturm_laguerre(ob, m, x, pivmin, G, S2) - n;
            if (c < rank) lo = x; else hi = x;
            if (!(hi - lo > 16.0 * 0x1p-52 * hi)) { conv = true; break; }
            const double H = -S2;
            double disc = (Nd - 1.0) * (Nd * H - G * G);
            disc = disc > 0.0 ? disc : 0.0;
            const double sq = sqrt(disc);
            const double xa = x - Nd / (G + sq), xb = x - Nd / (G - sq);
            double xn;
            if (c < rank) xn = fmax(xa, xb);          // the value lies above x
            else xn = fmin(xa, xb);                   // ... below (or at) x
            // a step within rounding noise: x sits on the value (the count
            // and the derivatives may then disagree about the side)
            if (fabs(xn - x) <= 64.0 * 0x1p-52 * fabs(x)) { conv = true; break; }
            if (!(xn > lo && xn < hi)) xn = 0.5 * (lo + hi);
            x = xn;
        }
        if (conv) {                                   // close the bracket around x
            double dl = kProbeUlps * 0x1p-52 * fabs(x) + pivmin;
            for (int rep = 0; rep < 4; ++rep) {
                const double xl = x - dl, xh = x + dl;
                const bool inl = xl > lo && xl < hi, inh = xh > lo && xh < hi;
                int cl = 0, ch = 0;                   // both probes in one pass
                ++n_probe;
                if (inl && inh) negcount2(ob, m, xl, xh, pivmin, cl, ch);
                else if (inl) cl = negcount(ob, m, xl, pivmin);
                else if (inh) ch = negcount(ob, m, xh, pivmin);
                if (inl) {
                    if (cl - n < rank) lo = xl; else hi = xl;
                }
                if (inh && xh > lo && xh < hi) {
                    if (ch - n < rank) lo = xh; else hi = xh;
                }
                if (hi - lo <= 2.5 * dl) break;
                dl *= 16.0;
            }
        }
    }
    if constexpr (K > 1) {                           // multisection to adjacent doubles
        n_bis = multisect<K>(ob, n, rank, lo, hi, clo, chi, pivmin, floor_, false);
    } else {
        for (int it = 0; it < 200; ++it) {           // bisection to adjacent doubles
            const double mid = 0.5 * (lo + hi);
            if (!(mid > lo && mid < hi) || hi <= floor_) break;
            ++n_bis;
            const int64_t cnt = negcount(ob, m, mid, pivmin) - n;
            if (cnt < rank) lo = mid; else hi = mid;
        }
    }
    if (g_s3stats && blockIdx.y == 0) {
        int *st = g_s3stats + 8 * (n - rank);
        st[1] = n_lag; st[2] = n_probe; st[3] = n_bis;
    }
    return lo;
}

// Multisection: a group of kLanes lanes owns one value; each round the lanes
// evaluate 2*kLanes interior points of [lo, hi] (two interleaved Sturm
// chains per lane) and keep the sub-interval where the count crosses the
// value's rank (4.1 bits per round instead of 1), until the value is
// isolated (exactly one eigenvalue in the bracket) or the points collapse.
// With kLanes == 1 plain bisection plays that role.  finish_value then
// converges by Laguerre's method (one lane).  The invariant
// N(lo) < rank <= N(hi) holds throughout, so the result equals bisection to
// adjacent doubles.
template <int kLanes, typename OutT>
__global__ void __launch_bounds__(128) k_bisect(const double *__restrict__ o2,
                                                const double *__restrict__ scal, int64_t n,
                                                int64_t n_out, OutT *__restrict__ out,
                                                int64_t out_stride) {
    const int lane = threadIdx.x & 31;
    const int sub = lane % kLanes;                       // lane within the value's group
    const unsigned gmask = ((1u << kLanes) - 1u) << (lane - sub);
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kLanes;   // output slot
    const int64_t b = blockIdx.y;
    const bool active = k < n_out;
    const double *ob = o2 + b * (2 * n - 1);
    const double unscale = scal[2 * b], gersh = scal[2 * b + 1];
    const int64_t rank = n - (active ? k : 0);           // ascending rank of the k-th largest
    double res = 0.0;
    if (gersh > 0.0) {
        const double pivmin = 0x1p-1000;
        const double floor_ = 0x1p-120 * gersh;
        double lo = 0.0, hi = 2.0 * gersh;
        int64_t clo = 0, chi = n;                        // N(lo), N(hi)
        constexpr int NP = 2 * kLanes;                   // points per round
        if constexpr (kLanes > 1) {
            for (int round = 0; round < 40; ++round) {
                if (hi <= floor_ || chi - clo == 1) break;
                const double h = (hi - lo) / (NP + 1);
                const double x0 = lo + h * (2 * sub + 1), x1 = lo + h * (2 * sub + 2);
                // points must be strictly increasing inside (lo, hi); else stop
                const bool ok = h > 0.0 && (lo + h) > lo && (lo + h * NP) < hi && x0 < x1;
                if (!__all_sync(gmask, ok)) break;
                int c0, c1;
                negcount2(ob, 2 * n - 1, x0, x1, pivmin, c0, c1);
                c0 -= (int)n;
                c1 -= (int)n;
                // bit t-1 of M <=> point t has N(x) < rank; lo moves to the HIGHEST such
                // point (robust even if rounding made the computed counts non-monotone:
                // every point above it has N >= rank, so hi = the next point).
                const unsigned below = __ballot_sync(gmask, c0 < rank) >> (lane - sub);
                const unsigned below1 = __ballot_sync(gmask, c1 < rank) >> (lane - sub);
                unsigned M = 0;
#pragma unroll
                for (int s = 0; s < kLanes; ++s)
                    M |= (((below >> s) & 1u) << (2 * s)) | (((below1 >> s) & 1u) << (2 * s + 1));
                const int nb = M ? 32 - __clz(M) : 0;             // highest point index below rank
                // counts at the new ends: point t is chain (t-1)&1 of lane (t-1)>>1
                const int base = lane - sub;
                const int tl = nb > 0 ? nb - 1 : 0, th = nb < NP ? nb : 0;
                const int l0 = __shfl_sync(gmask, c0, base + (tl >> 1)), l1 = __shfl_sync(gmask, c1, base + (tl >> 1));
                const int h0 = __shfl_sync(gmask, c0, base + (th >> 1)), h1 = __shfl_sync(gmask, c1, base + (th >> 1));
                if (nb > 0) clo = (tl & 1) ? l1 : l0;
                if (nb < NP) chi = (th & 1) ? h1 : h0;
                const double nlo = nb > 0 ? lo + h * nb : lo;
                const double nhi = nb < NP ? lo + h * (nb + 1) : hi;
                lo = nlo;
                hi = nhi;
            }
        } else {
            for (int it = 0; it < 64; ++it) {               // bisect until isolated
                if (hi <= floor_ || chi - clo == 1) break;
                const double mid = 0.5 * (lo + hi);
                if (!(mid > lo && mid < hi)) break;
                const int64_t cnt = negcount(ob, 2 * n - 1, mid, pivmin) - n;
                if (cnt < rank) { lo = mid; clo = cnt; } else { hi = mid; chi = cnt; }
            }
        }
        if (sub == 0) res = finish_value(ob, n, rank, lo, hi, clo, chi, pivmin, floor_) * unscale;
    }
    if (active && sub == 0) out[b * out_stride + k] = (OutT)res;
}

// Spectrum slicing: Sturm counts at P uniform points x_p = p h of
// (0, 2 gersh], two interleaved chains per thread.  cnt[p] = N(x_p) =
// #{sigma < x_p}; one count serves every value (a value's cell is found by
// binary search), so isolating n values costs P counts instead of ~n log.
__global__ void __launch_bounds__(128) k_slice(const double *__restrict__ o2,
                                               const double *__restrict__ scal, int64_t n, int P,
                                               int *__restrict__ cnt) {
    const int64_t b = blockIdx.y;
    const double *ob = o2 + b * (2 * n - 1);
    int *cb = cnt + b * (int64_t)(P + 1);
    const double gersh = scal[2 * b + 1];
    const double h = 2.0 * gersh / P;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 > P) return;
    if (i == 0) cb[0] = 0;
    if (!(gersh > 0.0)) {
        cb[2 * i + 1] = (int)n;
        if (2 * i + 2 <= P) cb[2 * i + 2] = (int)n;
        return;
    }
    const double pivmin = 0x1p-1000;
    const int p0 = 2 * i + 1, p1 = min(2 * i + 2, P);
    int c0, c1;
    negcount2(ob, 2 * n - 1, p0 * h, p1 * h, pivmin, c0, c1);
    cb[p0] = c0 - (int)n;
    if (p1 != p0) cb[p1] = c1 - (int)n;
}

// One thread per value: its cell from the slice counts (binary search for
// the first x_p with N(x_p) >= rank), bisection until the value is isolated,
// then finish_value (Laguerre + probes + bisection to adjacent doubles).
template <typename OutT, int K>
__global__ void __launch_bounds__(128) k_values(const double *__restrict__ o2,
                                                const double *__restrict__ scal,
                                                const int *__restrict__ cnt, int P, int64_t n,
                                                int64_t n_out, OutT *__restrict__ out,
                                                int64_t out_stride) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    if (k >= n_out) return;
    const double *ob = o2 + b * (2 * n - 1);
    const int *cb = cnt + b * (int64_t)(P + 1);
    const double unscale = scal[2 * b], gersh = scal[2 * b + 1];
    const int64_t rank = n - k;
    double res = 0.0;
    if (gersh > 0.0) {
        const double pivmin = 0x1p-1000;
        const double floor_ = 0x1p-120 * gersh;
        const double h = 2.0 * gersh / P;
        int lo_p = 0, hi_p = P;                          // cb[lo_p] < rank <= cb[hi_p]
        while (hi_p - lo_p > 1) {
            const int mid = (lo_p + hi_p) >> 1;
            if (__ldg(cb + mid) < rank) lo_p = mid; else hi_p = mid;
        }
        double lo = lo_p * h, hi = hi_p < P ? hi_p * h : 2.0 * gersh;
        int64_t clo = __ldg(cb + lo_p), chi = __ldg(cb + hi_p);
        if (!(clo < rank && rank <= chi)) {              // non-monotone counts: full range
            lo = 0.0; hi = 2.0 * gersh; clo = 0; chi = n;
        }
        if constexpr (K > 1) {
            const int it = multisect<K>(ob, n, rank, lo, hi, clo, chi, pivmin, floor_, true);   // until isolated
            if (g_s3stats && b == 0) g_s3stats[8 * k] = it;
        } else {
            int it = 0;
            for (; it < 64; ++it) {                      // bisect until isolated
                if (hi <= floor_ || chi - clo == 1) break;
                const double mid = 0.5 * (lo + hi);
                if (!(mid > lo && mid < hi)) break;
                const int64_t c = negcount(ob, 2 * n - 1, mid, pivmin) - n;
                if (c < rank) { lo = mid; clo = c; } else { hi = mid; chi = c; }
            }
            if (g_s3stats && b == 0) g_s3stats[8 * k] = it;
        }
        res = finish_value<K>(ob, n, rank, lo, hi, clo, chi, pivmin, floor_) * unscale;
    }
    out[b * out_stride + k] = (OutT)res;
}

#ifndef BSVD_S3_RATIO
// One thread per value, every pass the SAME code for every lane (a warp's
// lanes otherwise serialise their different phases): the Laguerre sums at a
// point xc plus counts at xa < xc < xb (sturm_laguerre_pts<2>).  Per lane:
//  * not isolated (or Laguerre given up): xa, xc, xb quarter the bracket;
//  * isolated: xc = Laguerre's iterate (the cell midpoint first), xa, xb =
//    xc -+ delta with delta = one ulp once the last step predicts xc within
//    rounding of the value (cubic convergence: relative step < 2^-18), else
//    xc itself (no extra information).  The ulp stencil
//    brackets the value between adjacent doubles in the same pass that
//    evaluates the converged iterate, so no separate probe or bisection
//    passes follow.
// Every count keeps N(lo) < rank <= N(hi); a lane is done when lo and hi are
// adjacent doubles (or hi <= floor_), i.e. at the value plain bisection
// returns.
template <typename OutT>
__global__ void __launch_bounds__(128) k_values_u(const double *__restrict__ o2,
                                                  const double *__restrict__ scal,
                                                  const int *__restrict__ cnt, int P, int64_t n,
                                                  int64_t n_out, OutT *__restrict__ out,
                                                  int64_t out_stride) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t b = blockIdx.y;
    const double *ob = o2 + b * (2 * n - 1);
    const int *cb = cnt + b * (int64_t)(P + 1);
    const double unscale = scal[2 * b], gersh = scal[2 * b + 1];
    if (!(gersh > 0.0)) {
        if (k < n_out) out[b * out_stride + k] = (OutT)0.0;
        return;
    }
    const int64_t m = 2 * n - 1;
    const int64_t rank = n - (k < n_out ? k : n_out - 1);
    const double floor_ = 0x1p-120 * gersh;
    const double h = 2.0 * gersh / P;
    int lo_p = 0, hi_p = P;                              // cb[lo_p] < rank <= cb[hi_p]
    while (hi_p - lo_p > 1) {
        const int mid = (lo_p + hi_p) >> 1;
        if (__ldg(cb + mid) < rank) lo_p = mid; else hi_p = mid;
    }
    double lo = lo_p * h, hi = hi_p < P ? hi_p * h : 2.0 * gersh;
    int64_t clo = __ldg(cb + lo_p), chi = __ldg(cb + hi_p);
    if (!(clo < rank && rank <= chi)) {                  // non-monotone counts: full range
        lo = 0.0; hi = 2.0 * gersh; clo = 0; chi = n;
    }
    const double Nd = 2.0 * (double)n;
    bool done = k >= n_out || hi <= floor_;
    bool lag_ok = true;                                  // Laguerre not given up
    bool above = true;       // the value lies below the iterate (Laguerre keeps the side)
    bool hunt = false;       // geometric search out from the bracket end next to the value
    double x = 0.5 * (lo + hi), sprev = 1.0, hd = 0.0;
    int n_pass = 0, n_lag = 0, n_fail = 0;
    for (int it = 0; it < 400; ++it) {
        if (!__any_sync(0xffffffffu, !done)) break;
        const bool lag = !done && !hunt && lag_ok && chi - clo == 1;
        const bool stencil = lag && sprev < kStencilTrig;
        double u = 0.0;
        double px[3];                                    // ascending; px[ic] is the Laguerre point
        int ic = 1;
        if (done) {
            px[0] = px[1] = px[2] = hi;
        } else if (lag) {
            u = __hiloint2double((__double2hiint(fabs(x)) & 0x7ff00000) - (52 << 20), 0);
            // once converged, two more doubles on the value's side of the
            // iterate; before that no extra information (a point between the
            // iterate and the value would push Laguerre's step outside the bracket)
            const double d = stencil ? u : 0.0;
#if BSVD_STENCIL_SIDED
            if (above) { px[0] = x - 2.0 * d; px[1] = x - d; px[2] = x; ic = 2; }
            else       { px[0] = x; px[1] = x + d; px[2] = x + 2.0 * d; ic = 0; }
#else
            px[0] = x - d; px[1] = x; px[2] = x + d;
#endif
        } else if (hunt) {
            // the value is within a few doubles of the end B next to it (a
            // converged Laguerre iterate that the stencil missed): B -+ hd,
            // 4 hd, 16 hd; a wider gap multiplies hd by 64 for the next pass
            if (above) { px[0] = hi - 16.0 * hd; px[1] = hi - 4.0 * hd; px[2] = hi - hd; }
            else       { px[0] = lo + hd; px[1] = lo + 4.0 * hd; px[2] = lo + 16.0 * hd; }
        } else {
            const double w = hi - lo;
            px[0] = lo + 0.25 * w;
            px[1] = lo + 0.5 * w;
            px[2] = lo + 0.75 * w;
        }
        const double xc = px[ic];
        const double xs[2] = {px[ic == 0 ? 1 : 0], px[ic == 2 ? 1 : 2]};
        double G, S2;
        int cs[2];
        // a warp whose active lanes all run plain Laguerre passes (their extra
        // points coincide with x_c) skips the two extra chains
        int64_t cc;
        if (__any_sync(0xffffffffu, !done && (!lag || stencil))) {
            cc = sturm_laguerre_pts<2>(ob, m, xc, xs, G, S2, cs) - n;
        } else {
            const int c0 = sturm_laguerre(ob, m, xc, 0x1p-1000, G, S2);
            cs[0] = cs[1] = c0;
            cc = c0 - n;
        }
        if (done) continue;
        ++n_pass;
        n_lag += lag;
        int64_t pc[3];
        pc[ic] = cc;
        pc[ic == 0 ? 1 : 0] = cs[0] - n;
        pc[ic == 2 ? 1 : 2] = cs[1] - n;
        // lo -> the highest point inside (lo, hi) with N < rank, hi -> the
        // lowest point above it with N >= rank (robust to non-monotone counts)
        int top = -1;
#pragma unroll
        for (int i = 0; i < 3; ++i)
            if (px[i] > lo && px[i] < hi && pc[i] < rank) top = i;
        double nlo = lo, nhi = hi;
        int64_t nclo = clo, nchi = chi;
        if (top >= 0) { nlo = px[top]; nclo = pc[top]; }
#pragma unroll
        for (int i = 2; i >= 0; --i)
            if (i > top && px[i] > lo && px[i] < hi && pc[i] >= rank) { nhi = px[i]; nchi = pc[i]; }
        lo = nlo; hi = nhi; clo = nclo; chi = nchi;
#ifdef BSVD_S3_DEBUG
        if (k == g_s3trace && b == 0)
            printf("pass %d lag %d st %d xc %.17g cc %lld (rank %lld) lo %.17g hi %.17g w/ulp %.3g G %.6g S2 %.6g sprev %.3g\n",
                   n_pass, (int)lag, (int)stencil, xc, (long long)cc, (long long)rank, lo, hi,
                   (hi - lo) / (0x1p-52 * fabs(hi)), G, S2, sprev);
#endif
        const double mid = 0.5 * (lo + hi);
        if (hi <= floor_ || !(mid > lo && mid < hi)) { done = true; continue; }
        if (lag) {
            above = cc >= rank;
            const double H = -S2;
            double disc = (Nd - 1.0) * (Nd * H - G * G);
            disc = disc > 0.0 ? disc : 0.0;
            const double sq = sqrt(disc);
            const double xa = xc - Nd / (G + sq), xb = xc - Nd / (G - sq);
            double xn = above ? fmin(xa, xb) : fmax(xa, xb);
            const double stp = fabs(xn - xc) / fabs(xc);
            sprev = stp <= 64.0 * 0x1p-52 ? 0.0 : stp;
            if (stencil) {
                // the stencil missed: the value is more than a double away on
                // its side.  A large step from a point that close is rounding
                // noise in G, S2: walk three doubles instead.  A second miss
                // (Laguerre creeping a few doubles per pass) hunts from the
                // bracket end next to the value
                if (stp > 0x1p-18) xn = above ? xc - 3.0 * u : xc + 3.0 * u;
                if (++n_fail >= 2) { hunt = true; hd = u; lag_ok = false; }
            }
            if (n_lag >= 16) { hunt = true; hd = u; lag_ok = false; }
            // a step onto or past a bound (the value within rounding of it):
            // the double next to that bound
            if (!(xn < hi)) xn = hi - __hiloint2double((__double2hiint(hi) & 0x7ff00000) - (52 << 20), 0);
            if (!(xn > lo)) xn = lo + __hiloint2double((__double2hiint(fabs(lo)) & 0x7ff00000) - (52 << 20), 0);
            if (!(xn > lo && xn < hi)) xn = mid;
            x = xn;
        } else if (hunt) {
            if (hi - lo <= 16.5 * hd) {
                // found: quartering finishes the bracket (<= 16 hd)
                hunt = false;                            // (lag_ok stays false)
            } else {
                hd *= 64.0;
            }
        } else if (lag_ok && chi - clo == 1) {
            x = mid;                                     // just isolated: Laguerre from the midpoint
            sprev = 1.0;
        }
    }
    if (k < n_out) {
        out[b * out_stride + k] = (OutT)(lo * unscale);
        if (g_s3stats && b == 0) {
            int *st = g_s3stats + 8 * k;
            st[0] = n_pass - n_lag; st[1] = n_lag; st[6] = n_fail; st[7] = lag_ok;   // hunt passes count as [0]
        }
    }
}
#endif

static int slice_points(int64_t n) {
    static const int per = getenv("BSVD_SLICE_PER") ? atoi(getenv("BSVD_SLICE_PER")) : 4;
    int64_t P = per * n;
    if (P < 256) P = 256;
    if (P > 65536) P = 65536;
    return (int)P;
}

size_t bisect_workspace_bytes(int64_t n, int64_t batch) {
    return (size_t)batch * ((size_t)(2 * n) * sizeof(double) + 2 * sizeof(double) +
                            (size_t)(slice_points(n) + 1) * sizeof(int)) + 512;
}

template <typename OutT>
cudaError_t bidiagonal_values(const double *d, const double *e, int64_t n, int64_t batch,
                              OutT *out, int64_t n_out, int64_t out_stride, void *ws,
                              cudaStream_t st) {
    if (n < 1 || batch < 1) return cudaSuccess;
    double *o2 = (double *)ws;
    double *scal = o2 + batch * (2 * n - 1);
    k_bisect_prep<<<(unsigned)batch, 256, 0, st>>>(d, e, n, o2, scal);
    bsvd_host::count_launch();
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    if (!getenv("BSVD_BISECT_MULTI")) {
        // spectrum slicing + one thread per value (Laguerre finish)
        const int P = slice_points(n);
        int *cnt = (int *)(((uintptr_t)(scal + 2 * batch) + 15) & ~(uintptr_t)15);
        k_slice<<<dim3((unsigned)((P / 2 + 1 + 127) / 128), (unsigned)batch), 128, 0, st>>>(o2, scal, n, P, cnt);
        bsvd_host::count_launch();
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        // small blocks spread the values over every SM
        // (one warp per block while that leaves SMs idle; batches fill them anyway)
        const int vb = getenv("BSVD_VALUES_BLOCK") ? atoi(getenv("BSVD_VALUES_BLOCK"))
                       : (n_out * batch >= 148 * 128 ? 128 : 32);
        // BSVD_VALUES_K=4/8: multisection with K interleaved chains per thread
        // (same values bit for bit; continuant counts at 8192: K=1 8.14 ms,
        // K=4 7.85 ms, K=8 11.25 ms; 16384: K=1 30.3 ms, K=4 25.1 ms)
        int K = 1;
        if (const char *e = getenv("BSVD_VALUES_K")) K = atoi(e) == 8 ? 8 : (atoi(e) == 4 ? 4 : 1);
        const dim3 vg((unsigned)((n_out + vb - 1) / vb), (unsigned)batch);
        if (const char *tr = getenv("BSVD_S3_TRACE")) {
            const int64_t tk = atoll(tr);
            cudaMemcpyToSymbolAsync(g_s3trace, &tk, sizeof(tk), 0, cudaMemcpyHostToDevice, st);
        }
        const char *stats_path = getenv("BSVD_S3_STATS");
        int *stats = nullptr;
        if (stats_path) {
            cudaMalloc(&stats, (size_t)n_out * 8 * sizeof(int));
            cudaMemset(stats, 0, (size_t)n_out * 8 * sizeof(int));
            cudaMemcpyToSymbolAsync(g_s3stats, &stats, sizeof(void *), 0, cudaMemcpyHostToDevice, st);
        }
        static const bool legacy = getenv("BSVD_VALUES_LEGACY") != nullptr;
#ifndef BSVD_S3_RATIO
        if (!legacy && !getenv("BSVD_VALUES_K"))
            k_values_u<OutT><<<vg, vb, 0, st>>>(o2, scal, cnt, P, n, n_out, out, out_stride);
        else
#endif
        if (K == 8)
            k_values<OutT, 8><<<vg, vb, 0, st>>>(o2, scal, cnt, P, n, n_out, out, out_stride);
        else if (K == 4)
            k_values<OutT, 4><<<vg, vb, 0, st>>>(o2, scal, cnt, P, n, n_out, out, out_stride);
        else
            k_values<OutT, 1><<<vg, vb, 0, st>>>(o2, scal, cnt, P, n, n_out, out, out_stride);
        if (stats) {
            void *null_ptr = nullptr;
            cudaMemcpyToSymbolAsync(g_s3stats, &null_ptr, sizeof(void *), 0, cudaMemcpyHostToDevice, st);
            std::vector<int> h((size_t)n_out * 8);
            cudaMemcpyAsync(h.data(), stats, h.size() * sizeof(int), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            if (FILE *f = fopen(stats_path, "wb")) { fwrite(h.data(), sizeof(int), h.size(), f); fclose(f); }
            cudaFree(stats);
        }
        bsvd_host::count_launch();
        return cudaGetLastError();
    }
    // Multisection when values are scarce (one large matrix), plain bisection
    // (one lane per value, least total work) when a batch supplies the parallelism.
    if (n_out * batch >= 131072) {
        dim3 grid((unsigned)((n_out + 127) / 128), (unsigned)batch);
        k_bisect<1, OutT><<<grid, 128, 0, st>>>(o2, scal, n, n_out, out, out_stride);
    } else {
        dim3 grid((unsigned)((n_out * 8 + 127) / 128), (unsigned)batch);
        k_bisect<8, OutT><<<grid, 128, 0, st>>>(o2, scal, n, n_out, out, out_stride);
    }
    bsvd_host::count_launch();
    return cudaGetLastError();
}

template cudaError_t bidiagonal_values<double>(const double *, const double *, int64_t, int64_t,
                                               double *, int64_t, int64_t, void *, cudaStream_t);
template cudaError_t bidiagonal_values<float>(const double *, const double *, int64_t, int64_t,
                                              float *, int64_t, int64_t, void *, cudaStream_t);

}  // namespace bsvd
