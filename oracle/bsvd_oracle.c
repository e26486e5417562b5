/* bsvd_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference `bandsvd.svdvals` path (arXiv 2508.06339
 * reference package, /root/reference/pkg/src/bandsvd).  This is the checker
 * the parity tests compare the B200 engine against, and the CPU baseline
 * `bench.py --impl reference` times ("kind": "port").  It is never linked
 * into, loaded by, or called from the product path (paper_2508_06339_b200).
 *
 * Pinning: tests/test_oracle_pinning.py checks this file bit-for-bit against
 * golden vectors produced by the reference itself (tests/golden/, generated
 * by scripts/make_golden.py while /root/reference was importable): stage-1
 * bands, stage-2 (d, e) and final values for fp64/fp32/fp16-storage.
 *
 * Build: see oracle/Makefile (-O2 -ffp-contract=off: numba never contracts
 * a*b+c into FMA).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline float h2f(uint16_t u) { _Float16 h; memcpy(&h, &u, 2); return (float)h; }
static inline uint16_t f2h(float f) { _Float16 h = (_Float16)f; uint16_t u; memcpy(&u, &h, 2); return u; }

/* ---- fp64 instance ---------------------------------------------------- */
#define S double
#define C double
#define LD(x) (x)
#define ST(x) (x)
#define SQRT sqrt
#define EPS 2.220446049250313e-16
#define SUF _f64
#include "oracle_impl.h"
#undef S
#undef C
#undef LD
#undef ST
#undef SQRT
#undef EPS
#undef SUF

/* ---- fp32 instance ---------------------------------------------------- */
#define S float
#define C float
#define LD(x) (x)
#define ST(x) (x)
#define SQRT sqrtf
#define EPS 1.1920928955078125e-07f
#define SUF _f32
#include "oracle_impl.h"
#undef S
#undef C
#undef LD
#undef ST
#undef SQRT
#undef EPS
#undef SUF

/* ---- fp16-storage instance (fp32 compute, RNE rounding on every store) -- */
#define S uint16_t
#define C float
#define LD(x) h2f(x)
#define ST(x) f2h(x)
#define SQRT sqrtf
#define EPS 1.1920928955078125e-07f
#define SUF _f16
#include "oracle_impl.h"
#undef S
#undef C
#undef LD
#undef ST
#undef SQRT
#undef EPS
#undef SUF

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---- stage 3: secondstage.py:149-420, always float64 ------------------ */

static inline void rotg_d(double f, double g, double *c, double *s, double *r) {
    if (g == 0.0) { *c = 1.0; *s = 0.0; *r = f; return; }
    if (f == 0.0) { *c = 0.0; *s = 1.0; *r = g; return; }
    double f1 = fabs(f), g1 = fabs(g);
    double scale = f1 > g1 ? f1 : g1;
    double fs = f / scale, gs = g / scale;
    double dd = scale * sqrt(fs * fs + gs * gs);
    *c = f1 / dd;
    double rr = f >= 0.0 ? dd : -dd;
    *s = g / rr;
    *r = rr;
}

/* secondstage.py:149-173 `_las2_min` */
static double las2_min(double f, double g, double h) {
    const double zero = 0.0, one = 1.0, two = 2.0;
    double fa = fabs(f), ga = fabs(g), ha = fabs(h);
    double fhmn = fa < ha ? fa : ha;
    double fhmx = fa > ha ? fa : ha;
    if (fhmn == zero) return zero;
    if (ga < fhmx) {
        double as_ = one + fhmn / fhmx;
        double at = (fhmx - fhmn) / fhmx;
        double au = (ga / fhmx) * (ga / fhmx);
        double c = two / (sqrt(as_ * as_ + au) + sqrt(at * at + au));
        return fhmn * c;
    }
    double au = fhmx / ga;
    if (au == zero) return fhmn * fhmx / ga;
    double as_ = one + fhmn / fhmx;
    double at = (fhmx - fhmn) / fhmx;
    double t1 = as_ * au, t2 = at * au;
    double c = one / (sqrt(one + t1 * t1) + sqrt(one + t2 * t2));
    return (fhmn * c) * au * two;
}

/* secondstage.py:176-218 `_lasv2_values` -> (ssmin, ssmax) */
static void lasv2_values(double f, double g, double h, double eps, double *ssmin, double *ssmax) {
    const double zero = 0.0, one = 1.0, two = 2.0;
    double half = one / two;
    double fa = fabs(f), ha = fabs(h);
    double ft = f, ht = h;
    if (ha > fa) { double t = ft; ft = ht; ht = t; t = fa; fa = ha; ha = t; }
    double ga = fabs(g);
    if (ga == zero) { *ssmin = ha; *ssmax = fa; return; }
    int gasmal = 1;
    if (ga > fa) {
        if (fa / ga < eps) {
            gasmal = 0;
            *ssmax = ga;
            if (ha > one) *ssmin = fa / (ga / ha);
            else *ssmin = (fa / ga) * ha;
            return;
        }
    }
    if (gasmal) {
        double dd = fa - ha;
        double ll = (dd == fa) ? one : dd / fa;
        double mm_ = g / ft;
        double tt_ = two - ll;
        double mm2 = mm_ * mm_, tt2 = tt_ * tt_;
        double s = sqrt(tt2 + mm2);
        double r = (ll == zero) ? fabs(mm_) : sqrt(ll * ll + mm2);
        double a = half * (s + r);
        *ssmin = ha / a;
        *ssmax = fa * a;
        return;
    }
    *ssmin = zero; *ssmax = zero;
    (void)ht;
}

/* secondstage.py:221-420 `_bdsqr_values`; returns sweeps or -1. */
static int64_t bdsqr_values(double *d, double *e, int64_t n, double eps, double tol,
                            double thresh, double ndt, int64_t maxit) {
    const double zero = eps - eps, one = eps / eps, two = one + one;
    const double ten = two + two + two + two + two;
    const double hndrth = one / (ten * ten);
    if (n == 1) { d[0] = fabs(d[0]); return 0; }
    int64_t iters = 0, m = n - 1, oldll = -2, oldm = -2;
    int idir = 0;
    while (m > 0) {
        int64_t ll = -1;
        for (int64_t lll = m - 1; lll >= 0; --lll)
            if (fabs(e[lll]) <= thresh) { ll = lll; break; }
        if (ll == m - 1) { e[m - 1] = zero; m -= 1; continue; }
        ll += 1;
        if (m == ll + 1) {
            double smin2, smax2;
            lasv2_values(d[ll], e[ll], d[m], eps, &smin2, &smax2);
            d[ll] = smax2; d[m] = smin2; e[ll] = zero;
            m = ll;
            if (m > 0) m -= 1;
            continue;
        }
        if (iters >= maxit) return -1;
        if (ll > oldm || m < oldll) idir = fabs(d[ll]) >= fabs(d[m]) ? 1 : 2;
        double sminl = zero;
        if (idir == 1) {
            if (fabs(e[m - 1]) <= tol * fabs(d[m])) { e[m - 1] = zero; continue; }
            double mu = fabs(d[ll]);
            sminl = mu;
            int conv = 0;
            for (int64_t lll = ll; lll < m; ++lll) {
                if (fabs(e[lll]) <= tol * mu) { e[lll] = zero; conv = 1; break; }
                mu = fabs(d[lll + 1]) * (mu / (mu + fabs(e[lll])));
                if (mu < sminl) sminl = mu;
            }
            if (conv) continue;
        } else {
            if (fabs(e[ll]) <= tol * fabs(d[ll])) { e[ll] = zero; continue; }
            double mu = fabs(d[m]);
            sminl = mu;
            int conv = 0;
            for (int64_t lll = m - 1; lll >= ll; --lll) {
                if (fabs(e[lll]) <= tol * mu) { e[lll] = zero; conv = 1; break; }
                mu = fabs(d[lll]) * (mu / (mu + fabs(e[lll])));
                if (mu < sminl) sminl = mu;
            }
            if (conv) continue;
        }
        oldll = ll; oldm = m;
        iters += 1;
        double smax = fabs(d[m]);
        for (int64_t lll = ll; lll < m; ++lll) {
            if (fabs(d[lll]) > smax) smax = fabs(d[lll]);
            if (fabs(e[lll]) > smax) smax = fabs(e[lll]);
        }
        double shift = zero;
        int use_zero = 1;
        double rhs = hndrth * tol;
        if (eps > rhs) rhs = eps;   /* max(eps, hndrth*tol) */
        if (smax > zero && ndt * tol * (sminl / smax) > rhs) {
            double sll, dll;
            if (idir == 1) {
                sll = fabs(d[ll]);
                shift = las2_min(d[m - 1], e[m - 1], d[m]);
                dll = d[ll];
            } else {
                sll = fabs(d[m]);
                shift = las2_min(d[ll], e[ll], d[ll + 1]);
                dll = d[m];
            }
            if (shift > zero && sll > zero && dll != zero) {
                double t = shift / sll;
                if (t * t >= eps) use_zero = 0;
            }
        }
        int64_t lo = ll, hi = m;
        int down = idir == 1;
        if (use_zero && down) {
            double cs = one, oldcs = one, sn = zero, oldsn = zero;
            for (int64_t i = lo; i < hi; ++i) {
                double c1, s1, r1, c2, s2, r2;
                rotg_d(d[i] * cs, e[i], &c1, &s1, &r1);
                cs = c1; sn = s1;
                if (i > lo) e[i - 1] = oldsn * r1;
                rotg_d(oldcs * r1, d[i + 1] * sn, &c2, &s2, &r2);
                oldcs = c2; oldsn = s2;
                d[i] = r2;
            }
            double h = d[hi] * cs;
            e[hi - 1] = h * oldsn;
            d[hi] = h * oldcs;
        } else if (use_zero) {
            double cs = one, oldcs = one, sn = zero, oldsn = zero;
            for (int64_t i = hi; i > lo; --i) {
                double c1, s1, r1, c2, s2, r2;
                rotg_d(d[i] * cs, e[i - 1], &c1, &s1, &r1);
                cs = c1; sn = s1;
                if (i < hi) e[i] = oldsn * r1;
                rotg_d(oldcs * r1, d[i - 1] * sn, &c2, &s2, &r2);
                oldcs = c2; oldsn = s2;
                d[i] = r2;
            }
            double h = d[lo] * cs;
            e[lo] = h * oldsn;
            d[lo] = h * oldcs;
        } else if (down) {
            double f = (fabs(d[lo]) - shift) * ((d[lo] >= zero ? one : -one) + shift / d[lo]);
            double g = e[lo];
            for (int64_t i = lo; i < hi; ++i) {
                double c1, s1, r1, c2, s2, r2;
                rotg_d(f, g, &c1, &s1, &r1);
                if (i > lo) e[i - 1] = r1;
                f = c1 * d[i] + s1 * e[i];
                e[i] = c1 * e[i] - s1 * d[i];
                g = s1 * d[i + 1];
                d[i + 1] = c1 * d[i + 1];
                rotg_d(f, g, &c2, &s2, &r2);
                d[i] = r2;
                f = c2 * e[i] + s2 * d[i + 1];
                d[i + 1] = c2 * d[i + 1] - s2 * e[i];
                if (i < hi - 1) {
                    g = s2 * e[i + 1];
                    e[i + 1] = c2 * e[i + 1];
                }
            }
            e[hi - 1] = f;
        } else {
            double f = (fabs(d[hi]) - shift) * ((d[hi] >= zero ? one : -one) + shift / d[hi]);
            double g = e[hi - 1];
            for (int64_t i = hi; i > lo; --i) {
                double c1, s1, r1, c2, s2, r2;
                rotg_d(f, g, &c1, &s1, &r1);
                if (i < hi) e[i] = r1;
                f = c1 * d[i] + s1 * e[i - 1];
                e[i - 1] = c1 * e[i - 1] - s1 * d[i];
                g = s1 * d[i - 1];
                d[i - 1] = c1 * d[i - 1];
                rotg_d(f, g, &c2, &s2, &r2);
                d[i] = r2;
                f = c2 * e[i - 1] + s2 * d[i - 1];
                d[i - 1] = c2 * d[i - 1] - s2 * e[i - 1];
                if (i > lo + 1) {
                    g = s2 * e[i - 2];
                    e[i - 2] = c2 * e[i - 2];
                }
            }
            e[lo] = f;
        }
        if (down) {
            if (fabs(e[hi - 1]) <= thresh) e[hi - 1] = zero;
        } else if (fabs(e[lo]) <= thresh) {
            e[lo] = zero;
        }
    }
    for (int64_t i = 0; i < n; ++i) d[i] = fabs(d[i]);
    return iters;
}

static int cmp_desc(const void *a, const void *b) {
    double x = *(const double *)a, y = *(const double *)b;
    return (x < y) - (x > y);
}

/* secondstage.py:473-507 `bidiagonal_values`: d, e overwritten; values
 * written descending into d.  Returns 0, or -1 on ConvergenceError. */
int oracle_bidiagonal_values(double *d, double *e, int64_t n) {
    const double eps = 2.220446049250313e-16;
    const double tiny = 2.2250738585072014e-308;
    double t = pow(eps, -0.125);
    double tol = (t < 100.0 ? t : 100.0);
    if (tol < 10.0) tol = 10.0;
    tol = tol * eps;
    double mu = fabs(d[0]), sminoa = mu;
    for (int64_t i = 1; i < n; ++i) {
        if (mu == 0.0) break;
        mu = fabs(d[i]) * (mu / (mu + fabs(e[i - 1])));
        if (mu < sminoa) sminoa = mu;
    }
    double a1 = tol * sminoa / sqrt((double)n);
    double a2 = 6.0 * (double)n * (double)n * tiny;
    double thresh = a1 > a2 ? a1 : a2;
    int64_t maxit = 30 * n * n;
    int64_t swept = bdsqr_values(d, e, n, eps, tol, thresh, (double)n, maxit);
    if (swept < 0) return -1;
    qsort(d, (size_t)n, sizeof(double), cmp_desc);
    return 0;
}

/* secondstage.py:423-449 `_dense_bidiagonalize` (bandwidth >= n fallback).
 * The reference calls numpy BLAS (dot / matvec) here, whose summation order
 * is library-defined: this branch is value-parity, not bit-parity.  a is
 * row-major n x n float64, overwritten. */
void oracle_dense_bidiagonalize(double *A, int64_t n, double *d, double *e) {
    double *v = (double *)malloc(sizeof(double) * n);
    double *w = (double *)malloc(sizeof(double) * n);
#define A2(i, j) A[(int64_t)(i) * n + (j)]
    for (int64_t k = 0; k < n; ++k) {
        int64_t m = n - k;
        double nx = 0.0;
        for (int64_t i = 0; i < m; ++i) nx += A2(k + i, k) * A2(k + i, k);
        nx = sqrt(nx);
        if (nx > 0 && m > 1) {
            for (int64_t i = 0; i < m; ++i) v[i] = A2(k + i, k);
            v[0] += A2(k, k) >= 0 ? nx : -nx;
            double vv = 0.0;
            for (int64_t i = 0; i < m; ++i) vv += v[i] * v[i];
            if (vv > 0) {
                for (int64_t j = k; j < n; ++j) {
                    double s = 0.0;
                    for (int64_t i = 0; i < m; ++i) s += v[i] * A2(k + i, j);
                    w[j - k] = (2.0 / vv) * s;
                }
                for (int64_t i = 0; i < m; ++i)
                    for (int64_t j = k; j < n; ++j) A2(k + i, j) -= v[i] * w[j - k];
            }
        }
        if (k < n - 2) {
            int64_t mc = n - k - 1;
            double nx2 = 0.0;
            for (int64_t j = 0; j < mc; ++j) nx2 += A2(k, k + 1 + j) * A2(k, k + 1 + j);
            nx2 = sqrt(nx2);
            if (nx2 > 0 && mc > 1) {
                for (int64_t j = 0; j < mc; ++j) v[j] = A2(k, k + 1 + j);
                v[0] += A2(k, k + 1) >= 0 ? nx2 : -nx2;
                double vv = 0.0;
                for (int64_t j = 0; j < mc; ++j) vv += v[j] * v[j];
                if (vv > 0) {
                    for (int64_t i = k; i < n; ++i) {
                        double s = 0.0;
                        for (int64_t j = 0; j < mc; ++j) s += A2(i, k + 1 + j) * v[j];
                        w[i - k] = (2.0 / vv) * s;
                    }
                    for (int64_t i = k; i < n; ++i)
                        for (int64_t j = 0; j < mc; ++j) A2(i, k + 1 + j) -= w[i - k] * v[j];
                }
            }
        }
    }
    for (int64_t i = 0; i < n; ++i) d[i] = A2(i, i);
    for (int64_t i = 0; i + 1 < n; ++i) e[i] = A2(i, i + 1);
#undef A2
    free(v); free(w);
}

/* ---- whole pipeline: secondstage.py:510-542 `svdvals` ------------------
 * a: column-major n x n in storage precision (already validated finite).
 * Writes d/e of the bidiagonal (compute precision widened to double) when
 * non-NULL, and the orig_n values (descending, float64) into vals.
 * prec: 1 fp64, 2 fp32, 3 fp16-storage (BSVD dtype codes, matrix.py:18).
 * Returns 0 or -1 (ConvergenceError). */
#define PIPE(SUF_, S_, C_, LDX, STX)                                                  \
    static int pipeline##SUF_(const S_ *a, int64_t n, int ts, double *vals,            \
                              S_ *band_out, double *d_out, double *e_out, int nsplit) {\
        int N = (int)((n + ts - 1) / ts);                                               \
        if (N < 1) N = 1;                                                              \
        int64_t np_ = (int64_t)N * ts;                                                  \
        S_ *w = (S_ *)calloc((size_t)(np_ * np_), sizeof(S_));                          \
        for (int64_t c = 0; c < n; ++c)                                                 \
            memcpy(w + c * np_, a + c * n, sizeof(S_) * (size_t)n);                     \
        C_ *tau = (C_ *)calloc((size_t)ts * 2 * N * N, sizeof(C_));                     \
        oracle_banddiag##SUF_(w, N, ts, tau, nsplit);                                   \
        if (band_out) memcpy(band_out, w, sizeof(S_) * (size_t)(np_ * np_));            \
        double *d = (double *)malloc(sizeof(double) * np_);                             \
        double *e = (double *)calloc((size_t)(np_ > 1 ? np_ - 1 : 1), sizeof(double));  \
        if (np_ == 1) {                                                                 \
            C_ v = LDX(w[0]); d[0] = (double)(C_)(v < 0 ? -v : v);                      \
        } else if (ts >= np_) {                                                         \
            double *A = (double *)malloc(sizeof(double) * np_ * np_);                   \
            for (int64_t r = 0; r < np_; ++r)                                           \
                for (int64_t c = 0; c < np_; ++c)                                       \
                    A[r * np_ + c] = (double)(C_)LDX(w[c * np_ + r]);                   \
            oracle_dense_bidiagonalize(A, np_, d, e);                                   \
            for (int64_t i = 0; i < np_; ++i) d[i] = (double)(C_)d[i];                  \
            for (int64_t i = 0; i + 1 < np_; ++i) e[i] = (double)(C_)e[i];              \
            free(A);                                                                    \
        } else {                                                                        \
            C_ *A = (C_ *)malloc(sizeof(C_) * np_ * np_);                               \
            for (int64_t r = 0; r < np_; ++r)                                           \
                for (int64_t c = 0; c < np_; ++c) A[r * np_ + c] = LDX(w[c * np_ + r]); \
            oracle_chase_band##SUF_(A, np_, ts);                                        \
            for (int64_t i = 0; i < np_; ++i) d[i] = (double)A[i * np_ + i];            \
            for (int64_t i = 0; i + 1 < np_; ++i) e[i] = (double)A[i * np_ + i + 1];    \
            free(A);                                                                    \
        }                                                                               \
        if (d_out) memcpy(d_out, d, sizeof(double) * np_);                              \
        if (e_out && np_ > 1) memcpy(e_out, e, sizeof(double) * (np_ - 1));             \
        int rc = oracle_bidiagonal_values(d, e, np_);                                   \
        if (rc == 0)                                                                    \
            for (int64_t i = 0; i < n; ++i) vals[i] = (double)(C_)d[i];                 \
        free(w); free(tau); free(d); free(e);                                           \
        return rc;                                                                      \
    }

#define IDENT(x) (x)
PIPE(_f64, double, double, IDENT, IDENT)
PIPE(_f32, float, float, IDENT, IDENT)
PIPE(_f16, uint16_t, float, h2f, f2h)

int oracle_svdvals_splitk(int prec, const void *a, int64_t n, int ts, double *vals,
                          void *band_out, double *d_out, double *e_out, int splitk) {
    switch (prec) {
    case 1: return pipeline_f64((const double *)a, n, ts, vals, (double *)band_out, d_out, e_out, splitk);
    case 2: return pipeline_f32((const float *)a, n, ts, vals, (float *)band_out, d_out, e_out, splitk);
    case 3: return pipeline_f16((const uint16_t *)a, n, ts, vals, (uint16_t *)band_out, d_out, e_out, splitk);
    default: return -2;
    }
}
int oracle_svdvals(int prec, const void *a, int64_t n, int ts, double *vals,
                   void *band_out, double *d_out, double *e_out) {
    return oracle_svdvals_splitk(prec, a, n, ts, vals, band_out, d_out, e_out, 1);
}

/* Stage-1 only (for timing samples and band parity): a is the padded
 * column-major N*ts square, overwritten with the band; tau zeroed store.
 * splitk > 1: the split-K panel kernels (kernels.py:233-361). */
void oracle_banddiag_splitk(int prec, void *a, int N, int ts, void *tau, int splitk) {
    switch (prec) {
    case 1: oracle_banddiag_f64((double *)a, N, ts, (double *)tau, splitk); break;
    case 2: oracle_banddiag_f32((float *)a, N, ts, (float *)tau, splitk); break;
    case 3: oracle_banddiag_f16((uint16_t *)a, N, ts, (float *)tau, splitk); break;
    }
}
void oracle_banddiag(int prec, void *a, int N, int ts, void *tau) { oracle_banddiag_splitk(prec, a, N, ts, tau, 1); }

/* Kernel-level entry points (column-major ts x ts tiles, compute-dtype tau);
 * splitk > 1: geqrt_splitk (kernels.py:459-470). */
void oracle_geqrt_splitk(int prec, void *a, int ts, void *tau, int splitk) {
    switch (prec) {
    case 1: oracle_geqrt_f64((double *)a, 1, ts, ts, (double *)tau, splitk); break;
    case 2: oracle_geqrt_f32((float *)a, 1, ts, ts, (float *)tau, splitk); break;
    case 3: oracle_geqrt_f16((uint16_t *)a, 1, ts, ts, (float *)tau, splitk); break;
    }
}
void oracle_geqrt(int prec, void *a, int ts, void *tau) { oracle_geqrt_splitk(prec, a, ts, tau, 1); }
