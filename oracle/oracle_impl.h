/* oracle_impl.h -- TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * One precision instance of the CPU restatement of the reference `bandsvd`
 * path.  Included three times by bsvd_oracle.c with
 *   S   storage element type        (double / float / uint16_t half bits)
 *   C   compute element type        (double / float / float)
 *   LD(p)  storage -> compute        ST(c)  compute -> storage (RNE)
 *   SUF    symbol suffix             EPS    compute-type unit roundoff
 *
 * Arithmetic order follows the reference statement by statement: serial
 * ascending sums, no FMA contraction (built with -ffp-contract=off), IEEE
 * sqrt and division, exactly like the numba @njit bodies it restates.
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SUF)

/* kernels.py:96-116 `_reflector_scalars` */
static inline void FN(reflector_scalars)(C piv, C sigma, C aik, C rho, C eps10, C two,
                                          C *x_out, C *tau_out, C *rhop_out) {
    C zero = eps10 - eps10;
    C x;
    if (piv < zero)
        x = piv - (C)SQRT(piv * piv + sigma);
    else
        x = piv + (C)SQRT(piv * piv + sigma);
    C tau, rhop;
    if ((x < zero ? -x : x) < eps10) {
        x = eps10;
        tau = two;
        rhop = two * (aik + rho / x);
    } else {
        tau = two * x * x / (x * x + sigma);
        rhop = (tau / x) * (aik * x + rho);
    }
    *x_out = x; *tau_out = tau; *rhop_out = rhop;
}

/* Split-K sum of x[j]*y[j] over rows [lo, ts) (kernels.py:233-361): segment t
 * of nsplit covers rows [t*ts/nsplit, (t+1)*ts/nsplit); each segment's partial
 * is a serial sum from zero (zero when empty: _norm2_tail / _dot_seg :71-93),
 * combined by `_pairwise_sum` (:191-199) -- ascending pairs, an odd tail
 * carried.  nsplit == 1: the plain serial `_norm2_tail` / `_dot_tail`. */
static inline C FN(split_dot)(const C *x, const C *y, int lo, int ts, int nsplit) {
    if (nsplit <= 1) {
        C s = (C)0;
        for (int j = lo; j < ts; ++j) s += x[j] * y[j];
        return s;
    }
    C v[128];
    for (int t = 0; t < nsplit; ++t) {
        int s0 = t * ts / nsplit, s1 = (t + 1) * ts / nsplit;
        int l = lo > s0 ? lo : s0;
        C s = (C)0;
        for (int j = l; j < s1; ++j) s += x[j] * y[j];
        v[t] = l < s1 ? s : (C)0;
    }
    int len = nsplit;
    while (len > 1) {
        int m = 0;
        for (int j = 0; j + 1 < len; j += 2) v[m++] = v[j] + v[j + 1];
        if (len & 1) v[m++] = v[len - 1];
        len = m;
    }
    return v[0];
}

/* Split-K segment updates (kernels.py:134-141 `_geqrt_seg_update`, :159-166
 * `_tsqrt_seg_update`) are njit functions the Python-level split-K generator
 * calls with x and rho' as Python floats: numba specialises them for float64
 * scalars, so for fp32 compute each element is updated in double and rounded
 * once.  (Same value as the plain form in fp64.) */
#define SEG_UPD(v, rhop, c, x) ((C)((double)(v) - (double)(rhop) * ((double)(c) / (double)(x))))
#define SEG_DIV(v, x) ((C)((double)(v) / (double)(x)))


/* Element (i, j) of a strided view: base[i*rs + j*cs] (matrix.py:93-154;
 * the lazy transpose is rs/cs swapped, never a copy). */
#define AT(p, i, j, rs, cs) ((p)[(int64_t)(i) * (rs) + (int64_t)(j) * (cs)])

/* kernels.py:205-230 `geqrt_kernel` (+ `_geqrt_item` :119-131).
 * Each work-item's private column is emulated by column i of P; item order
 * within a phase is irrelevant because items only share `col`/`nrm`.
 * Row k is written back at step k in the reference; every P[k, i] is final
 * after step k, so a single store at the end is the same bytes. */
void FN(oracle_geqrt)(S *a, int64_t rs, int64_t cs, int ts, C *tau, int nsplit) {
    const C zero = (C)0, two = (C)2, eps10 = (C)10 * (C)EPS;
    C *P = (C *)malloc(sizeof(C) * ts * ts);
    C *col = (C *)malloc(sizeof(C) * ts);
    for (int i = 0; i < ts; ++i)
        for (int j = 0; j < ts; ++j) P[i * ts + j] = LD(AT(a, j, i, rs, cs));
    for (int i = 0; i < ts; ++i) tau[i] = zero;
    for (int k = 0; k < ts - 1; ++k) {
        C *ak = P + k * ts;
        for (int j = 0; j < ts; ++j) col[j] = ak[j];
        /* _norm2_tail :71-76 (split-K: nparts + _pairwise_sum, :252-265) */
        C nrm = FN(split_dot)(col, col, k + 1, ts, nsplit);
        for (int i = k; i < ts; ++i) {
            C *ai = P + i * ts;
            C rho = FN(split_dot)(ai, col, k + 1, ts, nsplit);   /* _dot_tail :79-84 */
            C x, t, rhop;
            FN(reflector_scalars)(col[k], nrm, ai[k], rho, eps10, two, &x, &t, &rhop);
            ai[k] = ai[k] - rhop;
            if (nsplit > 1) {
                if (i > k) {
                    for (int j = k + 1; j < ts; ++j) ai[j] = SEG_UPD(ai[j], rhop, col[j], x);
                } else {
                    for (int j = k + 1; j < ts; ++j) ai[j] = SEG_DIV(ai[j], x);
                    tau[k] = t;
                }
            } else if (i > k) {
                for (int j = k + 1; j < ts; ++j) ai[j] = ai[j] - rhop * (col[j] / x);
            } else {
                for (int j = k + 1; j < ts; ++j) ai[j] = ai[j] / x;
                tau[k] = t;
            }
        }
    }
    for (int i = 0; i < ts; ++i)
        for (int j = 0; j < ts; ++j) AT(a, j, i, rs, cs) = ST(P[i * ts + j]);
    free(P); free(col);
}

/* kernels.py:286-313 `tsqrt_kernel` (+ `_tsqrt_item` :144-156): the [R; B_l]
 * chain with R resident (compute precision) across all tiles l. */
void FN(oracle_tsqrt_chain)(S *r, int64_t rrs, int64_t rcs, S **bs, int64_t brs, int64_t bcs,
                            C **taus, int nb, int ts, int nsplit) {
    const C two = (C)2, eps10 = (C)10 * (C)EPS;
    C *R = (C *)malloc(sizeof(C) * ts * ts);
    C *B = (C *)malloc(sizeof(C) * ts * ts);
    C *bcol = (C *)malloc(sizeof(C) * ts);
    for (int i = 0; i < ts; ++i)
        for (int j = 0; j < ts; ++j) R[i * ts + j] = LD(AT(r, j, i, rrs, rcs));
    for (int l = 0; l < nb; ++l) {
        S *b = bs[l];
        C *tau = taus[l];
        for (int i = 0; i < ts; ++i)
            for (int j = 0; j < ts; ++j) B[i * ts + j] = LD(AT(b, j, i, brs, bcs));
        for (int k = 0; k < ts; ++k) {
            for (int j = 0; j < ts; ++j) bcol[j] = B[k * ts + j];
            C sigma = FN(split_dot)(bcol, bcol, 0, ts, nsplit);
            C rkk = R[k * ts + k];
            for (int i = k; i < ts; ++i) {
                C *ri = R + i * ts, *bi = B + i * ts;
                C rho = FN(split_dot)(bi, bcol, 0, ts, nsplit);
                C x, t, rhop;
                FN(reflector_scalars)(rkk, sigma, ri[k], rho, eps10, two, &x, &t, &rhop);
                ri[k] = ri[k] - rhop;
                if (nsplit > 1) {
                    if (i > k) {
                        for (int j = 0; j < ts; ++j) bi[j] = SEG_UPD(bi[j], rhop, bcol[j], x);
                    } else {
                        for (int j = 0; j < ts; ++j) bi[j] = SEG_DIV(bi[j], x);
                        tau[k] = t;
                    }
                } else if (i > k) {
                    for (int j = 0; j < ts; ++j) bi[j] = bi[j] - rhop * (bcol[j] / x);
                } else {
                    for (int j = 0; j < ts; ++j) bi[j] = bi[j] / x;
                    tau[k] = t;
                }
            }
        }
        for (int i = 0; i < ts; ++i)
            for (int j = 0; j < ts; ++j) AT(b, j, i, brs, bcs) = ST(B[i * ts + j]);
    }
    for (int i = 0; i < ts; ++i)
        for (int j = 0; j < ts; ++j) AT(r, j, i, rrs, rcs) = ST(R[i * ts + j]);
    free(R); free(B); free(bcol);
}

/* kernels.py:364-389 `unmqr_kernel` (+ `_unmqr_item` :169-177): Q^T of a
 * geqrt panel applied to ncols columns; columns are independent work-items,
 * so the OpenMP split over columns is the ParallelBackend's group split. */
void FN(oracle_unmqr)(const S *panel, int64_t prs, int64_t pcs, const C *tau,
                      S *x, int64_t xrs, int64_t xcs, int ncols, int ts) {
    const C zero = (C)0;
    C *V = (C *)malloc(sizeof(C) * ts * ts);
    for (int k = 0; k < ts; ++k)
        for (int j = 0; j < ts; ++j) V[k * ts + j] = LD(AT(panel, j, k, prs, pcs));
#pragma omp parallel for schedule(static)
    for (int c = 0; c < ncols; ++c) {
        C xi[128];
        for (int j = 0; j < ts; ++j) xi[j] = LD(AT(x, j, c, xrs, xcs));
        for (int k = 0; k < ts - 1; ++k) {
            const C *ak = V + k * ts;
            C s = zero;
            for (int j = k + 1; j < ts; ++j) s += xi[j] * ak[j];
            C rho = tau[k] * (xi[k] + s);
            xi[k] = xi[k] - rho;
            for (int j = k + 1; j < ts; ++j) xi[j] = xi[j] - rho * ak[j];
        }
        for (int j = 0; j < ts; ++j) AT(x, j, c, xrs, xcs) = ST(xi[j]);
    }
    free(V);
}

/* kernels.py:392-421 `tsmqr_kernel` (+ `_tsmqr_item` :180-188): Y resident in
 * compute precision across the body rows, written once at the end. */
void FN(oracle_tsmqr)(S *y, int64_t yrs, int64_t ycs, S **xs, int64_t xrs, int64_t xcs,
                      S **vs, int64_t vrs, int64_t vcs, C **taus, int nb, int ncols, int ts) {
    const C zero = (C)0;
    C *V = (C *)malloc(sizeof(C) * ts * ts * (nb > 0 ? nb : 1));
    for (int l = 0; l < nb; ++l)
        for (int k = 0; k < ts; ++k)
            for (int j = 0; j < ts; ++j)
                V[((int64_t)l * ts + k) * ts + j] = LD(AT(vs[l], j, k, vrs, vcs));
#pragma omp parallel for schedule(static)
    for (int c = 0; c < ncols; ++c) {
        C yi[128], xi[128];
        for (int j = 0; j < ts; ++j) yi[j] = LD(AT(y, j, c, yrs, ycs));
        for (int l = 0; l < nb; ++l) {
            S *x = xs[l];
            const C *tau = taus[l];
            for (int j = 0; j < ts; ++j) xi[j] = LD(AT(x, j, c, xrs, xcs));
            for (int k = 0; k < ts; ++k) {
                const C *ak = V + ((int64_t)l * ts + k) * ts;
                C s = zero;
                for (int j = 0; j < ts; ++j) s += ak[j] * xi[j];
                s = (s + yi[k]) * tau[k];
                yi[k] = yi[k] - s;
                for (int j = 0; j < ts; ++j) xi[j] = xi[j] - s * ak[j];
            }
            for (int j = 0; j < ts; ++j) AT(x, j, c, xrs, xcs) = ST(xi[j]);
        }
        for (int j = 0; j < ts; ++j) AT(y, j, c, yrs, ycs) = ST(yi[j]);
    }
    free(V);
}

/* bandreduce.py:31-88 `getsmqrt` (fused path) on a view of the padded
 * column-major n x n matrix `a`; lq selects the lazy transpose.
 * tau: compute-dtype TauStore, column slot(k,l,side) (matrix.py:184-215). */
static void FN(oracle_getsmqrt)(S *a, int64_t n, C *tau, int k, int N, int ts, int lq, int nsplit) {
    int64_t rs = lq ? n : 1, cs = lq ? 1 : n;      /* view (i,j) -> base */
    int side = lq ? 1 : 0;
    int top = lq ? k + 1 : k;
    if (top >= N) return;
#define TILE(tr, tc) (a + (int64_t)(tr) * ts * rs + (int64_t)(tc) * ts * cs)
#define TAU(kk, ll) (tau + ((int64_t)side * N * N + (int64_t)(kk) * N + (ll)) * ts)
    S *diag = TILE(top, k);
    FN(oracle_geqrt)(diag, rs, cs, ts, TAU(k, top), nsplit);
    int ntrail = N - 1 - k;
    S *top_slab = TILE(top, k + 1);
    if (ntrail > 0)
        FN(oracle_unmqr)(diag, rs, cs, TAU(k, top), top_slab, rs, cs, ntrail * ts, ts);
    int nrows = N - (top + 1);
    if (nrows <= 0) return;
    S **vt = (S **)malloc(sizeof(S *) * nrows);
    S **body = (S **)malloc(sizeof(S *) * nrows);
    C **tc = (C **)malloc(sizeof(C *) * nrows);
    for (int idx = 0; idx < nrows; ++idx) {
        int l = top + 1 + idx;
        vt[idx] = TILE(l, k);
        body[idx] = TILE(l, k + 1);
        tc[idx] = TAU(k, l);
    }
    FN(oracle_tsqrt_chain)(diag, rs, cs, vt, rs, cs, tc, nrows, ts, nsplit);
    if (ntrail > 0)
        FN(oracle_tsmqr)(top_slab, rs, cs, body, rs, cs, vt, rs, cs, tc, nrows, ntrail * ts, ts);
    free(vt); free(body); free(tc);
#undef TILE
#undef TAU
}

/* bandreduce.py:91-120 `banddiag` + `_clear_outside_band`.  a: padded
 * column-major N*ts square; tau: ts x 2N^2 compute-dtype store (zeroed). */
void FN(oracle_banddiag)(S *a, int N, int ts, C *tau, int nsplit) {
    int64_t n = (int64_t)N * ts;
    for (int k = 0; k < N - 1; ++k) {
        FN(oracle_getsmqrt)(a, n, tau, k, N, ts, 0, nsplit);
        FN(oracle_getsmqrt)(a, n, tau, k, N, ts, 1, nsplit);
    }
    FN(oracle_getsmqrt)(a, n, tau, N - 1, N, ts, 0, nsplit);
    for (int64_t r = 0; r < n; ++r) {
        for (int64_t c = 0; c < r; ++c) a[c * n + r] = ST((C)0);
        for (int64_t c = r + ts + 1; c < n; ++c) a[c * n + r] = ST((C)0);
    }
}

/* secondstage.py:77-92 `_rotg` */
static inline void FN(rotg)(C f, C g, C *c, C *s, C *r) {
    const C zero = (C)0, one = (C)1;
    if (g == zero) { *c = one; *s = zero; *r = f; return; }
    if (f == zero) { *c = zero; *s = one; *r = g; return; }
    C f1 = f < zero ? -f : f, g1 = g < zero ? -g : g;
    C scale = f1 > g1 ? f1 : g1;
    C fs = f / scale, gs = g / scale;
    C dd = scale * (C)SQRT(fs * fs + gs * gs);
    *c = f1 / dd;
    C rr = f >= zero ? dd : -dd;
    *s = g / rr;
    *r = rr;
}

/* secondstage.py:95-146 `_chase_band` on a row-major (C-order) n x n array
 * in compute precision (band_to_bidiagonal copies with ascontiguousarray). */
void FN(oracle_chase_band)(C *a, int64_t n, int bw) {
    const C zero = (C)0;
#define A2(i, j) a[(int64_t)(i) * n + (j)]
    for (int64_t i = 0; i < n - 2; ++i) {
        int64_t jhi = i + bw <= n - 1 ? i + bw : n - 1;
        for (int64_t j = jhi; j > i + 1; --j) {
            C g = A2(i, j);
            if (g == zero) continue;
            C c, s, r;
            FN(rotg)(A2(i, j - 1), g, &c, &s, &r);
            A2(i, j - 1) = r;
            A2(i, j) = zero;
            int64_t rhi = j <= n - 1 ? j : n - 1;
            for (int64_t rr = i + 1; rr <= rhi; ++rr) {
                C t1 = A2(rr, j - 1), t2 = A2(rr, j);
                A2(rr, j - 1) = c * t1 + s * t2;
                A2(rr, j) = c * t2 - s * t1;
            }
            int64_t brow = j;
            for (;;) {
                int64_t bcol = brow - 1;
                C g1 = A2(brow, bcol);
                if (g1 != zero) {
                    FN(rotg)(A2(brow - 1, bcol), g1, &c, &s, &r);
                    A2(brow - 1, bcol) = r;
                    A2(brow, bcol) = zero;
                    int64_t chi = brow + bw <= n - 1 ? brow + bw : n - 1;
                    for (int64_t cc = bcol + 1; cc <= chi; ++cc) {
                        C t1 = A2(brow - 1, cc), t2 = A2(brow, cc);
                        A2(brow - 1, cc) = c * t1 + s * t2;
                        A2(brow, cc) = c * t2 - s * t1;
                    }
                }
                int64_t newcol = brow + bw;
                if (newcol > n - 1) break;
                C g2 = A2(brow - 1, newcol);
                if (g2 == zero) break;
                FN(rotg)(A2(brow - 1, newcol - 1), g2, &c, &s, &r);
                A2(brow - 1, newcol - 1) = r;
                A2(brow - 1, newcol) = zero;
                int64_t rhi2 = newcol <= n - 1 ? newcol : n - 1;
                for (int64_t rr = brow; rr <= rhi2; ++rr) {
                    C t1 = A2(rr, newcol - 1), t2 = A2(rr, newcol);
                    A2(rr, newcol - 1) = c * t1 + s * t2;
                    A2(rr, newcol) = c * t2 - s * t1;
                }
                brow = newcol;
            }
        }
    }
#undef A2
}

#undef AT
#undef FN
#undef CAT
#undef CAT_
