/*
 * iir_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU oracle for the hot path of
 * arXiv 2511.14390 ("differentiable (transposed) direct-form filters").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2511_14390_b200/csrc).
 *
 * Every quantity is computed sample by sample, in the paper's order and
 * notation, with DENSE M x M matrices -- no companion-structure shortcuts,
 * no chunking, no blocking.  Citations are to /root/reference/PAPER.md
 * lines (the LaTeX source) and equation numbers:
 *   Eq.1  rational transfer function
 *   Eq.2-3 direct form (type II)
 *   Eq.4-5 state space recursion / output
 *   companion realisation (A,B,C,D)
 *   TDF = (A^T, C, B, D)  ("swap B and C")
 *   Eq.6  dL/dv(n), dL/dC, dL/dD
 *   Eq.7  adjoint recursion dL/dz(n)
 *   Eq.8  dL/dx(n)
 *   Eq.9  dL/dv(0), dL/dB, dL/dA
 *   App. A.1 finite-N start dz(N-1)=0
 *   App. A.2 dA = sum dz(n)^T v(n)^T (vec)
 *   App. A.3 dv(0) = A^T dz(0) + C dy(0)
 *
 * Readings of the paper used here (DESIGN.md "Readings" lists them all):
 *   R1 companion orientation: row 0 = -a_1..-a_M, ones on the sub-diagonal,
 *      B = e_1 (the unique choice making Eqs.4-5 equal Eqs.2-3).
 *   R4 zf = v(N); the reverse recursion starts from dz(N-1) = grad_zf
 *      (grad_zf = 0 reproduces the paper's dz(N-1) = 0).
 *   R5 dA[i][j] = sum_n dz(n)[i] * v(n)[j]  (A.2 final line, Listing 1 l.341).
 *   R6 Eq.8's "B dL/dz^T" is the scalar B^T dz(n).
 *   R8 a_0 != 1 is accepted: coefficients are normalised by a_0 (Eq.1 is
 *      monic) and the gradient is chained back to the un-normalised b, a.
 *   R10 time-varying all-pole DF: row n of a applies at output time n,
 *      y(n) = x(n) - sum_i a_i(n) y(n-i)  ("easily extended").
 *   R11 its adjoint is Eq.7 with the time-varying A(n+1), C(n+1).
 *   R19 general time-varying DF (b(n) and a(n)): both rows apply at output
 *      time n; a(n) monic (orc_tv_df).
 *   R20 general time-varying TDF: the TDF realisation of PAPER.md:67-68
 *      ("replace A with its transpose and swap B and C") at every sample n,
 *      with the coefficient rows of sample n (orc_tv_tdf).
 */
#include <stdlib.h>
#include <string.h>

#define IDX(i, j, M) ((i) * (M) + (j))

/* ---- dense state-space realisation of Eq.1 ---------- */
/* form 0 = DF-II   : (A, B, C, D) = (companion(a), e1, c, b0)
 * form 1 = TDF-II  : (A^T, C, B, D) i.e. (companion(a)^T, c, e1, b0)
 * with c_k = b_k - a_k b_0 (k = 1..M), all on the a_0-normalised
 * coefficients.                                                          */
static void build_ss(int form, int M, const double *bn, const double *an,
                     double *Af, double *Bf, double *Cf, double *D)
{
    double *A = (double *)calloc((size_t)M * M, sizeof(double));
    double *c = (double *)malloc((size_t)M * sizeof(double));
    for (int k = 1; k <= M; ++k) {
        A[IDX(0, k - 1, M)] = -an[k];          /* first row: -a_1 .. -a_M */
        c[k - 1] = bn[k] - an[k] * bn[0];      /* C = [b_k - a_k b_0]     */
    }
    for (int i = 1; i < M; ++i) A[IDX(i, i - 1, M)] = 1.0; /* sub-diagonal */
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < M; ++j)
            Af[IDX(i, j, M)] = (form == 0) ? A[IDX(i, j, M)] : A[IDX(j, i, M)];
    for (int i = 0; i < M; ++i) {
        double e1 = (i == 0) ? 1.0 : 0.0;
        Bf[i] = (form == 0) ? e1 : c[i];
        Cf[i] = (form == 0) ? c[i] : e1;
    }
    *D = bn[0];
    free(A);
    free(c);
}

/*
 * orc_lti: one sequence of the LTI filter, forward (Eqs.4-5) and closed-form
 * backward (Eqs.6-9) for L = sum_n gy(n) y(n) + sum_i gzf[i] zf[i].
 *   form  0 = DF-II, 1 = TDF-II;  M >= 1;  N >= 1
 *   b[M+1], a[M+1] (a[0] != 0), x[N], zi[M] (NULL = 0), gy[N] (NULL = 0),
 *   gzf[M] (NULL = 0).
 *   Outputs (each may be NULL = skip): y[N], zf[M], gx[N], gb[M+1],
 *   ga[M+1], gzi[M].
 * Returns 0 on success, 1 on bad arguments, 2 on allocation failure.
 */
int orc_lti(int form, int M, long N, const double *b, const double *a,
            const double *x, const double *zi, const double *gy,
            const double *gzf, double *y, double *zf, double *gx,
            double *gb, double *ga, double *gzi)
{
    if (M < 1 || N < 1 || (form != 0 && form != 1) || a[0] == 0.0) return 1;
    const double a0 = a[0];
    double *bn = (double *)malloc((size_t)(M + 1) * sizeof(double));
    double *an = (double *)malloc((size_t)(M + 1) * sizeof(double));
    double *Af = (double *)malloc((size_t)M * M * sizeof(double));
    double *Bf = (double *)malloc((size_t)M * sizeof(double));
    double *Cf = (double *)malloc((size_t)M * sizeof(double));
    double *v = (double *)malloc((size_t)(N + 1) * M * sizeof(double));
    double *dz = (double *)malloc((size_t)N * M * sizeof(double));
    double *tmp = (double *)malloc((size_t)M * sizeof(double));
    double D;
    if (!bn || !an || !Af || !Bf || !Cf || !v || !dz || !tmp) return 2;

    /* Eq.1 is monic: normalise by a_0 (reading R8). */
    for (int k = 0; k <= M; ++k) { bn[k] = b[k] / a0; an[k] = a[k] / a0; }
    build_ss(form, M, bn, an, Af, Bf, Cf, &D);

    /* ---- forward, Eqs.4-5: v(n+1) = A v(n) + B x(n); y = C^T v + D x -- */
    for (int i = 0; i < M; ++i) v[i] = zi ? zi[i] : 0.0;
    for (long n = 0; n < N; ++n) {
        const double *vn = v + n * M;
        double *vn1 = v + (n + 1) * M;
        double yn = D * x[n];
        for (int i = 0; i < M; ++i) yn += Cf[i] * vn[i];
        if (y) y[n] = yn;
        for (int i = 0; i < M; ++i) {
            double s = Bf[i] * x[n];
            for (int j = 0; j < M; ++j) s += Af[IDX(i, j, M)] * vn[j];
            vn1[i] = s;
        }
    }
    if (zf) for (int i = 0; i < M; ++i) zf[i] = v[N * M + i];

    /* ---- backward ------------------------------------------------------ */
    /* Eq.7 with the finite-N start (A.1, reading R4): dz(N-1) = grad_zf,
     * dz(n) = A^T dz(n+1) + C dy(n+1),  n = N-2 .. 0.                     */
    for (int i = 0; i < M; ++i) dz[(N - 1) * M + i] = gzf ? gzf[i] : 0.0;
    for (long n = N - 2; n >= 0; --n) {
        const double *d1 = dz + (n + 1) * M;
        double dy1 = gy ? gy[n + 1] : 0.0;
        for (int i = 0; i < M; ++i) {
            double s = Cf[i] * dy1;
            for (int j = 0; j < M; ++j) s += Af[IDX(j, i, M)] * d1[j];
            dz[n * M + i] = s;
        }
    }
    /* Eq.8: dx(n) = B^T dz(n) + D dy(n) (reading R6). */
    if (gx)
        for (long n = 0; n < N; ++n) {
            double s = D * (gy ? gy[n] : 0.0);
            for (int i = 0; i < M; ++i) s += Bf[i] * dz[n * M + i];
            gx[n] = s;
        }
    /* Eq.9 / A.3: dv(0) = dz(-1) = A^T dz(0) + C dy(0). */
    if (gzi) {
        double dy0 = gy ? gy[0] : 0.0;
        for (int i = 0; i < M; ++i) {
            double s = Cf[i] * dy0;
            for (int j = 0; j < M; ++j) s += Af[IDX(j, i, M)] * dz[j];
            gzi[i] = s;
        }
    }
    if (gb || ga) {
        /* Eq.6 and Eq.9 sums over n = 0..N-1 (reading R7):
         *   dC = sum dy(n) v(n),  dD = sum dy(n) x(n),
         *   dB = sum dz(n) x(n),  dA[i][j] = sum dz(n)[i] v(n)[j] (R5).    */
        double *dA = (double *)calloc((size_t)M * M, sizeof(double));
        double *dB = (double *)calloc((size_t)M, sizeof(double));
        double *dC = (double *)calloc((size_t)M, sizeof(double));
        double dD = 0.0;
        if (!dA || !dB || !dC) return 2;
        for (long n = 0; n < N; ++n) {
            const double *vn = v + n * M;
            const double *dzn = dz + n * M;
            double dyn = gy ? gy[n] : 0.0;
            dD += dyn * x[n];
            for (int i = 0; i < M; ++i) {
                dC[i] += dyn * vn[i];
                dB[i] += dzn[i] * x[n];
                for (int j = 0; j < M; ++j) dA[IDX(i, j, M)] += dzn[i] * vn[j];
            }
        }
        /* Chain rule from (A_f, B_f, C_f, D) to the normalised b', a'.
         * DF : A_f[0][k-1] = -a'_k, C_f[k-1] = b'_k - a'_k b'_0, D = b'_0.
         * TDF: A_f[k-1][0] = -a'_k, B_f[k-1] = b'_k - a'_k b'_0, D = b'_0. */
        double *gbn = (double *)calloc((size_t)(M + 1), sizeof(double));
        double *gan = (double *)calloc((size_t)(M + 1), sizeof(double));
        const double *dc = (form == 0) ? dC : dB;   /* gradient w.r.t. c   */
        gbn[0] = dD;
        for (int k = 1; k <= M; ++k) {
            double dAk = (form == 0) ? dA[IDX(0, k - 1, M)] : dA[IDX(k - 1, 0, M)];
            gan[k] = -dAk - bn[0] * dc[k - 1];
            gbn[k] = dc[k - 1];
            gbn[0] += -an[k] * dc[k - 1];
        }
        /* Undo the a_0 normalisation b' = b / a0, a' = a / a0 (R8). */
        double s = 0.0;
        for (int k = 0; k <= M; ++k) s += bn[k] * gbn[k];
        for (int k = 1; k <= M; ++k) s += an[k] * gan[k];
        if (gb) for (int k = 0; k <= M; ++k) gb[k] = gbn[k] / a0;
        if (ga) {
            ga[0] = -s / a0;
            for (int k = 1; k <= M; ++k) ga[k] = gan[k] / a0;
        }
        free(dA); free(dB); free(dC); free(gbn); free(gan);
    }
    free(bn); free(an); free(Af); free(Bf); free(Cf); free(v); free(dz); free(tmp);
    return 0;
}

/*
 * orc_tv_allpole: one sequence of the time-varying all-pole DF filter
 * (reading R10), in the dense per-sample state-space form
 *   v(n) = [y(n-1) .. y(n-M)],  A(n) = companion(a(n)),  B = e1,
 *   C(n) = -a(n), D = 1:
 *   y(n) = C(n)^T v(n) + x(n),  v(n+1) = A(n) v(n) + B x(n),  v(0) = zi.
 * Backward = Eq.7 with time-varying matrices (reading R11):
 *   dz(N-1) = gzf,  dz(n) = A(n+1)^T dz(n+1) + C(n+1) dy(n+1),
 *   dx(n) = B^T dz(n) + dy(n),  dzi = A(0)^T dz(0) + C(0) dy(0),
 *   dA(n) = dz(n) v(n)^T,  dC(n) = dy(n) v(n)  =>
 *   ga[n][i-1] = -dA(n)[0][i-1] - dC(n)[i-1].
 *   a: (N, M) row-major, a[n*M + i-1] = a_i(n) (monic a_0 = 1 implied).
 * Outputs (NULL = skip): y[N], zf[M], gx[N], ga[N*M], gzi[M].
 */
int orc_tv_allpole(int M, long N, const double *a, const double *x,
                   const double *zi, const double *gy, const double *gzf,
                   double *y, double *zf, double *gx, double *ga, double *gzi)
{
    if (M < 1 || N < 1) return 1;
    double *v = (double *)malloc((size_t)(N + 1) * M * sizeof(double));
    double *dz = (double *)malloc((size_t)N * M * sizeof(double));
    double *A = (double *)malloc((size_t)M * M * sizeof(double));
    double *C = (double *)malloc((size_t)M * sizeof(double));
    if (!v || !dz || !A || !C) return 2;
    const double B0 = 1.0;              /* B = e1 */

#define BUILD_AC(n)                                                        \
    do {                                                                   \
        memset(A, 0, (size_t)M * M * sizeof(double));                     \
        for (int k = 1; k <= M; ++k) {                                     \
            A[IDX(0, k - 1, M)] = -a[(n) * M + (k - 1)];                   \
            C[k - 1] = -a[(n) * M + (k - 1)];                              \
        }                                                                  \
        for (int i = 1; i < M; ++i) A[IDX(i, i - 1, M)] = 1.0;             \
    } while (0)

    for (int i = 0; i < M; ++i) v[i] = zi ? zi[i] : 0.0;
    for (long n = 0; n < N; ++n) {
        BUILD_AC(n);
        const double *vn = v + n * M;
        double *vn1 = v + (n + 1) * M;
        double yn = x[n];
        for (int i = 0; i < M; ++i) yn += C[i] * vn[i];
        if (y) y[n] = yn;
        for (int i = 0; i < M; ++i) {
            double s = (i == 0 ? B0 : 0.0) * x[n];
            for (int j = 0; j < M; ++j) s += A[IDX(i, j, M)] * vn[j];
            vn1[i] = s;
        }
    }
    if (zf) for (int i = 0; i < M; ++i) zf[i] = v[N * M + i];

    for (int i = 0; i < M; ++i) dz[(N - 1) * M + i] = gzf ? gzf[i] : 0.0;
    for (long n = N - 2; n >= 0; --n) {
        BUILD_AC(n + 1);
        const double *d1 = dz + (n + 1) * M;
        double dy1 = gy ? gy[n + 1] : 0.0;
        for (int i = 0; i < M; ++i) {
            double s = C[i] * dy1;
            for (int j = 0; j < M; ++j) s += A[IDX(j, i, M)] * d1[j];
            dz[n * M + i] = s;
        }
    }
    if (gx)
        for (long n = 0; n < N; ++n) gx[n] = B0 * dz[n * M] + (gy ? gy[n] : 0.0);
    if (gzi) {
        BUILD_AC(0);
        double dy0 = gy ? gy[0] : 0.0;
        for (int i = 0; i < M; ++i) {
            double s = C[i] * dy0;
            for (int j = 0; j < M; ++j) s += A[IDX(j, i, M)] * dz[j];
            gzi[i] = s;
        }
    }
    if (ga)
        for (long n = 0; n < N; ++n) {
            double dyn = gy ? gy[n] : 0.0;
            for (int k = 1; k <= M; ++k) {
                double dA0k = dz[n * M + 0] * v[n * M + (k - 1)]; /* dA(n)[0][k-1] */
                double dCk = dyn * v[n * M + (k - 1)];            /* dC(n)[k-1]    */
                ga[n * M + (k - 1)] = -dA0k - dCk;
            }
        }
#undef BUILD_AC
    free(v); free(dz); free(A); free(C);
    return 0;
}

/*
 * orc_tv_df: one sequence of the general time-varying DF-II filter (SURVEY
 * 8(f) f2): per-sample numerator b(n) (M+1) and monic denominator a(n) (M),
 * row n applied at output time n (reading R10 extended to b):
 *     u(n) = x(n) - sum_{i=1..M} a_i(n) u(n-i),   y(n) = sum_{k=0..M} b_k(n) u(n-k),
 * u(-k) = zi[k-1], zf[k-1] = u(N-k).  Coded as the per-sample state space of
 * Eqs.4-5 with the DF realisation of PAPER.md:66 at every n:
 * A(n) = companion(a(n)), B = e1, C(n) = b(n)[1..M] - a(n) b_0(n), D(n) = b_0(n),
 * v(n) = [u(n-1) .. u(n-M)].  Backward: Eq.7 with A(n+1), C(n+1) (R11),
 * Eq.8 with D(n), and per sample dA(n) = dz(n) v(n)^T, dC(n) = dy(n) v(n),
 * dD(n) = dy(n) x(n) (Eqs.6, 9 before the sum over n), mapped to (b(n), a(n))
 * as in the LTI DF chain rule: gb_k(n) = dC(n)[k-1] (k >= 1),
 * gb_0(n) = dD(n) - sum_k a_k(n) dC(n)[k-1],
 * ga_k(n) = -dA(n)[0][k-1] - b_0(n) dC(n)[k-1].
 * b: N x (M+1), a: N x M, gb: N x (M+1), ga: N x M (row-major, per sample).
 */
int orc_tv_df(int M, long N, const double *b, const double *a, const double *x,
              const double *zi, const double *gy, const double *gzf,
              double *y, double *zf, double *gx, double *gb, double *ga, double *gzi)
{
    if (M < 1 || N < 1) return 1;
    double *v = (double *)malloc((size_t)(N + 1) * M * sizeof(double));
    double *dz = (double *)malloc((size_t)N * M * sizeof(double));
    double *A = (double *)malloc((size_t)M * M * sizeof(double));
    double *C = (double *)malloc((size_t)M * sizeof(double));
    if (!v || !dz || !A || !C) return 2;
    const int K = M + 1;

#define BUILD_ACD(n)                                                       \
    do {                                                                   \
        memset(A, 0, (size_t)M * M * sizeof(double));                     \
        for (int k = 1; k <= M; ++k) {                                     \
            A[IDX(0, k - 1, M)] = -a[(n) * M + (k - 1)];                   \
            C[k - 1] = b[(n) * K + k] - a[(n) * M + (k - 1)] * b[(n) * K]; \
        }                                                                  \
        for (int i = 1; i < M; ++i) A[IDX(i, i - 1, M)] = 1.0;             \
    } while (0)

    for (int i = 0; i < M; ++i) v[i] = zi ? zi[i] : 0.0;
    for (long n = 0; n < N; ++n) {                  /* Eqs.4-5 with A(n), C(n), D(n) */
        BUILD_ACD(n);
        const double D = b[n * K];
        const double *vn = v + n * M;
        double *vn1 = v + (n + 1) * M;
        double yn = D * x[n];
        for (int i = 0; i < M; ++i) yn += C[i] * vn[i];
        if (y) y[n] = yn;
        for (int i = 0; i < M; ++i) {
            double s = (i == 0 ? 1.0 : 0.0) * x[n];
            for (int j = 0; j < M; ++j) s += A[IDX(i, j, M)] * vn[j];
            vn1[i] = s;
        }
    }
    if (zf) for (int i = 0; i < M; ++i) zf[i] = v[N * M + i];

    for (int i = 0; i < M; ++i) dz[(N - 1) * M + i] = gzf ? gzf[i] : 0.0;   /* R4 */
    for (long n = N - 2; n >= 0; --n) {             /* Eq.7 */
        BUILD_ACD(n + 1);
        const double *d1 = dz + (n + 1) * M;
        const double dy1 = gy ? gy[n + 1] : 0.0;
        for (int i = 0; i < M; ++i) {
            double s = C[i] * dy1;
            for (int j = 0; j < M; ++j) s += A[IDX(j, i, M)] * d1[j];
            dz[n * M + i] = s;
        }
    }
    if (gx)                                         /* Eq.8: B^T dz(n) + D(n) dy(n) */
        for (long n = 0; n < N; ++n) gx[n] = dz[n * M] + b[n * K] * (gy ? gy[n] : 0.0);
    if (gzi) {                                      /* A.3 with A(0), C(0) */
        BUILD_ACD(0);
        const double dy0 = gy ? gy[0] : 0.0;
        for (int i = 0; i < M; ++i) {
            double s = C[i] * dy0;
            for (int j = 0; j < M; ++j) s += A[IDX(j, i, M)] * dz[j];
            gzi[i] = s;
        }
    }
    for (long n = 0; n < N; ++n) {                  /* per-sample Eqs.6, 9 -> (b(n), a(n)) */
        const double dyn = gy ? gy[n] : 0.0;
        const double dD = dyn * x[n];
        double gb0 = dD;
        for (int k = 1; k <= M; ++k) {
            const double dCk = dyn * v[n * M + (k - 1)];
            const double dA0k = dz[n * M + 0] * v[n * M + (k - 1)];
            if (gb) gb[n * K + k] = dCk;
            if (ga) ga[n * M + (k - 1)] = -dA0k - b[n * K] * dCk;
            gb0 -= a[n * M + (k - 1)] * dCk;
        }
        if (gb) gb[n * K] = gb0;
    }
#undef BUILD_ACD
    free(v); free(dz); free(A); free(C);
    return 0;
}

/*
 * orc_tv_tdf: one sequence of the general time-varying TDF-II filter (SURVEY
 * 8(f) f2, reading R20): the TDF realisation of PAPER.md:67-68 ("replacing A
 * with its transpose and swapping B and C") built from the coefficient rows of
 * sample n, i.e. the per-sample state space of Eqs.4-5 with
 *   A_f(n) = companion(a(n))^T,  B_f(n) = c(n) = b(n)[1..M] - a(n) b_0(n),
 *   C_f = e1,  D(n) = b_0(n);
 *   v(n+1) = A_f(n) v(n) + B_f(n) x(n),   y(n) = C_f^T v(n) + D(n) x(n),
 * v(0) = zi, zf = v(N) (the scipy lfilter TDF state when the rows are
 * constant).  Backward: Eq.7 with A_f(n+1), C_f (R11 in transposed form),
 * Eq.8 with B_f(n), D(n), A.3 with A_f(0); per sample dA_f(n) = dz(n) v(n)^T,
 * dB_f(n) = dz(n) x(n), dD(n) = dy(n) x(n) (Eqs.6, 9 before the sum over n),
 * mapped to (b(n), a(n)) as in the LTI TDF chain rule (A_f[k-1][0] = -a_k,
 * c_{k-1} = b_k - a_k b_0):
 *   gb_k(n) = dB_f(n)[k-1] (k >= 1),  gb_0(n) = dD(n) - sum_k a_k(n) dB_f(n)[k-1],
 *   ga_k(n) = -dA_f(n)[k-1][0] - b_0(n) dB_f(n)[k-1].
 * b: N x (M+1), a: N x M (monic), gb: N x (M+1), ga: N x M (row-major).
 */
int orc_tv_tdf(int M, long N, const double *b, const double *a, const double *x,
               const double *zi, const double *gy, const double *gzf,
               double *y, double *zf, double *gx, double *gb, double *ga, double *gzi)
{
    if (M < 1 || N < 1) return 1;
    double *v = (double *)malloc((size_t)(N + 1) * M * sizeof(double));
    double *dz = (double *)malloc((size_t)N * M * sizeof(double));
    double *Af = (double *)malloc((size_t)M * M * sizeof(double));
    double *Bf = (double *)malloc((size_t)M * sizeof(double));
    if (!v || !dz || !Af || !Bf) return 2;
    const int K = M + 1;

    /* the TDF matrices of sample n: A_f = A^T with A = companion(a(n)), B_f = c(n) */
#define BUILD_TDF(n)                                                       \
    do {                                                                   \
        double *A_ = (double *)calloc((size_t)M * M, sizeof(double));      \
        for (int k = 1; k <= M; ++k) {                                     \
            A_[IDX(0, k - 1, M)] = -a[(n) * M + (k - 1)];                  \
            Bf[k - 1] = b[(n) * K + k] - a[(n) * M + (k - 1)] * b[(n) * K];\
        }                                                                  \
        for (int i = 1; i < M; ++i) A_[IDX(i, i - 1, M)] = 1.0;            \
        for (int i = 0; i < M; ++i)                                        \
            for (int j = 0; j < M; ++j) Af[IDX(i, j, M)] = A_[IDX(j, i, M)];\
        free(A_);                                                          \
    } while (0)

    for (int i = 0; i < M; ++i) v[i] = zi ? zi[i] : 0.0;
    for (long n = 0; n < N; ++n) {                  /* Eqs.4-5 with A_f(n), B_f(n), D(n) */
        BUILD_TDF(n);
        const double *vn = v + n * M;
        double *vn1 = v + (n + 1) * M;
        const double yn = vn[0] + b[n * K] * x[n];  /* C_f = e1 */
        if (y) y[n] = yn;
        for (int i = 0; i < M; ++i) {
            double s = Bf[i] * x[n];
            for (int j = 0; j < M; ++j) s += Af[IDX(i, j, M)] * vn[j];
            vn1[i] = s;
        }
    }
    if (zf) for (int i = 0; i < M; ++i) zf[i] = v[N * M + i];

    for (int i = 0; i < M; ++i) dz[(N - 1) * M + i] = gzf ? gzf[i] : 0.0;   /* R4 */
    for (long n = N - 2; n >= 0; --n) {             /* Eq.7: dz(n) = A_f(n+1)^T dz(n+1) + C_f dy(n+1) */
        BUILD_TDF(n + 1);
        const double *d1 = dz + (n + 1) * M;
        const double dy1 = gy ? gy[n + 1] : 0.0;
        for (int i = 0; i < M; ++i) {
            double s = (i == 0 ? 1.0 : 0.0) * dy1;
            for (int j = 0; j < M; ++j) s += Af[IDX(j, i, M)] * d1[j];
            dz[n * M + i] = s;
        }
    }
    for (long n = 0; n < N; ++n) {                  /* Eq.8 and the per-sample Eqs.6, 9 */
        BUILD_TDF(n);
        const double dyn = gy ? gy[n] : 0.0;
        const double *dzn = dz + n * M;
        double bfd = 0.0;
        for (int i = 0; i < M; ++i) bfd += Bf[i] * dzn[i];
        if (gx) gx[n] = bfd + b[n * K] * dyn;
        double gb0 = dyn * x[n];                    /* dD(n) */
        for (int k = 1; k <= M; ++k) {
            const double dBk = dzn[k - 1] * x[n];   /* dB_f(n)[k-1] */
            const double dAk0 = dzn[k - 1] * v[n * M + 0];   /* dA_f(n)[k-1][0] */
            if (gb) gb[n * K + k] = dBk;
            if (ga) ga[n * M + (k - 1)] = -dAk0 - b[n * K] * dBk;
            gb0 -= a[n * M + (k - 1)] * dBk;
        }
        if (gb) gb[n * K] = gb0;
    }
    if (gzi) {                                      /* A.3 with A_f(0), C_f */
        BUILD_TDF(0);
        const double dy0 = gy ? gy[0] : 0.0;
        for (int i = 0; i < M; ++i) {
            double s = (i == 0 ? 1.0 : 0.0) * dy0;
            for (int j = 0; j < M; ++j) s += Af[IDX(j, i, M)] * dz[j];
            gzi[i] = s;
        }
    }
#undef BUILD_TDF
    free(v); free(dz); free(Af); free(Bf);
    return 0;
}

/*
 * orc_recurrence: the bare recurrence of Listing 1,
 * v(n+1) = A v(n) + z(n) for a general dense A (M x M, row-major), with its
 * VJP: given gv (dL/dv(1..N), (N, M)), returns
 *   gz(n) = dL/dz(n) by Eq.7 run on z (dz(N-1) = gv(N)),
 *   gv0  = A^T gz(0),  gA = sum_n gz(n) v(n)^T (v(n) = v0 for n = 0).
 * Outputs (NULL = skip): v[N*M] (= v(1..N)), gz[N*M], gv0[M], gA[M*M].
 */
int orc_recurrence(int M, long N, const double *A, const double *v0,
                   const double *z, const double *gv, double *v, double *gz,
                   double *gv0, double *gA)
{
    if (M < 1 || N < 1) return 1;
    double *vv = (double *)malloc((size_t)(N + 1) * M * sizeof(double));
    double *g = (double *)malloc((size_t)N * M * sizeof(double));
    if (!vv || !g) return 2;
    for (int i = 0; i < M; ++i) vv[i] = v0 ? v0[i] : 0.0;
    for (long n = 0; n < N; ++n)
        for (int i = 0; i < M; ++i) {
            double s = z[n * M + i];
            for (int j = 0; j < M; ++j) s += A[IDX(i, j, M)] * vv[n * M + j];
            vv[(n + 1) * M + i] = s;
        }
    if (v) memcpy(v, vv + M, (size_t)N * M * sizeof(double));
    /* v(n+1) depends on z(n): dL/dz(n) = gv(n+1) + A^T dL/dz(n+1). */
    for (int i = 0; i < M; ++i) g[(N - 1) * M + i] = gv ? gv[(N - 1) * M + i] : 0.0;
    for (long n = N - 2; n >= 0; --n)
        for (int i = 0; i < M; ++i) {
            double s = gv ? gv[n * M + i] : 0.0;
            for (int j = 0; j < M; ++j) s += A[IDX(j, i, M)] * g[(n + 1) * M + j];
            g[n * M + i] = s;
        }
    if (gz) memcpy(gz, g, (size_t)N * M * sizeof(double));
    if (gv0)
        for (int i = 0; i < M; ++i) {
            double s = 0.0;
            for (int j = 0; j < M; ++j) s += A[IDX(j, i, M)] * g[j];
            gv0[i] = s;
        }
    if (gA) {
        for (int i = 0; i < M * M; ++i) gA[i] = 0.0;
        for (long n = 0; n < N; ++n)
            for (int i = 0; i < M; ++i)
                for (int j = 0; j < M; ++j)
                    gA[IDX(i, j, M)] += g[n * M + i] * vv[n * M + j];
    }
    free(vv); free(g);
    return 0;
}
