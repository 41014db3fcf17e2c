/*
 * oracle/frob_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for Frobenius inversion of complex
 * matrices (Dai, Lim & Ye, arXiv 2208.01239).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path in
 * paper_2208_01239_b200/csrc, and the CUDA path never calls it.
 *
 * Everything is IEEE fp64, row-major, planar (real part and imaginary part in two
 * separate n*n arrays, leading dimension n).  Compiled with -ffp-contract=off so
 * every multiply and add rounds separately; OpenMP only splits independent rows or
 * columns, so the rounding order of every entry is fixed and independent of the
 * thread count.
 *
 * Paper passages followed (P:Lxxx = line of the paper's LaTeX source):
 *   or_dgetrf        Alg 3 line 1 "compute LU factorization of A = LU", partial
 *                    pivoting, first index of max |a_ik| (LAPACK idamax convention).
 *   or_dtrtri_upper  Alg 3 line 2 "compute U^{-1}" by column substitutions
 *                    ("inverting a triangular matrix can be done by a sequence of ...
 *                    substitutions", proof of Thm 5.1).
 *   or_dgetri_solve  Alg 3 line 3 "solve for X from XL = U^{-1}", then the column
 *                    interchanges that undo P (A = P^T L U  =>  A^{-1} = U^{-1} L^{-1} P).
 *   or_dinv          Alg 3 = the real inversion inv_{n,R} used twice by Alg 1.
 *   or_dgemm         m_{n,R}: C = A B, plain triple loop, k ascending.
 *   or_dpotrf_upper  Alg 10 Cholesky; or_hpd_frob_inv Alg 6;
 *   or_zhpd_inv_chol Alg 8 complex Cholesky inversion
 *   or_frob_inv_rand Alg 5 randomized Frobenius inversion, mu given
 *   or_frob_inv      Alg 1 "Frobenius inversion I" with tau = 1 (f = x^2+1,
 *                    P:L123): S1 branch returns J - iK, S2 branch returns K - iJ.  The
 *                    numerical branch choice (the paper's S1/S2 are algebraic)
 *                    follows DESIGN.md reading R1' (kappa_inf of the part, Thm 5.2).
 *   or_zinv_gj       The plain definition: complex Gauss-Jordan inverse with partial
 *                    pivoting on |re|+|im| (the object Lemma 4.1, reaches exactly).
 *   or_zinv_lu       Alg 3 applied over C (the paper's comparator).
 *   or_zgetrf        Alg 3 line 1 over C on its own; or_zgetrs solves Z Y = R or
 *                    Z^H Y = R with its factors -- the plain definition of Z^{-1} R used for
 *                    sketch parity at n >= 8192 (the object Lemma 4.1 reaches, applied to R).
 *   or_frob_inv_many or_frob_inv on independent matrices (config 3 full-set parity).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_EPS 1.1102230246251565e-16 /* u = 2^-53, unit roundoff of fp64 */

/* ------------------------------------------------------------------ real */

/* LU with partial pivoting, in place.  On return a holds L (strict lower, unit
 * diagonal implied) and U (upper); ipiv[k] = row swapped with row k at step k
 * (0-based, LAPACK order).  Returns 0 or the 1-based index of the first exactly
 * zero pivot (elimination of that column is skipped, as LAPACK does). */
int or_dgetrf(int n, double *a, int *ipiv)
{
    int info = 0;
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = fabs(a[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            double v = fabs(a[(size_t)i * n + k]);
            if (v > best) { best = v; p = i; }
        }
        ipiv[k] = p;
        if (p != k) {
            for (int j = 0; j < n; ++j) {
                double t = a[(size_t)k * n + j];
                a[(size_t)k * n + j] = a[(size_t)p * n + j];
                a[(size_t)p * n + j] = t;
            }
        }
        double piv = a[(size_t)k * n + k];
        if (piv == 0.0) { if (!info) info = k + 1; continue; }
        #pragma omp parallel for schedule(static) if (n - k > 256)
        for (int i = k + 1; i < n; ++i) {
            double l = a[(size_t)i * n + k] / piv;
            a[(size_t)i * n + k] = l;
            for (int j = k + 1; j < n; ++j)
                a[(size_t)i * n + j] = a[(size_t)i * n + j] - l * a[(size_t)k * n + j];
        }
    }
    return info;
}

/* X = U^{-1} for the upper triangle U of lu (out of place, X full n*n with zeros
 * below the diagonal).  Column j solves U x = e_j by back substitution. */
int or_dtrtri_upper(int n, const double *lu, double *x)
{
    for (int j = 0; j < n; ++j)
        if (lu[(size_t)j * n + j] == 0.0) return j + 1;
    double *xt = (double *)malloc(sizeof(double) * (size_t)n * n); /* xt[j*n+i] = X[i][j] */
    #pragma omp parallel for schedule(dynamic, 8) if (n > 128)
    for (int j = 0; j < n; ++j) {
        double *col = xt + (size_t)j * n;
        for (int i = j + 1; i < n; ++i) col[i] = 0.0;
        col[j] = 1.0 / lu[(size_t)j * n + j];
        for (int i = j - 1; i >= 0; --i) {
            double s = 0.0;
            for (int k = i + 1; k <= j; ++k) s = s + lu[(size_t)i * n + k] * col[k];
            col[i] = -s / lu[(size_t)i * n + i];
        }
    }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) x[(size_t)i * n + j] = xt[(size_t)j * n + i];
    free(xt);
    return 0;
}

/* Solve X L = W for X (L = unit lower triangle of lu), column j from n-1 down to 0:
 * X[:,j] = W[:,j] - sum_{k>j} X[:,k] L[k][j].  Rows are independent. */
void or_dgetri_solve(int n, const double *lu, const double *w, double *x)
{
    double *lt = (double *)malloc(sizeof(double) * (size_t)n * n); /* lt[j*n+k] = L[k][j] */
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j) lt[(size_t)j * n + k] = lu[(size_t)k * n + j];
    #pragma omp parallel for schedule(static) if (n > 128)
    for (int i = 0; i < n; ++i) {
        double *xi = x + (size_t)i * n;
        const double *wi = w + (size_t)i * n;
        for (int j = n - 1; j >= 0; --j) {
            double s = 0.0;
            const double *lj = lt + (size_t)j * n;
            for (int k = j + 1; k < n; ++k) s = s + xi[k] * lj[k];
            xi[j] = wi[j] - s;
        }
    }
    free(lt);
}

/* A^{-1} = X P: undo the row interchanges as column interchanges, last first. */
void or_col_unswap(int n, double *x, const int *ipiv)
{
    for (int k = n - 1; k >= 0; --k) {
        int p = ipiv[k];
        if (p == k) continue;
        for (int i = 0; i < n; ++i) {
            double t = x[(size_t)i * n + k];
            x[(size_t)i * n + k] = x[(size_t)i * n + p];
            x[(size_t)i * n + p] = t;
        }
    }
}

static double max_abs(size_t cnt, const double *v)
{
    double m = 0.0;
    for (size_t i = 0; i < cnt; ++i) { double t = fabs(v[i]); if (t > m) m = t; }
    return m;
}

/* Pivot diagnostics of an LU: rho = max|u_ii| / min|u_ii| and the singularity test
 * |u_kk| < 100*n*u*max_i|u_ii| (reading R2); xmax is unused (kept for the
 * ABI of the helper). */
static void pivot_diag(int n, const double *lu, double xmax, double *rho, int *singular_col)
{
    double mx = 0.0, mn = INFINITY;
    int sc = 0;
    (void)xmax;
    for (int i = 0; i < n; ++i) {
        double d = fabs(lu[(size_t)i * n + i]);
        if (d > mx) mx = d;
        if (d < mn) mn = d;
    }
    double thr = 100.0 * (double)n * ORACLE_EPS * mx;
    for (int i = 0; i < n; ++i) {
        double d = fabs(lu[(size_t)i * n + i]);
        if (!(d >= thr) || d == 0.0) { sc = i + 1; break; }
    }
    *rho = (mn > 0.0) ? mx / mn : INFINITY;
    *singular_col = sc;
}

/* Alg 3: A^{-1} via LU.  ainv receives the inverse.  Returns 0 or 1-based singular
 * pivot column; *rho receives the pivot ratio. */
int or_dinv(int n, const double *a, double *ainv, double *rho)
{
    double *lu = (double *)malloc(sizeof(double) * (size_t)n * n);
    double *w = (double *)malloc(sizeof(double) * (size_t)n * n);
    int *ipiv = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    memcpy(lu, a, sizeof(double) * (size_t)n * n);
    or_dgetrf(n, lu, ipiv);
    int sc;
    double r;
    pivot_diag(n, lu, max_abs((size_t)n * n, a), &r, &sc);
    if (rho) *rho = r;
    int info = sc;
    if (!info) {
        or_dtrtri_upper(n, lu, w);
        or_dgetri_solve(n, lu, w, ainv);
        or_col_unswap(n, ainv, ipiv);
    }
    free(lu); free(w); free(ipiv);
    return info;
}

/* C = A B (m x k times k x n); C[i][j] = sum_{k ascending} A[i][k] B[k][j]. */
void or_dgemm(int m, int n, int k, const double *a, const double *b, double *c)
{
    #pragma omp parallel for schedule(static) if ((long)m * n * k > 2000000L)
    for (int i = 0; i < m; ++i) {
        double *ci = c + (size_t)i * n;
        for (int j = 0; j < n; ++j) ci[j] = 0.0;
        for (int q = 0; q < k; ++q) {
            double aiq = a[(size_t)i * k + q];
            const double *bq = b + (size_t)q * n;
            for (int j = 0; j < n; ++j) ci[j] = ci[j] + aiq * bq[j];
        }
    }
}

/* ||A||_inf = max_i sum_j |a_ij| (j ascending) */
static double norm_inf(int n, const double *a)
{
    double m = 0.0;
    for (int i = 0; i < n; ++i) {
        double r = 0.0;
        for (int j = 0; j < n; ++j) r = r + fabs(a[(size_t)i * n + j]);
        if (r > m) m = r;
    }
    return m;
}

/* Alg 1 with tau = 1.
 *   branch: 0 = AUTO (reading R1'), 1 = S1 (X=A, Y=B), 2 = S2 (X=B, Y=A).
 *   kappa_sw: AUTO switch threshold on kappa_inf(X) / sqrt(n), kappa_inf(X) = ||X||_inf ||X^{-1}||_inf.
 * AUTO (R1'): invert A (line "compute X^{-1}" with X = A); keep S1 unless A is singular (R2) or
 * kappa_inf(A) / sqrt(n) > kappa_sw (an O(1)-accurate stand-in for kappa_2(A) of a dense matrix) -- the leading term of the Thm 5.2 bound is
 * |X^{-1}| |L_X| |U_X| |X^{-1}| |Y| |J|, i.e. the error grows with the conditioning of X; then
 * also invert B and keep the branch whose part has the smaller kappa_inf (the computed inverse
 * of the chosen part is used as "X^{-1}").
 * Returns 0 ok, 1 singular (out[0] = 1-based column), 2 both parts singular.
 * out[0]=info, out[1]=branch used (1|2); rho[0..3] = rho_A, rho_B (pivot ratios), kappa_inf(A),
 * kappa_inf(B) (NaN where that part was not factored / inverted). */
int or_frob_inv(int n, const double *A, const double *B, double *Xre, double *Xim,
                int branch, double kappa_sw, int *out, double *rho)
{
    size_t nn = (size_t)n * n;
    double *Xinv = (double *)malloc(sizeof(double) * nn);
    double *Xinv2 = (double *)malloc(sizeof(double) * nn);
    double *F = (double *)malloc(sizeof(double) * nn);
    double *G = (double *)malloc(sizeof(double) * nn);
    double *J = (double *)malloc(sizeof(double) * nn);
    double *K = (double *)malloc(sizeof(double) * nn);
    int use = branch, info = 0;
    rho[0] = rho[1] = rho[2] = rho[3] = NAN;
    if (branch == 0) {
        int ia = or_dinv(n, A, Xinv, &rho[0]);          /* compute X^{-1}, X = A            */
        double ka = ia ? INFINITY : norm_inf(n, A) * norm_inf(n, Xinv);
        rho[2] = ka;
        use = 1;
        if (ia || !(ka <= kappa_sw * sqrt((double)n))) {
            int ib = or_dinv(n, B, Xinv2, &rho[1]);     /* compute X^{-1}, X = B            */
            double kb = ib ? INFINITY : norm_inf(n, B) * norm_inf(n, Xinv2);
            rho[3] = kb;
            if (ia && ib) { out[0] = ia; out[1] = 0; info = -1; goto done; }
            if (ia || (!ib && kb < ka)) {
                double *t = Xinv; Xinv = Xinv2; Xinv2 = t;
                use = 2;
            }
        }
    } else {
        double rx;
        info = or_dinv(n, use == 1 ? A : B, Xinv, &rx);  /* compute X^{-1}                 */
        rho[use == 1 ? 0 : 1] = rx;
        if (info) { out[0] = info; out[1] = use; goto done; }
        rho[use == 1 ? 2 : 3] = norm_inf(n, use == 1 ? A : B) * norm_inf(n, Xinv);
    }
    out[1] = use;
    {
        const double *X = (use == 1) ? A : B;   /* line 2 / line 4 of Alg 1 */
        const double *Y = (use == 1) ? B : A;
        or_dgemm(n, n, n, Xinv, Y, F);                 /* compute X^{-1} Y               */
        or_dgemm(n, n, n, Y, F, G);                    /* compute Y X^{-1} Y             */
        for (size_t i = 0; i < nn; ++i) G[i] = X[i] + G[i]; /* tau1 X + tau2 Y X^{-1} Y    */
        info = or_dinv(n, G, J, NULL);                 /* J = (tau1 X + tau2 Y X^-1 Y)^-1 */
        if (info) { out[0] = info; goto done; }
        or_dgemm(n, n, n, F, J, K);                    /* K = X^{-1} Y J                 */
        if (use == 1) {                                /* return J - iK                  */
            for (size_t i = 0; i < nn; ++i) { Xre[i] = J[i]; Xim[i] = -K[i]; }
        } else {                                       /* return K - iJ                  */
            for (size_t i = 0; i < nn; ++i) { Xre[i] = K[i]; Xim[i] = -J[i]; }
        }
        out[0] = 0;
    }
done:
    free(Xinv); free(Xinv2); free(F); free(G); free(J); free(K);
    return info < 0 ? 2 : (info ? 1 : 0);
}

/* Alg 5 "randomized Frobenius inversion", mu supplied by the caller (line 1 draws
 * it from [0,1]; random numbers are inputs here).
 *   line 2: X = A - mu B, Y = mu A + B
 *   line 3: W = (X + iY)^{-1} by Alg 1 (AUTO branch rule, R1)
 *   line 4: W1 = Re W, W2 = Im W
 *   line 5: Z^{-1} = (W1 - mu W2) + i (mu W1 + W2)
 * Returns the status of the inner Alg 1 call (out / rho as there). */
int or_frob_inv_rand(int n, const double *A, const double *B, double mu, double *Xre, double *Xim,
                     double kappa_sw, int *out, double *rho)
{
    size_t nn = (size_t)n * n;
    double *X = (double *)malloc(sizeof(double) * nn);
    double *Y = (double *)malloc(sizeof(double) * nn);
    double *W1 = (double *)malloc(sizeof(double) * nn);
    double *W2 = (double *)malloc(sizeof(double) * nn);
    for (size_t i = 0; i < nn; ++i) {           /* line 2 */
        X[i] = A[i] - mu * B[i];
        Y[i] = mu * A[i] + B[i];
    }
    int st = or_frob_inv(n, X, Y, W1, W2, 0, kappa_sw, out, rho);   /* lines 3-4 */
    if (st == 0) {
        for (size_t i = 0; i < nn; ++i) {       /* line 5 */
            Xre[i] = W1[i] - mu * W2[i];
            Xim[i] = mu * W1[i] + W2[i];
        }
    }
    free(X); free(Y); free(W1); free(W2);
    return st;
}

/* --------------------------------------------------------------- HPD (Section 6) */

/* Alg 10 "Cholesky decomposition", real case, column by column:
 *   Z[1:k-1,k] = (Z[1:k-1,1:k-1]^T)^{-1} Z[1:k-1,k]        (forward substitution)
 *   Z[k,k]     = sqrt(Z[k,k] - Z[1:k-1,k]^T Z[1:k-1,k])
 * on the upper triangle of a; u (n x n) receives U with A = U^T U (zeros below).
 * Returns 0, or the 1-based column whose pivot is not positive. */
int or_dpotrf_upper(int n, const double *a, double *u)
{
    size_t nn = (size_t)n * n;
    for (size_t i = 0; i < nn; ++i) u[i] = 0.0;
    for (int k = 0; k < n; ++k) {
        for (int i = 0; i < k; ++i) {                 /* forward substitution with U^T */
            double s = a[(size_t)i * n + k];
            for (int q = 0; q < i; ++q) s -= u[(size_t)q * n + i] * u[(size_t)q * n + k];
            u[(size_t)i * n + k] = s / u[(size_t)i * n + i];
        }
        double d = a[(size_t)k * n + k];
        for (int q = 0; q < k; ++q) d -= u[(size_t)q * n + k] * u[(size_t)q * n + k];
        if (!(d > 0.0)) return k + 1;
        u[(size_t)k * n + k] = sqrt(d);
    }
    return 0;
}

/* X = U^{-T} Y for upper U: forward substitution per column of Y (U^T X = Y) */
static void fwd_ut(int n, const double *u, const double *y, double *x)
{
    for (int c = 0; c < n; ++c)
        for (int i = 0; i < n; ++i) {
            double s = y[(size_t)i * n + c];
            for (int q = 0; q < i; ++q) s -= u[(size_t)q * n + i] * x[(size_t)q * n + c];
            x[(size_t)i * n + c] = s / u[(size_t)i * n + i];
        }
}
/* X = U^{-1} Y for upper U: back substitution per column of Y */
static void back_u(int n, const double *u, const double *y, double *x)
{
    for (int c = 0; c < n; ++c)
        for (int i = n - 1; i >= 0; --i) {
            double s = y[(size_t)i * n + c];
            for (int q = i + 1; q < n; ++q) s -= u[(size_t)i * n + q] * x[(size_t)q * n + c];
            x[(size_t)i * n + c] = s / u[(size_t)i * n + i];
        }
}
static void transpose(int n, const double *a, double *t)
{
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) t[(size_t)j * n + i] = a[(size_t)i * n + j];
}

/* Alg 6 "first variant of Frobenius inversion" for HPD Z = A + iB (Lemma 6.1:
 * Z is in S1, so X = A, Y = B):
 *   l.6  X = U^T U            l.7  K1 = (U^T)^{-1} Y      l.8  K2 = U^{-1} K1
 *   l.9  K3 = K1^T K1         l.10 K4 = X - K3            l.11 K4 = V^T V
 *   l.12 K5 = V^{-1}          l.13 K6 = K5 K5^T           l.14 K7 = K2 K6
 *   return K6 - i K7.
 * Returns 0, or 1 (U) / 2 (V) when a Cholesky pivot is not positive (out_col: column). */
int or_hpd_frob_inv(int n, const double *A, const double *B, double *Xre, double *Xim, int *out_col)
{
    size_t nn = (size_t)n * n;
    double *U = (double *)malloc(sizeof(double) * nn), *K1 = (double *)malloc(sizeof(double) * nn);
    double *K2 = (double *)malloc(sizeof(double) * nn), *T = (double *)malloc(sizeof(double) * nn);
    double *K4 = (double *)malloc(sizeof(double) * nn), *V = (double *)malloc(sizeof(double) * nn);
    double *K5 = (double *)malloc(sizeof(double) * nn), *K6 = (double *)malloc(sizeof(double) * nn);
    int st = 0, c;
    if ((c = or_dpotrf_upper(n, A, U))) { st = 1; *out_col = c; goto done; }      /* l.6  */
    fwd_ut(n, U, B, K1);                                                           /* l.7  */
    back_u(n, U, K1, K2);                                                          /* l.8  */
    transpose(n, K1, T);
    or_dgemm(n, n, n, T, K1, K4);                                                  /* l.9  */
    for (size_t i = 0; i < nn; ++i) K4[i] = A[i] - K4[i];                          /* l.10 */
    if ((c = or_dpotrf_upper(n, K4, V))) { st = 2; *out_col = c; goto done; }      /* l.11 */
    if (or_dtrtri_upper(n, V, K5)) { st = 2; *out_col = 0; goto done; }           /* l.12 */
    transpose(n, K5, T);
    or_dgemm(n, n, n, K5, T, K6);                                                  /* l.13 */
    or_dgemm(n, n, n, K2, K6, T);                                                  /* l.14 */
    for (size_t i = 0; i < nn; ++i) { Xre[i] = K6[i]; Xim[i] = -T[i]; }            /* K6 - iK7 */
    *out_col = 0;
done:
    free(U); free(K1); free(K2); free(T); free(K4); free(V); free(K5); free(K6);
    return st;
}

/* Alg 8 "first matrix inversion via Cholesky decomposition" over C:
 * Z = U^H U (Alg 10 with conjugates), K = U^{-1}, X = K K^H.  Returns 0 or the 1-based
 * column of a non-positive pivot. */
int or_zhpd_inv_chol(int n, const double *zr, const double *zi, double *xr, double *xi)
{
    size_t nn = (size_t)n * n;
    double *ur = (double *)calloc(nn, sizeof(double)), *ui = (double *)calloc(nn, sizeof(double));
    double *kr = (double *)calloc(nn, sizeof(double)), *ki = (double *)calloc(nn, sizeof(double));
    int st = 0;
    for (int k = 0; k < n && !st; ++k) {
        for (int i = 0; i < k; ++i) {     /* U[i][k] = (z[i][k] - sum_q conj(U[q][i]) U[q][k]) / U[i][i] */
            double sr = zr[(size_t)i * n + k], si = zi[(size_t)i * n + k];
            for (int q = 0; q < i; ++q) {
                const double ar = ur[(size_t)q * n + i], ai = -ui[(size_t)q * n + i];
                const double br = ur[(size_t)q * n + k], bi = ui[(size_t)q * n + k];
                sr -= ar * br - ai * bi;
                si -= ar * bi + ai * br;
            }
            const double d = ur[(size_t)i * n + i];  /* real, positive */
            ur[(size_t)i * n + k] = sr / d;
            ui[(size_t)i * n + k] = si / d;
        }
        double d = zr[(size_t)k * n + k];
        for (int q = 0; q < k; ++q)
            d -= ur[(size_t)q * n + k] * ur[(size_t)q * n + k] + ui[(size_t)q * n + k] * ui[(size_t)q * n + k];
        if (!(d > 0.0)) { st = k + 1; break; }
        ur[(size_t)k * n + k] = sqrt(d);
    }
    if (!st) {
        /* K = U^{-1}: column j by back substitution, U K[:, j] = e_j */
        for (int j = 0; j < n; ++j)
            for (int i = j; i >= 0; --i) {
                double sr = (i == j) ? 1.0 : 0.0, si = 0.0;
                for (int q = i + 1; q <= j; ++q) {
                    const double ar = ur[(size_t)i * n + q], ai = ui[(size_t)i * n + q];
                    const double br = kr[(size_t)q * n + j], bi = ki[(size_t)q * n + j];
                    sr -= ar * br - ai * bi;
                    si -= ar * bi + ai * br;
                }
                const double d = ur[(size_t)i * n + i];
                kr[(size_t)i * n + j] = sr / d;
                ki[(size_t)i * n + j] = si / d;
            }
        /* X = K K^H */
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) {
                double sr = 0.0, si = 0.0;
                for (int q = 0; q < n; ++q) {
                    const double ar = kr[(size_t)i * n + q], ai = ki[(size_t)i * n + q];
                    const double br = kr[(size_t)j * n + q], bi = -ki[(size_t)j * n + q];
                    sr += ar * br - ai * bi;
                    si += ar * bi + ai * br;
                }
                xr[(size_t)i * n + j] = sr;
                xi[(size_t)i * n + j] = si;
            }
    }
    free(ur); free(ui); free(kr); free(ki);
    return st;
}

/* --------------------------------------------------------------- complex */

static double cabs1(double re, double im) { return fabs(re) + fabs(im); }

/* Complex Gauss-Jordan inverse with partial pivoting (first max of |re|+|im|), in
 * place on (re, im).  Returns 0 or the 1-based column of an exactly zero pivot. */
int or_zinv_gj(int n, double *re, double *im)
{
    int *piv = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    int info = 0;
    for (int k = 0; k < n && !info; ++k) {
        int p = k;
        double best = cabs1(re[(size_t)k * n + k], im[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            double v = cabs1(re[(size_t)i * n + k], im[(size_t)i * n + k]);
            if (v > best) { best = v; p = i; }
        }
        piv[k] = p;
        if (best == 0.0) { info = k + 1; break; }
        if (p != k) {
            for (int j = 0; j < n; ++j) {
                double t = re[(size_t)k * n + j]; re[(size_t)k * n + j] = re[(size_t)p * n + j]; re[(size_t)p * n + j] = t;
                t = im[(size_t)k * n + j]; im[(size_t)k * n + j] = im[(size_t)p * n + j]; im[(size_t)p * n + j] = t;
            }
        }
        /* 1/p = conj(p) / |p|^2 */
        double pr = re[(size_t)k * n + k], pi = im[(size_t)k * n + k];
        double den = pr * pr + pi * pi;
        double ir = pr / den, ii = -pi / den;
        re[(size_t)k * n + k] = 1.0; im[(size_t)k * n + k] = 0.0;
        for (int j = 0; j < n; ++j) {
            double xr = re[(size_t)k * n + j], xi = im[(size_t)k * n + j];
            re[(size_t)k * n + j] = xr * ir - xi * ii;
            im[(size_t)k * n + j] = xr * ii + xi * ir;
        }
        #pragma omp parallel for schedule(static) if (n > 256)
        for (int i = 0; i < n; ++i) {
            if (i == k) continue;
            double fr = re[(size_t)i * n + k], fi = im[(size_t)i * n + k];
            re[(size_t)i * n + k] = 0.0; im[(size_t)i * n + k] = 0.0;
            if (fr == 0.0 && fi == 0.0) continue;
            for (int j = 0; j < n; ++j) {
                double xr = re[(size_t)k * n + j], xi = im[(size_t)k * n + j];
                re[(size_t)i * n + j] = re[(size_t)i * n + j] - (fr * xr - fi * xi);
                im[(size_t)i * n + j] = im[(size_t)i * n + j] - (fr * xi + fi * xr);
            }
        }
    }
    if (!info) {
        for (int k = n - 1; k >= 0; --k) {
            int p = piv[k];
            if (p == k) continue;
            for (int i = 0; i < n; ++i) {
                double t = re[(size_t)i * n + k]; re[(size_t)i * n + k] = re[(size_t)i * n + p]; re[(size_t)i * n + p] = t;
                t = im[(size_t)i * n + k]; im[(size_t)i * n + k] = im[(size_t)i * n + p]; im[(size_t)i * n + p] = t;
            }
        }
    }
    free(piv);
    return info;
}

/* Alg 3 over C (the comparator): complex LU with partial pivoting (|re|+|im|), U^{-1}
 * by column substitution, solve X L = U^{-1}, undo interchanges.  Out of place.
 * Returns 0 or 1-based zero-pivot column. */
int or_zinv_lu(int n, const double *zr, const double *zi, double *xr, double *xi)
{
    size_t nn = (size_t)n * n;
    double *ar = (double *)malloc(sizeof(double) * nn), *ai = (double *)malloc(sizeof(double) * nn);
    double *wr = (double *)malloc(sizeof(double) * nn), *wi = (double *)malloc(sizeof(double) * nn);
    int *ipiv = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    memcpy(ar, zr, sizeof(double) * nn);
    memcpy(ai, zi, sizeof(double) * nn);
    int info = 0;
    /* line 1: LU */
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = cabs1(ar[(size_t)k * n + k], ai[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            double v = cabs1(ar[(size_t)i * n + k], ai[(size_t)i * n + k]);
            if (v > best) { best = v; p = i; }
        }
        ipiv[k] = p;
        if (p != k) {
            for (int j = 0; j < n; ++j) {
                double t = ar[(size_t)k * n + j]; ar[(size_t)k * n + j] = ar[(size_t)p * n + j]; ar[(size_t)p * n + j] = t;
                t = ai[(size_t)k * n + j]; ai[(size_t)k * n + j] = ai[(size_t)p * n + j]; ai[(size_t)p * n + j] = t;
            }
        }
        double pr = ar[(size_t)k * n + k], pi = ai[(size_t)k * n + k];
        if (pr == 0.0 && pi == 0.0) { if (!info) info = k + 1; continue; }
        double den = pr * pr + pi * pi;
        double ir = pr / den, ii = -pi / den;
        #pragma omp parallel for schedule(static) if (n - k > 256)
        for (int i = k + 1; i < n; ++i) {
            double vr = ar[(size_t)i * n + k], vi = ai[(size_t)i * n + k];
            double lr = vr * ir - vi * ii, li = vr * ii + vi * ir;
            ar[(size_t)i * n + k] = lr; ai[(size_t)i * n + k] = li;
            for (int j = k + 1; j < n; ++j) {
                double ur = ar[(size_t)k * n + j], ui = ai[(size_t)k * n + j];
                ar[(size_t)i * n + j] = ar[(size_t)i * n + j] - (lr * ur - li * ui);
                ai[(size_t)i * n + j] = ai[(size_t)i * n + j] - (lr * ui + li * ur);
            }
        }
    }
    if (info) goto done;
    /* line 2: W = U^{-1}, column j by back substitution */
    #pragma omp parallel for schedule(dynamic, 8) if (n > 128)
    for (int j = 0; j < n; ++j) {
        for (int i = j + 1; i < n; ++i) { wr[(size_t)i * n + j] = 0.0; wi[(size_t)i * n + j] = 0.0; }
        double ur = ar[(size_t)j * n + j], ui = ai[(size_t)j * n + j];
        double den = ur * ur + ui * ui;
        wr[(size_t)j * n + j] = ur / den; wi[(size_t)j * n + j] = -ui / den;
        for (int i = j - 1; i >= 0; --i) {
            double sr = 0.0, si = 0.0;
            for (int k = i + 1; k <= j; ++k) {
                double a_r = ar[(size_t)i * n + k], a_i = ai[(size_t)i * n + k];
                double b_r = wr[(size_t)k * n + j], b_i = wi[(size_t)k * n + j];
                sr = sr + (a_r * b_r - a_i * b_i);
                si = si + (a_r * b_i + a_i * b_r);
            }
            double dr = ar[(size_t)i * n + i], di = ai[(size_t)i * n + i];
            double dd = dr * dr + di * di;
            /* -s / d = -s * conj(d) / |d|^2 */
            wr[(size_t)i * n + j] = -(sr * dr + si * di) / dd;
            wi[(size_t)i * n + j] = -(si * dr - sr * di) / dd;
        }
    }
    /* line 3: solve X L = W, rows independent, column j from n-1 down */
    #pragma omp parallel for schedule(static) if (n > 128)
    for (int i = 0; i < n; ++i) {
        for (int j = n - 1; j >= 0; --j) {
            double sr = 0.0, si = 0.0;
            for (int k = j + 1; k < n; ++k) {
                double x_r = xr[(size_t)i * n + k], x_i = xi[(size_t)i * n + k];
                double l_r = ar[(size_t)k * n + j], l_i = ai[(size_t)k * n + j];
                sr = sr + (x_r * l_r - x_i * l_i);
                si = si + (x_r * l_i + x_i * l_r);
            }
            xr[(size_t)i * n + j] = wr[(size_t)i * n + j] - sr;
            xi[(size_t)i * n + j] = wi[(size_t)i * n + j] - si;
        }
    }
    for (int k = n - 1; k >= 0; --k) {
        int p = ipiv[k];
        if (p == k) continue;
        for (int i = 0; i < n; ++i) {
            double t = xr[(size_t)i * n + k]; xr[(size_t)i * n + k] = xr[(size_t)i * n + p]; xr[(size_t)i * n + p] = t;
            t = xi[(size_t)i * n + k]; xi[(size_t)i * n + k] = xi[(size_t)i * n + p]; xi[(size_t)i * n + p] = t;
        }
    }
done:
    free(ar); free(ai); free(wr); free(wi); free(ipiv);
    return info;
}

/* --------------------------------------------------------------- solves (sketch parity) */

/* Alg 3 line 1 over C on its own: P Z = L U in place on (ar, ai) with partial
 * pivoting on |re|+|im| (LAPACK izamax convention), ipiv[k] = row swapped with row k at
 * step k (0-based, LAPACK order).  Right-looking, one column per step, exactly the
 * elimination of or_zinv_lu line 1.  Returns 0 or the 1-based first exactly-zero pivot. */
int or_zgetrf(int n, double *ar, double *ai, int *ipiv)
{
    int info = 0;
    for (int k = 0; k < n; ++k) {
        int p = k;
        double best = cabs1(ar[(size_t)k * n + k], ai[(size_t)k * n + k]);
        for (int i = k + 1; i < n; ++i) {
            double v = cabs1(ar[(size_t)i * n + k], ai[(size_t)i * n + k]);
            if (v > best) { best = v; p = i; }
        }
        ipiv[k] = p;
        if (p != k) {
            for (int j = 0; j < n; ++j) {
                double t = ar[(size_t)k * n + j]; ar[(size_t)k * n + j] = ar[(size_t)p * n + j]; ar[(size_t)p * n + j] = t;
                t = ai[(size_t)k * n + j]; ai[(size_t)k * n + j] = ai[(size_t)p * n + j]; ai[(size_t)p * n + j] = t;
            }
        }
        double pr = ar[(size_t)k * n + k], pi = ai[(size_t)k * n + k];
        if (pr == 0.0 && pi == 0.0) { if (!info) info = k + 1; continue; }
        double den = pr * pr + pi * pi;
        double ir = pr / den, ii = -pi / den;
        #pragma omp parallel for schedule(static) if (n - k > 256)
        for (int i = k + 1; i < n; ++i) {
            double vr = ar[(size_t)i * n + k], vi = ai[(size_t)i * n + k];
            double lr = vr * ir - vi * ii, li = vr * ii + vi * ir;
            ar[(size_t)i * n + k] = lr; ai[(size_t)i * n + k] = li;
            double *rr = ar + (size_t)i * n, *ri = ai + (size_t)i * n;
            const double *kr = ar + (size_t)k * n, *ki = ai + (size_t)k * n;
            for (int j = k + 1; j < n; ++j) {
                rr[j] = rr[j] - (lr * kr[j] - li * ki[j]);
                ri[j] = ri[j] - (lr * ki[j] + li * kr[j]);
            }
        }
    }
    return info;
}

/* Solve with the factors of or_zgetrf (P Z = L U), k right-hand sides in place on the
 * row-major n x k arrays (br, bi):
 *   trans = 0:  Z Y = R     -> apply the interchanges to R in order, L W = P R (forward
 *               substitution, unit diagonal), U Y = W (back substitution);
 *   trans = 1:  Z^H Y = R   (Z^H = U^H L^H P) -> U^H W = R (forward), L^H V = W (back,
 *               unit diagonal), Y = P^T V (interchanges in reverse order).
 * The plain definition of Y = Z^{-1} R (Z^{-H} R): Gaussian elimination on the augmented
 * system.  Right-hand sides are independent (OpenMP over them). */
void or_zgetrs(int n, const double *ar, const double *ai, const int *ipiv, int trans, int k,
               double *br, double *bi)
{
    #pragma omp parallel for schedule(dynamic, 1) if (k > 1 && (long)n * n > 65536L)
    for (int c = 0; c < k; ++c) {
        double *yr = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        double *yi = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
        for (int i = 0; i < n; ++i) { yr[i] = br[(size_t)i * k + c]; yi[i] = bi[(size_t)i * k + c]; }
        if (trans == 0) {
            for (int q = 0; q < n; ++q) {               /* P R */
                int p = ipiv[q];
                if (p != q) { double t = yr[q]; yr[q] = yr[p]; yr[p] = t; t = yi[q]; yi[q] = yi[p]; yi[p] = t; }
            }
            for (int i = 0; i < n; ++i) {               /* L W = P R */
                double sr = yr[i], si = yi[i];
                for (int q = 0; q < i; ++q) {
                    double lr = ar[(size_t)i * n + q], li = ai[(size_t)i * n + q];
                    sr = sr - (lr * yr[q] - li * yi[q]);
                    si = si - (lr * yi[q] + li * yr[q]);
                }
                yr[i] = sr; yi[i] = si;
            }
            for (int i = n - 1; i >= 0; --i) {          /* U Y = W */
                double sr = yr[i], si = yi[i];
                for (int q = i + 1; q < n; ++q) {
                    double ur = ar[(size_t)i * n + q], ui = ai[(size_t)i * n + q];
                    sr = sr - (ur * yr[q] - ui * yi[q]);
                    si = si - (ur * yi[q] + ui * yr[q]);
                }
                double dr = ar[(size_t)i * n + i], di = ai[(size_t)i * n + i];
                double dd = dr * dr + di * di;          /* s / d = s conj(d) / |d|^2 */
                yr[i] = (sr * dr + si * di) / dd;
                yi[i] = (si * dr - sr * di) / dd;
            }
        } else {
            for (int i = 0; i < n; ++i) {               /* U^H W = R: (U^H)[i][q] = conj(U[q][i]) */
                double sr = yr[i], si = yi[i];
                for (int q = 0; q < i; ++q) {
                    double ur = ar[(size_t)q * n + i], ui = -ai[(size_t)q * n + i];
                    sr = sr - (ur * yr[q] - ui * yi[q]);
                    si = si - (ur * yi[q] + ui * yr[q]);
                }
                double dr = ar[(size_t)i * n + i], di = -ai[(size_t)i * n + i];
                double dd = dr * dr + di * di;
                yr[i] = (sr * dr + si * di) / dd;
                yi[i] = (si * dr - sr * di) / dd;
            }
            for (int i = n - 1; i >= 0; --i) {          /* L^H V = W: (L^H)[i][q] = conj(L[q][i]) */
                double sr = yr[i], si = yi[i];
                for (int q = i + 1; q < n; ++q) {
                    double lr = ar[(size_t)q * n + i], li = -ai[(size_t)q * n + i];
                    sr = sr - (lr * yr[q] - li * yi[q]);
                    si = si - (lr * yi[q] + li * yr[q]);
                }
                yr[i] = sr; yi[i] = si;
            }
            for (int q = n - 1; q >= 0; --q) {          /* Y = P^T V */
                int p = ipiv[q];
                if (p != q) { double t = yr[q]; yr[q] = yr[p]; yr[p] = t; t = yi[q]; yi[q] = yi[p]; yi[p] = t; }
            }
        }
        for (int i = 0; i < n; ++i) { br[(size_t)i * k + c] = yr[i]; bi[(size_t)i * k + c] = yi[i]; }
        free(yr); free(yi);
    }
}

/* Alg 1 on `count` independent matrices (config 3 full-set parity): or_frob_inv per matrix,
 * OpenMP over the matrices (each matrix's arithmetic is exactly or_frob_inv's). */
int or_frob_inv_many(int count, int n, const double *A, const double *B, double *Xre, double *Xim,
                     int branch, double kappa_sw, int *out, double *rho, int *status)
{
    size_t nn = (size_t)n * n;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int m = 0; m < count; ++m)
        status[m] = or_frob_inv(n, A + m * nn, B + m * nn, Xre + m * nn, Xim + m * nn, branch, kappa_sw,
                                out + 2 * (size_t)m, rho + 4 * (size_t)m);
    return 0;
}

/* thread count of the OpenMP loops (measurement control only: the arithmetic of every row is
   independent of it) */
void or_set_threads(int t)
{
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

int or_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
