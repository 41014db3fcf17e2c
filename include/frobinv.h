/*
 * frobinv.h -- C ABI of the B200-native Frobenius inversion library (libfrobinv.so).
 *
 * Method: Dai, Lim & Ye, "Inverting a complex matrix", arXiv 2208.01239.
 *   Lemma 4.1 / Alg 1:  for Z = A + iB with A, B real n x n,
 *     S1 (A invertible):  Z^{-1} = (A + B A^{-1} B)^{-1} - i A^{-1} B (A + B A^{-1} B)^{-1}
 *     S2 (B invertible):  Z^{-1} = B^{-1} A (A B^{-1} A + B)^{-1} - i (A B^{-1} A + B)^{-1}
 *   computed with two real inversions (Alg 3: LU with partial pivoting,
 *   U^{-1}, solve X L = U^{-1}) and three real GEMMs.
 *
 * Conventions shared by every entry point
 *   - Matrices are dense, ROW-MAJOR.  Complex matrices are interleaved complex128
 *     (re, im pairs of IEEE fp64; the layout of torch.complex128 and cuDoubleComplex);
 *     a leading dimension `ld*` counts complex elements per row (>= n).  Real matrices
 *     are fp64 with a leading dimension in doubles.
 *   - All matrix / workspace pointers are DEVICE pointers owned by the caller (except
 *     the *_host entry points and the host_* out-parameters, which are host memory).
 *     The library never allocates device memory and keeps no per-call state: calls are
 *     re-entrant given distinct workspaces.
 *   - `stream` is a cudaStream_t passed as void*; NULL means the legacy default
 *     stream.  Work is enqueued asynchronously on it.  LUs of order > 4096 (blocked
 *     getrf) fork onto two library-owned streams per device (created on first use: the
 *     panel chain at the highest priority, the far-column updates at the lowest) through
 *     events and join back to `stream` before the call returns, so stream order and CUDA
 *     graph capture are preserved; concurrent host threads serialise on that fork (one
 *     mutex per device).  The only host synchronisations
 *     are (a) FROB_BRANCH_AUTO in frob_inv (one small device->host read of LU(A)'s
 *     diagnostics and the norms of A and A^{-1}; a second one if B is inverted too), (b) a non-NULL host_info / host-side outputs, (c) the
 *     Newton drivers (one 16-byte read of delta_t per iteration), (d) *_host entries.
 *   - Outputs must not alias inputs (X != Z, S != Z, ...): FROB_ERR_INVALID_ARG.
 *   - Singular pivots: a pivot u_kk of an LU is "singular" when
 *       |u_kk| < 100 * n * 2^-53 * max_i |u_ii|        (reading R2);
 *     info = 1-based column k+1 of the first such pivot (LAPACK-style).
 *   - Errors are returned as frob_status; CUDA launch/runtime failures give
 *     FROB_ERR_CUDA (query frob_last_cuda_error()).
 */
#ifndef FROBINV_H
#define FROBINV_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FROB_OK = 0,
    FROB_ERR_SINGULAR = 1,       /* chosen branch (or the inner M) has a singular pivot; info = column */
    FROB_ERR_BOTH_SINGULAR = 2,  /* AUTO: neither A nor B usable (Z outside S1 u S2) */
    FROB_ERR_NOT_CONVERGED = 3,  /* Newton driver hit max_iter; the last iterate is returned */
    FROB_ERR_INVALID_ARG = 4,
    FROB_ERR_NONFINITE = 5,      /* NaN/Inf in the input */
    FROB_ERR_WORKSPACE = 6,      /* ws NULL or ws_bytes below the *_workspace_bytes query */
    FROB_ERR_CUDA = 7
} frob_status;

typedef enum {
    FROB_BRANCH_AUTO = 0, /* S1 unless A is singular or kappa_inf(A) = ||A||_inf ||A^{-1}||_inf of the
                             computed inverse exceeds 1e6; then also B is inverted and the part with
                             the smaller kappa_inf is used (reading R1', Thm 5.2)      */
    FROB_BRANCH_A = 1,    /* S1: X = A, Y = B (Alg 1 line 2)                                      */
    FROB_BRANCH_B = 2     /* S2: X = B, Y = A (Alg 1 line 4)                                      */
} frob_branch;

typedef enum { FROB_INV_FROBENIUS = 0, FROB_INV_ZLU = 1 } frob_inv_method;

typedef struct {
    int info;          /* 0 or the 1-based singular pivot column                         */
    int branch_used;   /* 1 = S1, 2 = S2, 0 = none                                       */
    double rho_a;      /* max|u_ii|/min|u_ii| of LU(A) (NaN if A was not factored)       */
    double rho_b;      /* same for LU(B)                                                 */
    double rho_m;      /* same for LU(M), M = X + Y X^{-1} Y                              */
    double kappa_a;    /* kappa_inf(A) = ||A||_inf ||A^{-1}||_inf from the computed inverse (AUTO
                          rule R1'; NEXT-1: ||A||_inf times the Hager-Higham estimate of ||A^{-1}||_inf);
                          NaN if A was not inverted                                     */
    double kappa_b;    /* same for B                                                     */
} frob_info;

/* Status record written ON THE DEVICE at the end of a call's stream work (frob_inv_dev), so
 * errors are visible without a host synchronisation inside the library: read it after the
 * stream (e.g. cudaMemcpyAsync + sync, or a later kernel). */
typedef struct {
    int status;        /* frob_status of the call: FROB_OK, FROB_ERR_SINGULAR (X or M has a singular
                          pivot, info = column), FROB_ERR_BOTH_SINGULAR, FROB_ERR_NONFINITE        */
    int info;          /* 0 or the 1-based singular pivot column                                   */
    int branch_used;   /* 1 = S1, 2 = S2, 0 = none                                                 */
    int nonfinite;     /* 1 if NaN/Inf was seen in the input                                       */
    double rho_a, rho_b, rho_m;   /* pivot ratios (NaN where the LU did not run)                   */
    double kappa_a, kappa_b;      /* kappa_inf of the parts as in frob_info                        */
} frob_dev_status;

/* ---------------------------------------------------------------- single matrix */

/* Bytes of device workspace frob_inv needs for order n (256-byte aligned pointer). */
size_t frob_inv_workspace_bytes(int n);

/* Z^{-1} by Frobenius inversion (Alg 1; steps SURVEY.md 8(a) a0-a7).
 *   n      order (>= 1)
 *   Z      device, n x n complex128 row-major, leading dim ldz (complex elements)
 *   X      device output, n x n complex128, leading dim ldx; must not overlap Z
 *   branch frob_branch
 *   ws     device workspace of at least frob_inv_workspace_bytes(n) bytes
 *   host_info  nullable; if non-NULL the call synchronises `stream`, fills it and returns the
 *              status found on the device (singular X or M, non-finite input).  With host_info
 *              NULL those device-side findings are NOT returned (only argument, workspace, CUDA
 *              errors and, for AUTO, non-finite input / both parts singular are): use
 *              frob_inv_dev to receive them asynchronously in a device status record.
 * Returns FROB_OK, or an error status (X is then unspecified). */
frob_status frob_inv(int n, const double *Z, long long ldz, double *X, long long ldx,
                     int branch, void *ws, size_t ws_bytes, void *stream, frob_info *host_info);

/* frob_inv with options (bit mask):
 *   FROB_OPT_FUSED_FIRST_STEP  NEXT-1 (Thm 5.1 proof): C = X^{-1} Y is computed by
 *     solving L G = P Y and U C = G (blocked substitution with the LU factors) -- X^{-1} itself is
 *     never formed, 8 2/3 n^3 instead of 10 n^3 flops.  Same results up to rounding order.
 * Unknown bits give FROB_ERR_INVALID_ARG.  Everything else as frob_inv. */
#define FROB_OPT_FUSED_FIRST_STEP 1
/*   FROB_OPT_DEVICE_AUTO  (branch must be FROB_BRANCH_AUTO, not with FROB_OPT_FUSED_FIRST_STEP)
 *     reading R1' decided ON THE DEVICE: A and B are both factored and inverted (one extra real
 *     inversion, 2 n^3 flops), a one-thread kernel picks the branch from their kappa_inf, and B's
 *     inverse / permutation and the rotated parts move into the S1 slots by predicated copies.
 *     No host synchronisation at all, so the call can be captured in a CUDA graph; results are
 *     bitwise those of the host-decided AUTO. */
#define FROB_OPT_DEVICE_AUTO 2
frob_status frob_inv_opts(int n, const double *Z, long long ldz, double *X, long long ldx, int branch,
                          int options, void *ws, size_t ws_bytes, void *stream, frob_info *host_info);

/* frob_inv_opts with a DEVICE status record: d_status (device frob_dev_status*, nullable) receives
 * the call's status at the end of its stream work.  The library never synchronises for forced
 * branches or with FROB_OPT_DEVICE_AUTO (plain AUTO still reads LU(A)'s statistics on the host).
 * The return value reports only argument / workspace / CUDA errors and the host-decided AUTO
 * outcomes (non-finite input, both parts singular); everything else is in *d_status. */
frob_status frob_inv_dev(int n, const double *Z, long long ldz, double *X, long long ldx, int branch,
                         int options, frob_dev_status *d_status, void *ws, size_t ws_bytes, void *stream);

/* Randomized Frobenius inversion (Alg 5): X = A - mu B, Y = mu A + B,
 * W = (X + iY)^{-1} by Alg 1 (AUTO branch rule), Z^{-1} = (W1 - mu W2) + i (mu W1 + W2).
 * Works for invertible Z whose real and imaginary parts are both singular (Lemma 5.4,
 * A - mu B is singular for at most n values of mu).  mu in [0, 1] is drawn by the
 * CALLER (line 1; the Python binding uses a seeded generator); mu outside [0, 1] gives
 * FROB_ERR_INVALID_ARG.  Workspace, layout, aliasing and errors as frob_inv (host_info
 * describes the inner Alg 1 call on X + iY).  Cost: frob_inv + 8 n^2, fused into
 * the ingest and final-epilogue kernels. */
frob_status frob_inv_rand(int n, const double *Z, long long ldz, double *X, long long ldx, double mu,
                          void *ws, size_t ws_bytes, void *stream, frob_info *host_info);

/* Same computation with HOST input/output buffers (pinned memory recommended): copies
 * Z host->device, runs frob_inv, copies X device->host, synchronises.  Z_host/X_host
 * are dense (ld = n).  ws must hold frob_inv_host_workspace_bytes(n) bytes.  For n >= 8192 the
 * final GEMM runs in 8 row blocks and each block's device->host copy (a library-owned copy stream)
 * overlaps the next block (results bitwise those of frob_inv).  The status found on the device
 * (singular X or M, non-finite input) is always returned. */
size_t frob_inv_host_workspace_bytes(int n);
frob_status frob_inv_host(int n, const double *Z_host, double *X_host, int branch,
                          void *ws, size_t ws_bytes, void *stream, frob_info *host_info);

/* `count` independent matrices with HOST buffers, pipelined: Z_host / X_host hold count
 * dense n x n interleaved complex128 matrices back to back (count * n * n * 16 bytes each,
 * pinned memory required for the overlap).  Matrix i + 1 is copied host->device and matrix
 * i - 1 device->host (two library-owned copy streams per device) while matrix i is inverted on
 * `stream` (frob_inv with `branch`), double-buffered in ws; the call synchronises `stream`
 * before returning.  Results equal count frob_inv_host calls bit for bit.  ws must hold
 * frob_inv_host_many_workspace_bytes(n) bytes (independent of count).
 *   h_status  nullable host int[count] (pinned recommended): per-matrix frob_status found on the
 *             device (singular X or M, non-finite input, both parts singular), copied back with
 *             each result.
 * Returns the first failing matrix's status (device findings included; with an error that stops
 * the loop -- AUTO both-singular / non-finite, CUDA -- later matrices are not computed and their
 * h_status entries are FROB_ERR_INVALID_ARG).  On every return path both copy streams have been
 * joined and `stream` synchronised, so the host buffers are no longer in use. */
size_t frob_inv_host_many_workspace_bytes(int n);
frob_status frob_inv_host_many(int n, int count, const double *Z_host, double *X_host, int branch,
                               int *h_status, void *ws, size_t ws_bytes, void *stream);

/* Complex-LU inversion: Alg 3 over C (the paper's comparator `X\eye(n)`,
 * P:L1057): complex LU with partial pivoting on |re|+|im|, U^{-1}, X = U^{-1} L^{-1},
 * column interchanges.  Same layout/ownership rules as frob_inv.
 * host_info: nullable host int receiving info (forces a synchronisation). */
size_t zinv_lu_workspace_bytes(int n);
frob_status zinv_lu(int n, const double *Z, long long ldz, double *X, long long ldx,
                    void *ws, size_t ws_bytes, void *stream, int *host_info);

/* ---------------------------------------------------------------- batched small n */

/* One CTA per matrix for n <= 64 (registers/shared memory), a resident
 * shared-memory pipeline per matrix for 64 < n <= 128.  Z and X hold `batch`
 * n x n complex128 matrices, dense (ld = n), matrix b at Z + 2*b*strideZ doubles
 * (strideZ in complex elements, >= n*n).
 *   d_info         device int[batch]: 0 or 1-based singular column per matrix
 *   d_branch_used  device uint8[batch]: 1 (S1) or 2 (S2) per matrix (nullable)
 * No host synchronisation; per-matrix failures are reported only in d_info.
 * FROB_BRANCH_AUTO applies reading R1 per matrix (lazy: B is factored only if LU(A)
 * fails the pivot-ratio test). */
size_t frob_inv_batched_workspace_bytes(int n, int batch);
frob_status frob_inv_batched(int n, int batch, const double *Z, long long strideZ,
                             double *X, long long strideX, int branch, int *d_info,
                             unsigned char *d_branch_used, void *ws, size_t ws_bytes,
                             void *stream);

/* frob_inv_batched with HOST buffers, pipelined in chunks of `chunk` matrices: the copy of
 * chunk j + 1 in and of chunk j - 1 out (two library-owned copy streams per device) overlap the
 * inversion of chunk j on `stream`; synchronises before returning.  Z_host / X_host: batch
 * dense n x n complex128 matrices back to back (pinned memory required for the overlap);
 * h_info: host int[batch] (nullable) receives d_info.  Results equal frob_inv_batched bit for
 * bit.  ws must hold frob_inv_batched_host_workspace_bytes(n, chunk) bytes. */
size_t frob_inv_batched_host_workspace_bytes(int n, int chunk);
frob_status frob_inv_batched_host(int n, int batch, const double *Z_host, double *X_host, int branch,
                                  int *h_info, int chunk, void *ws, size_t ws_bytes, void *stream);

/* Batched complex-LU comparator (complex Gauss-Jordan with partial pivoting, |re|+|im|),
 * 1 <= n <= 128: one CTA per matrix for n <= 64, a cluster of two CTAs (rows split, pivot
 * candidates and pivot rows exchanged through distributed shared memory) for 64 < n <= 128.
 * Layout, strides and d_info as frob_inv_batched. */
size_t zinv_lu_batched_workspace_bytes(int n, int batch);
frob_status zinv_lu_batched(int n, int batch, const double *Z, long long strideZ,
                            double *X, long long strideX, int *d_info, void *ws,
                            size_t ws_bytes, void *stream);

/* ---------------------------------------------------------------- Newton drivers */

/* Matrix sign by Newton X_{t+1} = (X_t + X_t^{-1})/2, X_0 = Z.
 * Stops when delta_t = ||X_{t+1} - X_t||_F / ||X_{t+1}||_F < tol or after max_iter
 * steps (BASELINE config 4; reading R6); at least one step.
 *   Z, S        device n x n complex128 (ld = n); S receives sign(Z); S != Z
 *   method      frob_inv_method used for X_t^{-1}
 *   host_iters, host_final_delta   host out (required)
 *   host_trace  nullable host double[max_iter] receiving delta_t per step
 * Returns FROB_OK, FROB_ERR_NOT_CONVERGED (S = last iterate) or an inversion error. */
size_t frob_newton_workspace_bytes(int n, int method);
frob_status frob_sign_newton(int n, const double *Z, double *S, double tol, int max_iter,
                             int method, void *ws, size_t ws_bytes, void *stream,
                             int *host_iters, double *host_final_delta, double *host_trace);

/* Polar decomposition A = U H by Newton X_{t+1} = (X_t + X_t^{-*})/2, X_0 = A
 * (P:L1231-1233); H = (U^H A + (U^H A)^H)/2 (reading R7).  Same stopping
 * rule and outputs as frob_sign_newton; U, H device n x n complex128 (ld = n). */
frob_status frob_polar_newton(int n, const double *A, double *U, double *H, double tol,
                              int max_iter, int method, void *ws, size_t ws_bytes,
                              void *stream, int *host_iters, double *host_final_delta,
                              double *host_trace);

/* ---------------------------------------------------------------- real building blocks
 * Exposed so the paper's threshold quantities T_inv and T_mult (Thm 5.1)
 * can be measured on the very kernels the Frobenius path uses. */

/* C = alpha * A B + beta * C; A m x k, B k x n, C m x n, all fp64 row-major. */
frob_status frob_dgemm(int m, int n, int k, double alpha, const double *A, long long lda,
                       const double *B, long long ldb, double beta, double *C, long long ldc,
                       void *stream);

/* C = alpha * tri(T) B (T n x n triangular: uplo 1 = upper, 2 = lower, B n x m, C n x m), fp64
 * row-major.  The GEMM engine skips the zero triangle tile by tile, so T's other strict triangle
 * must hold zeros (as the library's triangular inverses do).  Used to measure Thm 5.1's lambda
 * (triangular x dense costs lambda T_mult). */
frob_status frob_dtrmm(int uplo, int n, int m, double alpha, const double *T, long long ldt, const double *B,
                       long long ldb, double *C, long long ldc, void *stream);

/* Real inversion Alg 3: Ainv = A^{-1}, fp64 n x n row-major.
 * host_info nullable (info + pivot ratio via rho_a). */
size_t frob_dinv_workspace_bytes(int n);
frob_status frob_dinv(int n, const double *A, long long lda, double *Ainv, long long ldainv,
                      void *ws, size_t ws_bytes, void *stream, frob_info *host_info);

/* LU with partial pivoting in place (Alg 3 line 1): on return A holds L\U of P A
 * and perm[i] = original row index of row i of P A (device int[n]).  Needs
 * frob_dgetrf_workspace_bytes(n). */
size_t frob_dgetrf_workspace_bytes(int n);
frob_status frob_dgetrf(int n, double *A, long long lda, int *perm, void *ws, size_t ws_bytes,
                        void *stream, frob_info *host_info);

/* Hermitian positive definite inversion (paper Section 6).
 * frob_hpd_inv: Alg 6 "first variant of Frobenius inversion" -- for HPD Z = A + iB
 *   (Lemma 6.1: A symmetric positive definite, B skew, Z in S1): Cholesky A = U^T U,
 *   K1 = U^{-T} B, K2 = U^{-1} K1, K4 = A - K1^T K1 = V^T V, K6 = V^{-1} V^{-T}, K7 = K2 K6,
 *   Z^{-1} = K6 - i K7 (Cholesky blocked right-looking, Alg 10).
 * zhpd_inv_chol: Alg 8 over C, the comparator: Z = U^H U, X = U^{-1} U^{-H}.
 *   Z, X: device n x n complex128 (ldz, ldx complex elements), Z is not checked for being
 *   Hermitian (only its upper triangle is read by the Cholesky factorisations).
 *   host_info: nullable; if non-NULL the call synchronises and stores 0 or the 1-based column
 *   of the first non-positive Cholesky pivot (FROB_ERR_SINGULAR: not positive definite). */
size_t frob_hpd_inv_workspace_bytes(int n);
frob_status frob_hpd_inv(int n, const double *Z, long long ldz, double *X, long long ldx, void *ws,
                         size_t ws_bytes, void *stream, int *host_info);
/* frob_dpoinv: real symmetric positive definite inversion, Alg 8 over R: A = U^T U
 *   (blocked Cholesky, upper triangle of A read), K = U^{-1}, X = K K^T.  Its time is Thm 6.2's
 *   T_pinv (defined on Alg 9, which has the same flop count).  A, X: device n x n
 *   fp64 row-major (lda, ldx doubles); host_info as frob_hpd_inv. */
size_t frob_dpoinv_workspace_bytes(int n);
frob_status frob_dpoinv(int n, const double *A, long long lda, double *X, long long ldx, void *ws,
                        size_t ws_bytes, void *stream, int *host_info);
size_t zhpd_inv_chol_workspace_bytes(int n);
frob_status zhpd_inv_chol(int n, const double *Z, long long ldz, double *X, long long ldx, void *ws,
                          size_t ws_bytes, void *stream, int *host_info);

/* Sylvester equation A X + X B = C through the matrix sign function:
 * sign([[A, -C], [0, -B]]) = [[I, -2X], [0, -I]] when sign(A) = I_m and sign(B) = I_n
 * (spectra in the open right half plane); the sign of the order-(m+n) block matrix is computed
 * by frob_sign_newton's iteration (each step one inversion by `method`), X = -S_12 / 2.
 *   A  device m x m, B device n x n, C device m x n, X device m x n output: complex128,
 *      row-major, dense (ld = number of columns).
 *   tol, max_iter, method, host_iters, host_final_delta: as frob_sign_newton.
 * Returns FROB_OK, FROB_ERR_NOT_CONVERGED (X from the last iterate), or an error status.
 * Synchronises `stream` (the Newton driver reads delta_t every step). */
size_t frob_sylvester_workspace_bytes(int m, int n, int method);
frob_status frob_sylvester(int m, int n, const double *A, const double *B, const double *C, double *X,
                           double tol, int max_iter, int method, void *ws, size_t ws_bytes, void *stream,
                           int *host_iters, double *host_final_delta);
/* Lyapunov equation A X + X A^* = C: frob_sylvester with B = A^* (built on the
 * device).  Workspace: frob_sylvester_workspace_bytes(n, n, method). */
frob_status frob_lyapunov(int n, const double *A, const double *C, double *X, double tol, int max_iter,
                          int method, void *ws, size_t ws_bytes, void *stream, int *host_iters,
                          double *host_final_delta);

/* ---------------------------------------------------------------- misc */
const char *frob_status_string(int status);
const char *frob_last_cuda_error(void);
int frob_version(void);
/* Diagnostics: number of CUDA kernels this process has launched through the library
 * (monotonic; used by bench.py to report gpu_launches). */
unsigned long long frob_launch_count(void);

/* Optional per-kernel timing for measurement tools (off by default; not thread-safe with
 * concurrent library calls).  frob_profile_enable(1) clears and starts recording: every
 * instrumented launch (LU panel, fused LU update, GEMM engine) is bracketed by CUDA events
 * on the stream it is launched on.  frob_profile_read synchronises the recorded events and
 * writes {"name": {"launches": L, "total_ms": T}, ...} (JSON, NUL-terminated) into buf;
 * returns the JSON length (call with buf = NULL to size it) or -1 on a CUDA error.
 * Instrumented runs are slower (events between launches); time the product separately. */
void frob_profile_enable(int on);
int frob_profile_read(char *buf, size_t len);

#ifdef __cplusplus
}
#endif
#endif /* FROBINV_H */
