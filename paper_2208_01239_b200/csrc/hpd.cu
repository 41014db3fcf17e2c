// hpd.cu -- Hermitian positive definite inversion (paper Section 6):
//   frob_hpd_inv   Alg 6 "first variant of Frobenius inversion": two real
//                  Cholesky factorisations, triangular inverses and five real GEMMs
//   zhpd_inv_chol  Alg 8 "first matrix inversion via Cholesky" over C, the
//                  comparator: complex Cholesky, U^{-1}, X = U^{-1} U^{-H}
//   frob_dpoinv    Alg 8 over R: the real SPD inversion whose time is Thm 6.2's T_pinv (P:L845,
//                  defined on Alg 9, which has the same flop count)
// Cholesky (Alg 10, upper form A = U^H U) is blocked right-looking with
// CHOL_NB-row block rows:
//   chol_diag_kernel  one CTA factors the diagonal block in shared memory (column by column,
//                     sqrt + row scaling + rank-1 update) and also writes W^H = (U_kk^{-1})^H
//   panel             U_k,right = W^H A_k,right   (GEMM engine, triangular A operand)
//   trailing          A_right -= (U_k,right)^H U_k,right  (conjugate transpose + GEMM, beta = 1;
//                     tiles strictly below the diagonal skipped: only the upper triangle is read)
// The GEMM engine takes no transposed operands, so every ^T / ^H is an explicit transpose.
#include <algorithm>
#include <climits>
#include <cstdio>
#include "lu.cuh"
#include "../../include/frobinv.h"

namespace frob {

constexpr int CHOL_NB = 64;

FROB_DEV double conj_of(double v) { return v; }
FROB_DEV double2 conj_of(double2 v) { return make_double2(v.x, -v.y); }
FROB_DEV double re_part(double v) { return v; }
FROB_DEV double re_part(double2 v) { return v.x; }
FROB_DEV double2 from_real(double v, double2) { return make_double2(v, 0.0); }
FROB_DEV double shfl_xor4(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
FROB_DEV double2 shfl_xor4(double2 v, int o) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o));
}
FROB_DEV double from_real(double v, double) { return v; }

// Factor the diagonal block (k0, k0) in place (upper; zeros below inside the block) and write
// W^H = (U_kk^{-1})^H (lower triangular, CHOL_NB x CHOL_NB, ld CHOL_NB) to wh.  info: first
// 1-based column with a non-positive pivot (atomicMin; INT_MAX = none).
// 256 threads as 16 x 16: two barriers per column (every thread derives the pivot and its reciprocal
// from S[j][j] itself; the scaled row j, then the trailing upper triangle in 2-D strides, no index
// divisions); U_kk^{-1} by row-wise back substitution with 4 threads per column (shuffle-summed
// partial dot products, one barrier per row) from the reciprocals kept during the factorisation.
template <typename T>
__global__ void __launch_bounds__(256) chol_diag_kernel(T *__restrict__ A, long long ld, int n, int k0,
                                                        T *__restrict__ wh, int *__restrict__ info) {
    extern __shared__ __align__(16) unsigned char chol_smem[];
    typedef T Row[CHOL_NB + 1];
    Row *S = reinterpret_cast<Row *>(chol_smem);          // the block, then U_kk
    Row *W = S + CHOL_NB;                                  // U_kk^{-1}
    __shared__ double pdiag[CHOL_NB], rdiag[CHOL_NB];      // u_jj and 1 / u_jj
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const int nb = min(CHOL_NB, n - k0);
    for (int i = ty; i < CHOL_NB; i += 16)
        for (int j = tx; j < CHOL_NB; j += 16)
            S[i][j] = (i < nb && j < nb) ? A[(long long)(k0 + i) * ld + k0 + j]
                                         : ((i == j) ? one_of(T()) : zero_of(T()));
    __syncthreads();
    for (int j = 0; j < nb; ++j) {
        const double d = re_part(S[j][j]);
        const double p = sqrt(d);  // NaN for a failed pivot: the result is flagged through info
        const double ip = 1.0 / p;
        if (tid == 0) {
            if (!(d > 0.0)) atomicMin(info, k0 + j + 1);
            pdiag[j] = p;
            rdiag[j] = ip;
        }
        // row j of U: U[j][c] = S[j][c] / p (c > j); U[j][j] = p is written at the end
        for (int c = j + 1 + tid; c < nb; c += 256) S[j][c] = scal(S[j][c], ip);
        __syncthreads();
        // trailing upper part: S[r][c] -= conj(U[j][r]) U[j][c], j < r <= c
        for (int r = j + 1 + ty; r < nb; r += 16) {
            const T ur = conj_of(S[j][r]);
            for (int c = r + tx; c < nb; c += 16) S[r][c] = msub(S[r][c], ur, S[j][c]);
        }
        __syncthreads();
    }
    for (int i = ty; i < nb; i += 16)
        for (int j = tx; j < nb; j += 16)
            A[(long long)(k0 + i) * ld + k0 + j] = (j > i) ? S[i][j] : ((j == i) ? from_real(pdiag[i], T()) : zero_of(T()));
    // W = U_kk^{-1} (upper): rows from the bottom, W[i][c] = (delta_ic - sum_{i<q<=c} U[i][q] W[q][c]) / u_ii,
    // column c on the 4 consecutive lanes 4c .. 4c + 3 (a quarter of the q range each)
    {
        const int c = tid >> 2, l = tid & 3;
        for (int i = CHOL_NB - 1; i >= 0; --i) {
            T acc = zero_of(T());
            if (i < nb && c < nb && c > i)
                for (int q = i + 1 + l; q <= c; q += 4) acc = msub(acc, S[i][q], W[q][c]);
            acc = add(acc, shfl_xor4(acc, 1));
            acc = add(acc, shfl_xor4(acc, 2));
            if (l == 0) {
                T v = zero_of(T());
                if (i < nb && c < nb && c >= i) v = scal(add(acc, (c == i) ? one_of(T()) : zero_of(T())), rdiag[i]);
                else if (i >= nb && c == i) v = one_of(T());
                W[i][c] = v;
            }
            __syncthreads();
        }
    }
    for (int i = ty; i < CHOL_NB; i += 16)
        for (int j = tx; j < CHOL_NB; j += 16)
            wh[i * CHOL_NB + j] = (i < nb && j < nb) ? conj_of(W[j][i]) : zero_of(T());
}

// dst (cols x rows, ldd) = src (rows x cols, lds)^T (conjugated if conj)
template <typename T>
__global__ void __launch_bounds__(256) transpose_kernel(const T *__restrict__ src, long long lds, T *__restrict__ dst,
                                                        long long ldd, int rows, int cols, int conj) {
    __shared__ T tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const int tiles_c = (cols + 31) / 32;
    for (int t = blockIdx.x; t < ((rows + 31) / 32) * tiles_c; t += gridDim.x) {
        const int bi = t / tiles_c, bj = t % tiles_c;
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int i = bi * 32 + r, j = bj * 32 + tx;
            if (i < rows && j < cols) tile[r][tx] = src[(long long)i * lds + j];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int i = bj * 32 + r, j = bi * 32 + tx;  // dst row i = src column
            if (i < cols && j < rows) {
                const T v = tile[tx][r];
                dst[(long long)i * ldd + j] = conj ? conj_of(v) : v;
            }
        }
    }
}

// zero the strictly lower triangle
template <typename T>
__global__ void zero_lower_kernel(T *__restrict__ A, long long ld, int n) {
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        if (j < i) A[(long long)i * ld + j] = zero_of(T());
    }
}

static int grid_for(long long total) { return (int)std::min<long long>((total + 255) / 256, 148LL * 8); }

template <typename T>
static cudaError_t transpose(const T *src, long long lds, T *dst, long long ldd, int rows, int cols, bool conj,
                             cudaStream_t s) {
    const long long tiles = (long long)((rows + 31) / 32) * ((cols + 31) / 32);
    count_launch();
    transpose_kernel<T><<<(int)std::min<long long>(tiles, 148LL * 8), 256, 0, s>>>(src, lds, dst, ldd, rows, cols,
                                                                                  conj ? 1 : 0);
    return cudaGetLastError();
}

// Cholesky A = U^H U in place (upper; the strictly lower part is zeroed).  work: CHOL_NB^2 +
// n * CHOL_NB elements.  info: device int, INT_MAX on success (set by the caller).
template <typename T>
static cudaError_t potrf_upper(int n, T *A, long long ld, T *work, int *info, cudaStream_t s) {
    cudaError_t e;
    T *wh = work;
    T *tb = work + CHOL_NB * CHOL_NB;  // (n - k0 - nb) x CHOL_NB transposed panel
    for (int k0 = 0; k0 < n; k0 += CHOL_NB) {
        const int nb = std::min(CHOL_NB, n - k0), m = n - k0 - nb;
        const size_t smem = 2 * (size_t)CHOL_NB * (CHOL_NB + 1) * sizeof(T);
        static bool attr = false;
        if (!attr) {
            if ((e = cudaFuncSetAttribute(chol_diag_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
                cudaSuccess)
                return e;
            attr = true;
        }
        count_launch();
        chol_diag_kernel<T><<<1, 256, smem, s>>>(A, ld, n, k0, wh, info);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if (m <= 0) break;
        T *Ak = A + (long long)k0 * ld + k0 + nb;  // block row k, right part (nb x m)
        auto p = gemm_params<T>(nb, m, nb, 1.0, wh, CHOL_NB, Ak, ld, 0.0, nullptr, ld, Ak, ld);
        p.triA = TRI_LOWER;
        if ((e = gemm_launch<T>(p, 1, s)) != cudaSuccess) return e;
        if ((e = transpose<T>(Ak, ld, tb, CHOL_NB, nb, m, true, s)) != cudaSuccess) return e;
        T *Ar = A + (long long)(k0 + nb) * ld + k0 + nb;
        auto q = gemm_params<T>(m, m, nb, -1.0, tb, CHOL_NB, Ak, ld, 1.0, Ar, ld, Ar, ld);
        q.triC = TRI_UPPER;  // only the upper triangle of the trailing matrix is ever read (SYRK)
        if ((e = gemm_launch<T>(q, 1, s)) != cudaSuccess) return e;
    }
    count_launch();
    zero_lower_kernel<T><<<grid_for((long long)n * n), 256, 0, s>>>(A, ld, n);
    return cudaGetLastError();
}

static long long ld_hpd(int n) { return ((long long)n + 7) / 8 * 8; }
static size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

// planar parts of interleaved Z (X = Re, Y = Im)
__global__ void hpd_split_kernel(const double2 *__restrict__ Z, long long ldz, int n, double *__restrict__ X,
                                 double *__restrict__ Y, double *__restrict__ U, long long ld) {
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const double2 z = Z[(long long)i * ldz + j];
        const long long o = (long long)i * ld + j;
        X[o] = z.x;
        Y[o] = z.y;
        U[o] = z.x;
    }
}
__global__ void zcopy_kernel(const double2 *__restrict__ Z, long long ldz, int n, double2 *__restrict__ W,
                             long long ld) {
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        W[(long long)i * ld + j] = Z[(long long)i * ldz + j];
    }
}
__global__ void set_int_kernel(int *p, int v) { *p = v; }
__global__ void copy_real_kernel(const double *__restrict__ A, long long lda, int n, double *__restrict__ U,
                                 long long ld) {
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        U[(long long)i * ld + j] = A[(long long)i * lda + j];
    }
}

size_t hpd_ws_bytes(int n) {
    const long long ld = ld_hpd(n);
    return 7 * al256((size_t)n * ld * 8) + al256((size_t)(CHOL_NB * CHOL_NB + (size_t)n * CHOL_NB) * 8) + 256;
}
size_t zhpd_ws_bytes(int n) {
    const long long ld = ld_hpd(n);
    return 3 * al256((size_t)n * ld * 16) + al256((size_t)(CHOL_NB * CHOL_NB + (size_t)n * CHOL_NB) * 16) + 256;
}

}  // namespace frob

using namespace frob;

extern "C" {

size_t frob_hpd_inv_workspace_bytes(int n) { return n < 1 ? 0 : hpd_ws_bytes(n); }
size_t zhpd_inv_chol_workspace_bytes(int n) { return n < 1 ? 0 : zhpd_ws_bytes(n); }

frob_status frob_hpd_inv(int n, const double *Z, long long ldz, double *X, long long ldx, void *ws, size_t ws_bytes,
                         void *stream, int *host_info) {
    if (n < 1 || !Z || !X || ldz < n || ldx < n) return FROB_ERR_INVALID_ARG;
    if (!ws || ws_bytes < hpd_ws_bytes(n)) return FROB_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const long long ld = ld_hpd(n);
    unsigned char *b = reinterpret_cast<unsigned char *>(ws);
    const size_t mb = al256((size_t)n * ld * 8);
    double *Xm = (double *)(b), *Ym = (double *)(b + mb), *W1 = (double *)(b + 2 * mb), *W2 = (double *)(b + 3 * mb);
    double *W3 = (double *)(b + 4 * mb), *W4 = (double *)(b + 5 * mb), *W5 = (double *)(b + 6 * mb);
    double *work = (double *)(b + 7 * mb);
    int *info = (int *)(b + 7 * mb + al256((size_t)(CHOL_NB * CHOL_NB + (size_t)n * CHOL_NB) * 8));
    cudaError_t e;
#define HPD_CK(x) do { if ((e = (x)) != cudaSuccess) return FROB_ERR_CUDA; } while (0)
    count_launch();
    set_int_kernel<<<1, 1, 0, s>>>(info, INT_MAX);
    count_launch();
    hpd_split_kernel<<<grid_for((long long)n * n), 256, 0, s>>>(reinterpret_cast<const double2 *>(Z), ldz, n, Xm, Ym,
                                                                 W1, ld);
    HPD_CK(cudaGetLastError());
    // l.6: X = U^T U (W1), U <- U^{-1}
    HPD_CK(potrf_upper<double>(n, W1, ld, work, info, s));
    HPD_CK(tri_inverses<double>(n, W1, nullptr, ld, W2, s));
    // l.7: K1 = U^{-T} Y = (U^{-1})^T Y  (W3)
    HPD_CK(transpose<double>(W1, ld, W2, ld, n, n, false, s));
    {
        auto p = gemm_params<double>(n, n, n, 1.0, W2, ld, Ym, ld, 0.0, nullptr, ld, W3, ld);
        p.triA = TRI_LOWER;
        HPD_CK(gemm_launch<double>(p, 1, s));
    }
    // l.8: K2 = U^{-1} K1  (W4)
    {
        auto p = gemm_params<double>(n, n, n, 1.0, W1, ld, W3, ld, 0.0, nullptr, ld, W4, ld);
        p.triA = TRI_UPPER;
        HPD_CK(gemm_launch<double>(p, 1, s));
    }
    // l.9-10: K4 = X - K1^T K1  (W5)
    HPD_CK(transpose<double>(W3, ld, W2, ld, n, n, false, s));
    {
        auto p = gemm_params<double>(n, n, n, -1.0, W2, ld, W3, ld, 1.0, Xm, ld, W5, ld);
        HPD_CK(gemm_launch<double>(p, 1, s));
    }
    // l.11-12: K4 = V^T V, K5 = V^{-1}  (W5)
    HPD_CK(potrf_upper<double>(n, W5, ld, work, info, s));
    HPD_CK(tri_inverses<double>(n, W5, nullptr, ld, W2, s));
    // l.13: K6 = K5 K5^T  (W1)
    HPD_CK(transpose<double>(W5, ld, W2, ld, n, n, false, s));
    {
        auto p = gemm_params<double>(n, n, n, 1.0, W5, ld, W2, ld, 0.0, nullptr, ld, W1, ld);
        p.triA = TRI_UPPER;
        p.triB = TRI_LOWER;
        HPD_CK(gemm_launch<double>(p, 1, s));
    }
    // l.14 + return: X = K6 - i K2 K6  (final epilogue: (D, alpha acc) with alpha = -1)
    {
        auto p = gemm_params<double>(n, n, n, -1.0, W4, ld, W1, ld, 0.0, W1, ld, X, ldx);
        p.epi = EPI_FROB_A;
        HPD_CK(gemm_launch<double>(p, 1, s));
    }
    if (host_info) {
        int h = 0;
        HPD_CK(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, s));
        HPD_CK(cudaStreamSynchronize(s));
        *host_info = (h == INT_MAX) ? 0 : h;
        if (h != INT_MAX) return FROB_ERR_SINGULAR;
    }
    return FROB_OK;
#undef HPD_CK
}

size_t frob_dpoinv_workspace_bytes(int n) {
    if (n < 1) return 0;
    const long long ld = ld_hpd(n);
    return 3 * al256((size_t)n * ld * 8) + al256((size_t)(CHOL_NB * CHOL_NB + (size_t)n * CHOL_NB) * 8) + 256;
}

frob_status frob_dpoinv(int n, const double *A, long long lda, double *X, long long ldx, void *ws, size_t ws_bytes,
                        void *stream, int *host_info) {
    if (n < 1 || !A || !X || lda < n || ldx < n) return FROB_ERR_INVALID_ARG;
    if (!ws || ws_bytes < frob_dpoinv_workspace_bytes(n)) return FROB_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const long long ld = ld_hpd(n);
    unsigned char *b = reinterpret_cast<unsigned char *>(ws);
    const size_t mb = al256((size_t)n * ld * 8);
    double *U = (double *)b, *Kt = (double *)(b + mb), *T = (double *)(b + 2 * mb);
    double *work = (double *)(b + 3 * mb);
    int *info = (int *)(b + 3 * mb + al256((size_t)(CHOL_NB * CHOL_NB + (size_t)n * CHOL_NB) * 8));
    cudaError_t e;
#define DP_CK(x) do { if ((e = (x)) != cudaSuccess) return FROB_ERR_CUDA; } while (0)
    count_launch(2);
    set_int_kernel<<<1, 1, 0, s>>>(info, INT_MAX);
    copy_real_kernel<<<grid_for((long long)n * n), 256, 0, s>>>(A, lda, n, U, ld);
    DP_CK(cudaGetLastError());
    DP_CK(potrf_upper<double>(n, U, ld, work, info, s));      // A = U^T U       (Alg 8 line 1)
    DP_CK(tri_inverses<double>(n, U, nullptr, ld, T, s));      // K = U^{-1}      (line 2)
    DP_CK(transpose<double>(U, ld, Kt, ld, n, n, false, s));   // K^T
    {
        auto p = gemm_params<double>(n, n, n, 1.0, U, ld, Kt, ld, 0.0, nullptr, ld, X, ldx);
        p.triA = TRI_UPPER;
        p.triB = TRI_LOWER;
        DP_CK(gemm_launch<double>(p, 1, s));                   // X = K K^T       (line 3)
    }
    if (host_info) {
        int h = 0;
        DP_CK(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, s));
        DP_CK(cudaStreamSynchronize(s));
        *host_info = (h == INT_MAX) ? 0 : h;
        if (h != INT_MAX) return FROB_ERR_SINGULAR;
    }
    return FROB_OK;
#undef DP_CK
}

frob_status zhpd_inv_chol(int n, const double *Z, long long ldz, double *X, long long ldx, void *ws, size_t ws_bytes,
                          void *stream, int *host_info) {
    if (n < 1 || !Z || !X || ldz < n || ldx < n) return FROB_ERR_INVALID_ARG;
    if (!ws || ws_bytes < zhpd_ws_bytes(n)) return FROB_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const long long ld = ld_hpd(n);
    unsigned char *b = reinterpret_cast<unsigned char *>(ws);
    const size_t mb = al256((size_t)n * ld * 16);
    double2 *U = (double2 *)b, *Kh = (double2 *)(b + mb), *T = (double2 *)(b + 2 * mb);
    double2 *work = (double2 *)(b + 3 * mb);
    int *info = (int *)(b + 3 * mb + al256((size_t)(CHOL_NB * CHOL_NB + (size_t)n * CHOL_NB) * 16));
    cudaError_t e;
#define ZH_CK(x) do { if ((e = (x)) != cudaSuccess) return FROB_ERR_CUDA; } while (0)
    count_launch();
    set_int_kernel<<<1, 1, 0, s>>>(info, INT_MAX);
    count_launch();
    zcopy_kernel<<<grid_for((long long)n * n), 256, 0, s>>>(reinterpret_cast<const double2 *>(Z), ldz, n, U, ld);
    ZH_CK(cudaGetLastError());
    ZH_CK(potrf_upper<double2>(n, U, ld, work, info, s));     // Z = U^H U
    ZH_CK(tri_inverses<double2>(n, U, nullptr, ld, T, s));     // K = U^{-1}
    ZH_CK(transpose<double2>(U, ld, Kh, ld, n, n, true, s));   // K^H
    {
        auto p = gemm_params<double2>(n, n, n, 1.0, U, ld, Kh, ld, 0.0, nullptr, ld, reinterpret_cast<double2 *>(X),
                                      ldx);
        p.triA = TRI_UPPER;
        p.triB = TRI_LOWER;
        ZH_CK(gemm_launch<double2>(p, 1, s));                 // X = K K^H
    }
    if (host_info) {
        int h = 0;
        ZH_CK(cudaMemcpyAsync(&h, info, sizeof(int), cudaMemcpyDeviceToHost, s));
        ZH_CK(cudaStreamSynchronize(s));
        *host_info = (h == INT_MAX) ? 0 : h;
        if (h != INT_MAX) return FROB_ERR_SINGULAR;
    }
    return FROB_OK;
#undef ZH_CK
}

}  // extern "C"
