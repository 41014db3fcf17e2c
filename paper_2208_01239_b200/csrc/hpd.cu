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
#include <utility>
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
FROB_DEV double shfl_mask(double v, int src, unsigned mask) { return __shfl_sync(mask, v, src); }
FROB_DEV double2 shfl_mask(double2 v, int src, unsigned mask) {
    return make_double2(__shfl_sync(mask, v.x, src), __shfl_sync(mask, v.y, src));
}
template <typename F, int... J>
FROB_DEV void bstatic_for_h_impl(F &&f, std::integer_sequence<int, J...>) {
    (f(std::integral_constant<int, J>{}), ...);
}
template <int K, typename F>
FROB_DEV void bstatic_for_h(F &&f) {
    bstatic_for_h_impl(f, std::make_integer_sequence<int, K>{});
}
FROB_DEV double from_real(double v, double) { return v; }

// Factor the diagonal block (k0, k0) in place (upper; zeros below inside the block) and write
// W^H = (U_kk^{-1})^H (lower triangular, CHOL_NB x CHOL_NB, ld CHOL_NB) to wh.  info: first
// 1-based column with a non-positive pivot (atomicMin; INT_MAX = none).
// The 64 x 64 block lives in REGISTERS: 256 threads as 16 x 16, thread (ti, tj) owns rows 4 ti ..,
// columns 4 tj .. (the column index inside a 4-block is static: the steps are unrolled by 4).
// Cholesky step j: the 16 threads of row j's block-row (one half-warp) take u_jj from the diagonal
// owner by a shuffle, scale their part of row j and publish it (double-buffered); ONE barrier; every
// thread applies the rank-1 update conj(U[j][r]) U[j][c] to its upper-triangle entries.  Then
// U_kk^{-1} in place by the exchange (Gauss-Jordan) sweep without pivoting -- u_jj is unchanged by
// earlier steps of an upper-triangular sweep, so 1 / u_jj comes from the factorisation -- again
// one barrier per step (column j and the scaled row j published together).
template <typename T>
__global__ void __launch_bounds__(256) chol_diag_kernel(T *__restrict__ A, long long ld, int n, int k0,
                                                        T *__restrict__ wh, int *__restrict__ info) {
    __shared__ T rowb[2][CHOL_NB], colb[2][CHOL_NB];
    __shared__ double rdiag[CHOL_NB];
    const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15, r0 = ti * 4, c0 = tj * 4;
    const int half = (tid & 31) & 16;
    const unsigned hmask = 0xffffu << half;
    const int nb = min(CHOL_NB, n - k0);
    T a[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int i = r0 + q, j = c0 + c;
            a[q][c] = (i < nb && j < nb) ? A[(long long)(k0 + i) * ld + k0 + j] : ((i == j) ? one_of(T()) : zero_of(T()));
        }
    // ---- factorisation
    for (int jb = 0; jb * 4 < nb; ++jb) {
        bstatic_for_h<4>([&](auto JQc) {
            constexpr int jq = decltype(JQc)::value;
            const int j = jb * 4 + jq;
            if (j >= nb) return;
            const int par = j & 1;
            if (ti == jb) {
                const double d = re_part(shfl_mask(a[jq][jq], half + jb, hmask));  // a[jq][jq] of thread (jb, jb)
                const double p = sqrt(d);  // NaN for a failed pivot: flagged through info
                const double ip = 1.0 / p;
                if (tj == jb) {
                    rdiag[j] = ip;
                    if (!(d > 0.0)) atomicMin(info, k0 + j + 1);
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int col = c0 + c;
                    const T u = (col > j) ? scal(a[jq][c], ip) : ((col == j) ? from_real(p, T()) : zero_of(T()));
                    a[jq][c] = u;
                    rowb[par][col] = u;
                }
            }
            __syncthreads();
            T ur[4], uc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) ur[q] = conj_of(rowb[par][r0 + q]);
#pragma unroll
            for (int c = 0; c < 4; ++c) uc[c] = rowb[par][c0 + c];
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (r0 + q > j && c0 + c >= r0 + q) a[q][c] = msub(a[q][c], ur[q], uc[c]);
        });
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int i = r0 + q, j = c0 + c;
            if (j < i) a[q][c] = zero_of(T());   // U: zeros below the diagonal
            if (i < nb && j < nb) A[(long long)(k0 + i) * ld + k0 + j] = a[q][c];
        }
    __syncthreads();  // rdiag complete
    // ---- U_kk^{-1} in place: exchange step with pivot (j, j), j = 0 .. nb-1
    for (int jb = 0; jb * 4 < nb; ++jb) {
        bstatic_for_h<4>([&](auto JQc) {
            constexpr int jq = decltype(JQc)::value;
            const int j = jb * 4 + jq;
            if (j >= nb) return;
            const int par = j & 1;
            const double ip = rdiag[j];
            if (tj == jb) {
#pragma unroll
                for (int q = 0; q < 4; ++q) colb[par][r0 + q] = a[q][jq];
            }
            if (ti == jb) {
#pragma unroll
                for (int c = 0; c < 4; ++c) rowb[par][c0 + c] = (c0 + c == j) ? from_real(ip, T()) : scal(a[jq][c], ip);
            }
            __syncthreads();
            T ck[4], rp[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) ck[q] = colb[par][r0 + q];
#pragma unroll
            for (int c = 0; c < 4; ++c) rp[c] = rowb[par][c0 + c];
            if (tj == jb) {
#pragma unroll
                for (int q = 0; q < 4; ++q) a[q][jq] = zero_of(T());
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int c = 0; c < 4; ++c) a[q][c] = msub(a[q][c], ck[q], rp[c]);
            if (ti == jb) {
#pragma unroll
                for (int c = 0; c < 4; ++c) a[jq][c] = rp[c];
            }
        });
    }
    // W^H: wh[i][j] = conj(W[j][i])  (W = U_kk^{-1}: upper; padding zero)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int i = r0 + q, j = c0 + c;
            wh[j * CHOL_NB + i] = (i < nb && j < nb && j >= i) ? conj_of(a[q][c]) : zero_of(T());
        }
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
        count_launch();
        chol_diag_kernel<T><<<1, 256, 0, s>>>(A, ld, n, k0, wh, info);
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
