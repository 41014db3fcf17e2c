// frob.cu -- single-matrix Frobenius inversion (Alg 1), the complex-LU
// comparator (Alg 3 over C), real inversion / GEMM / LU entry points, and the Newton
// drivers.  Host orchestration only; every arithmetic step runs in the kernels of
// gemm.cuh / lu.cu / this file.
#include <cstdio>
#include <cstring>
#include <cmath>
#include <climits>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <algorithm>
#include "lu.cuh"
#include "../../include/frobinv.h"

namespace frob {

static thread_local char g_last_cuda[256] = "";

// ---------------------------------------------------------------------- kernel profiler
struct ProfEv {
    const char *name;
    cudaEvent_t a, b;
    double work;
};
static std::mutex g_prof_mu;
static std::vector<ProfEv> g_prof;
static bool g_prof_on = false;
struct ProfOpen {
    const char *name;
    cudaEvent_t e;
    double work;
};
static std::vector<ProfOpen> g_prof_open;

bool prof_enabled() { return g_prof_on; }
thread_local const char *g_gemm_tag = nullptr;
void prof_record(const char *name, cudaStream_t s, bool begin, double work) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    if (begin) {
        g_prof_open.push_back({name, e, work});
    } else {
        for (size_t i = g_prof_open.size(); i-- > 0;) {
            if (g_prof_open[i].name == name) {
                g_prof.push_back({name, g_prof_open[i].e, e, g_prof_open[i].work});
                g_prof_open.erase(g_prof_open.begin() + (long)i);
                return;
            }
        }
        cudaEventDestroy(e);
    }
}

unsigned long long &launch_counter() {
    static unsigned long long c = 0;
    return c;
}

static frob_status cuda_fail(cudaError_t e) {
    snprintf(g_last_cuda, sizeof(g_last_cuda), "%s", cudaGetErrorString(e));
    return FROB_ERR_CUDA;
}
#define FROB_CUDA(x)                                   \
    do {                                               \
        cudaError_t _e = (x);                          \
        if (_e != cudaSuccess) return cuda_fail(_e);   \
    } while (0)

static long long ld_of(int n) { return ((long long)n + 7) / 8 * 8; }
static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// Bump allocator over the caller's workspace.
struct Carve {
    unsigned char *base;
    size_t off, cap;
    template <typename T>
    T *take(size_t count) {
        T *p = reinterpret_cast<T *>(base ? base + off : nullptr);
        off += align256(count * sizeof(T));
        return p;
    }
};

// ---------------------------------------------------------------------- elementwise
// a0: split interleaved Z (ldz) into planar A, B (ld) and a copy of the branch matrix
// mu != 0: Alg 5 line 2 -- the parts of (1 + mu i) Z: X = A - mu B, Y = mu A + B
__global__ void split_kernel(const double2 *__restrict__ Z, long long ldz, int n, double *__restrict__ A,
                             double *__restrict__ B, double *__restrict__ W, int wsel, long long ld,
                             int *__restrict__ nonfinite, double mu) {
    const long long total = (long long)n * n;
    int bad = 0;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        double2 z = Z[(long long)i * ldz + j];
        if (mu != 0.0) z = make_double2(z.x - mu * z.y, mu * z.x + z.y);
        bad |= !(isfinite(z.x) && isfinite(z.y));
        const long long o = (long long)i * ld + j;
        A[o] = z.x;
        B[o] = z.y;
        if (W) W[o] = (wsel == 2) ? z.y : z.x;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
}

template <typename T>
__global__ void copy2d_kernel(const T *__restrict__ src, long long lds, T *__restrict__ dst, long long ldd,
                              int n, int *__restrict__ nonfinite) {
    const long long total = (long long)n * n;
    int bad = 0;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const T v = src[(long long)i * lds + j];
        if (nonfinite) bad |= !finite_of(v);
        dst[(long long)i * ldd + j] = v;
    }
    if (nonfinite && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------------- AUTO rule R1'
// ||M||_inf = max_i sum_j |M[i][j]| of an n x n row-major matrix: one warp per row (lanes stride
// the columns, fixed-order shuffle sum), the maximum over rows by atomicMax on the bit patterns
// of the non-negative sums (order-independent, so the result is deterministic).  *out must be 0.
__global__ void __launch_bounds__(256) norm_inf_kernel(const double *__restrict__ M, long long ld, int n,
                                                       unsigned long long *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    double best = 0.0;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const double *row = M + (long long)i * ld;
        double s = 0.0;
        for (int j = lane; j < n; j += 32) s += fabs(row[j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        best = fmax(best, s);   // NaN rows are dropped here; non-finite input is flagged at ingest
    }
    if (lane == 0 && best > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(best));
}

// kappa_inf of a part from its norm slots (s0 = ||X||, s1, s2 = norms whose product bounds / equals
// ||X^{-1}||: s2 = NULL for the exact ||X^{-1}||), infinity when the LU flagged it singular
FROB_DEV double kappa_of(const unsigned long long *nrm, int i0, int i1, int i2, int singular) {
    if (singular) return INFINITY;
    double k = __longlong_as_double((long long)nrm[i0]) * __longlong_as_double((long long)nrm[i1]);
    if (i2 >= 0) k *= __longlong_as_double((long long)nrm[i2]);
    return k;
}

// norm slots in the workspace (u64 bit patterns of non-negative doubles)
enum { NRM_A = 0, NRM_AINV = 1, NRM_AL = 2, NRM_B = 3, NRM_BINV = 4, NRM_BL = 5, NRM_SLOTS = 8 };

// Reading R1' decided on the device (FROB_OPT_DEVICE_AUTO): both parts factored and inverted;
// flags[1] = 1 (S1), 2 (S2) or 0 (both singular)
__global__ void auto_select_kernel(const LuStats *__restrict__ st, const unsigned long long *__restrict__ nrm,
                                   int n, int *__restrict__ flags) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const bool sa = st[0].info != 0, sb = st[1].info != 0;
    const double ka = kappa_of(nrm, NRM_A, NRM_AINV, -1, sa);
    int use = 1;
    if (sa || !(ka <= kappa_switch(n))) {
        const double kb = kappa_of(nrm, NRM_B, NRM_BINV, -1, sb);
        use = (sa && sb) ? 0 : ((sa || (!sb && kb < ka)) ? 2 : 1);
    }
    flags[1] = use;
}

// flags[1] == 2: (A, B) <- (B, -A) in place, so the S1 code computes the S2 branch (X = B, Y = -A;
// every step is the rotated S1 step bitwise, reading R3)
__global__ void branch_rotate_kernel(double *__restrict__ A, double *__restrict__ B, long long ld, int n,
                                     const int *__restrict__ flags) {
    if (flags[1] != 2) return;
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const long long o = (long long)i * ld + j;
        const double t = A[o];
        A[o] = B[o];
        B[o] = -t;
    }
}

// flags[1] == 2: dst <- src (the S2 inverse / permutation move into the S1 slots)
template <typename T>
__global__ void cond_copy_kernel(const T *__restrict__ src, T *__restrict__ dst, long long count,
                                 const int *__restrict__ flags) {
    if (flags[1] != 2) return;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < count;
         idx += (long long)gridDim.x * blockDim.x)
        dst[idx] = src[idx];
}

// Device status record of one call (frob_inv_dev / frob_inv_host_many's per-matrix status):
// use_host = branch chosen on the host (1 | 2), or 0 = read flags[1] (device AUTO);
// factored: bit 0 = LU(A) ran, bit 1 = LU(B) ran; kfused: kappa from ||U^-1|| ||L^-1|| (NEXT-1).
__global__ void finalize_status_kernel(const LuStats *__restrict__ st, const int *__restrict__ flags,
                                       const unsigned long long *__restrict__ nrm, int use_host, int factored,
                                       int kfused, int forced_status, frob_dev_status *__restrict__ out,
                                       int *__restrict__ status_copy) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int use = use_host ? use_host : flags[1];
    int status = FROB_OK, info = 0;
    if (forced_status) {
        status = forced_status;
    } else if (flags[0]) {
        status = FROB_ERR_NONFINITE;
    } else if (use == 0) {
        status = FROB_ERR_BOTH_SINGULAR;
        info = st[0].info;
    } else {
        const int ix = st[use - 1].info;
        info = ix ? ix : st[2].info;
        status = info ? FROB_ERR_SINGULAR : FROB_OK;
    }
    if (out) {
        frob_dev_status r;
        r.status = status;
        r.info = info;
        r.branch_used = (status == FROB_ERR_BOTH_SINGULAR || forced_status) ? 0 : use;
        r.nonfinite = flags[0];
        r.rho_a = (factored & 1) ? st[0].rho : NAN;
        r.rho_b = (factored & 2) ? st[1].rho : NAN;
        r.rho_m = (use && !forced_status) ? st[2].rho : NAN;
        r.kappa_a = (factored & 1) ? kappa_of(nrm, NRM_A, NRM_AINV, kfused ? NRM_AL : -1, st[0].info) : NAN;
        r.kappa_b = (factored & 2) ? kappa_of(nrm, NRM_B, NRM_BINV, kfused ? NRM_BL : -1, st[1].info) : NAN;
        *out = r;
    }
    if (status_copy) *status_copy = status;
}

static int ew_blocks(long long total) {
    return (int)std::min<long long>((total + 255) / 256, 148LL * 8);
}

// ---------------------------------------------------------------------- workspace
struct FrobWs {
    double *A, *B, *W1, *W2, *W3, *W4, *W5, *W6, *W7;  // W6, W7: n <= LU2_MAX_N only
    double *diag, *work;
    double *vec;      // 3 n-vectors: NEXT-1's estimate of ||X^{-1}||_inf (Hager-Higham)
    int *perm_x, *perm_b, *perm_m, *mv, *iw;
    LuStats *stats;   // [0] A, [1] B, [2] M
    int *flags;       // [0] nonfinite, [1] device-AUTO branch, [2] GEMM tile counter
    unsigned long long *nrm;  // NRM_* slots (inside the flags block: one memset clears both)
    size_t bytes;
};

static FrobWs carve_frob(void *ws, int n) {
    const long long ld = ld_of(n);
    Carve c{reinterpret_cast<unsigned char *>(ws), 0, 0};
    FrobWs w{};
    w.A = c.take<double>((size_t)n * ld);
    w.B = c.take<double>((size_t)n * ld);
    w.W1 = c.take<double>((size_t)n * ld);
    w.W2 = c.take<double>((size_t)n * ld);
    w.W3 = c.take<double>((size_t)n * ld);
    w.W4 = c.take<double>((size_t)n * ld);
    w.W5 = c.take<double>((size_t)n * ld);
    const bool small = n <= lu2_max_n();
    w.W6 = small ? c.take<double>((size_t)n * ld) : nullptr;
    w.W7 = small ? c.take<double>((size_t)n * ld) : nullptr;
    w.diag = c.take<double>((size_t)n);
    w.work = c.take<double>(getrf_work_elems<double>(n));
    w.vec = c.take<double>(3 * (size_t)ld_of(n));
    w.perm_x = c.take<int>((size_t)n);
    w.perm_b = c.take<int>((size_t)n);
    w.perm_m = c.take<int>((size_t)n);
    w.mv = c.take<int>(lu_mv_ints(n));
    w.iw = small ? c.take<int>(lu2_int_elems(n)) : nullptr;
    w.stats = c.take<LuStats>(3);
    w.flags = c.take<int>(64);  // 256 bytes: flags[0..31] + NRM_SLOTS u64 norm slots
    w.nrm = w.flags ? reinterpret_cast<unsigned long long *>(w.flags + 32) : nullptr;
    w.bytes = c.off;
    return w;
}

struct ZluWs {
    double2 *W, *U, *L, *W2, *diag, *work;  // W2: n <= LU2_MAX_N only
    int *perm, *mv, *iw;
    LuStats *stats;
    int *flags;
    size_t bytes;
};

static ZluWs carve_zlu(void *ws, int n) {
    const long long ld = ld_of(n);
    Carve c{reinterpret_cast<unsigned char *>(ws), 0, 0};
    ZluWs w{};
    w.W = c.take<double2>((size_t)n * ld);
    w.U = c.take<double2>((size_t)n * ld);
    w.L = c.take<double2>((size_t)n * ld);
    const bool small = n <= lu2_max_n();
    w.W2 = small ? c.take<double2>((size_t)n * ld) : nullptr;
    w.diag = c.take<double2>((size_t)n);
    w.work = c.take<double2>(getrf_work_elems<double2>(n));
    w.perm = c.take<int>((size_t)n);
    w.mv = c.take<int>(lu_mv_ints(n));
    w.iw = small ? c.take<int>(lu2_int_elems(n)) : nullptr;
    w.stats = c.take<LuStats>(1);
    w.flags = c.take<int>(4);
    w.bytes = c.off;
    return w;
}

static bool overlap(const void *a, size_t na, const void *b, size_t nb) {
    const char *x = (const char *)a, *y = (const char *)b;
    return x < y + nb && y < x + na;
}

// ---------------------------------------------------------------------- frob_inv
// Optional outputs of one call: a device status record and/or a device int receiving the status
// (frob_inv_host_many's per-matrix status), both written by finalize_status_kernel.
struct StatusOut {
    frob_dev_status *rec = nullptr;
    int *code = nullptr;
    bool any() const { return rec || code; }
};
// Optional row-block split of the final GEMM (a6): chunk c (rows [c rows_per, ...)) records ev[c]
// on the stream when stored, so a caller can copy it out while the next chunk is computed.
struct OutChunks {
    int k = 1;
    cudaEvent_t *ev = nullptr;
};

static cudaError_t finalize_status(const FrobWs &w, int use_host, int factored, bool kfused, int forced,
                                   StatusOut so, cudaStream_t s) {
    if (!so.any()) return cudaSuccess;
    count_launch();
    finalize_status_kernel<<<1, 32, 0, s>>>(w.stats, w.flags, w.nrm, use_host, factored, kfused ? 1 : 0, forced,
                                            so.rec, so.code);
    return cudaGetLastError();
}

static cudaError_t norm_inf(const double *M, long long ld, int n, unsigned long long *slot, cudaStream_t s) {
    count_launch();
    const int blocks = (int)std::min<long long>(((long long)n * 32 + 255) / 256, 148LL * 4);
    norm_inf_kernel<<<blocks, 256, 0, s>>>(M, ld, n, slot);
    return cudaGetLastError();
}

static double nrm_val(unsigned long long v) {
    double d;
    std::memcpy(&d, &v, sizeof(d));
    return d;
}

// ---------------------------------------------------------------------- NEXT-1 triangular solves
// The paper's fused first step (Thm 5.1 proof) solves with the LU factors instead of
// forming X^{-1}: L G = P Y, U C = G.  Blocked substitution on the GEMM engine: the NB x NB diagonal
// blocks of L and U are inverted in place once (tri_inverses on each block; their strict off-block
// parts stay the factors), then block row k: X_k = T_kk^{-1} W_k (triangular-operand GEMM) and the
// not-yet-solved block rows W -= T_{.,k} X_k (K = NB GEMM).  NB = 2048 (A/B at n = 2048 ... 16384:
// 256 / 512 / 1024 / 2048 / 4096 -> 1368 / 1308 / 1284 / 1278 / 1279 ms at n = 16384).  n^3 flops per solve with n right-hand
// sides, so the fused step costs 2/3 n^3 (LU) + 2 n^3 = the paper's T_inv + lambda T_mult.
#ifndef FROB_TRSM_NB  // A/B build knob (tools/build_variant.sh)
#define FROB_TRSM_NB 2048
#endif
constexpr int TRSM_NB = FROB_TRSM_NB;

static cudaError_t block_diag_invert(int n, double *U, double *L, long long ld, double *tmp, cudaStream_t s) {
    for (int r0 = 0; r0 < n; r0 += TRSM_NB) {
        const int rk = std::min(TRSM_NB, n - r0);
        const cudaError_t e = tri_inverses<double>(rk, U + (long long)r0 * ld + r0, L ? L + (long long)r0 * ld + r0 : nullptr,
                                                   ld, tmp, s);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Solve T X = W (T n x n triangular, its TRSM_NB diagonal blocks inverted by block_diag_invert; W n x m,
// destroyed; X n x m).  lower: forward substitution by block rows, else backward.
static cudaError_t trsm_blocked(int n, int m, const double *T, long long ldt, bool lower, double *W, long long ldw,
                                double *X, long long ldx, cudaStream_t s) {
    const int nb = (n + TRSM_NB - 1) / TRSM_NB;
    cudaError_t e;
    for (int step = 0; step < nb; ++step) {
        const int kb = lower ? step : nb - 1 - step;
        const int r0 = kb * TRSM_NB, rk = std::min(TRSM_NB, n - r0);
        auto p = gemm_params<double>(rk, m, rk, 1.0, T + (long long)r0 * ldt + r0, ldt, W + (long long)r0 * ldw, ldw,
                                     0.0, nullptr, ldx, X + (long long)r0 * ldx, ldx);
        p.triA = lower ? TRI_LOWER : TRI_UPPER;
        if ((e = gemm_launch<double>(p, 1, s)) != cudaSuccess) return e;
        const int u0 = lower ? r0 + rk : 0, ur = lower ? n - r0 - rk : r0;  // rows still to solve
        if (ur > 0) {
            auto q = gemm_params<double>(ur, m, rk, -1.0, T + (long long)u0 * ldt + r0, ldt, X + (long long)r0 * ldx,
                                         ldx, 1.0, W + (long long)u0 * ldw, ldw, W + (long long)u0 * ldw, ldw);
            if ((e = gemm_launch<double>(q, 1, s)) != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

// dst (n x n, ldd) = src^T
__global__ void __launch_bounds__(256) transpose_d_kernel(const double *__restrict__ src, long long lds,
                                                          double *__restrict__ dst, long long ldd, int n) {
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int tiles = (n + 31) / 32;
    for (int t = blockIdx.x; t < tiles * tiles; t += gridDim.x) {
        const int bi = t / tiles, bj = t % tiles;
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int i = bi * 32 + r, j = bj * 32 + tx;
            if (i < n && j < n) tile[r][tx] = src[(long long)i * lds + j];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {
            const int i = bj * 32 + r, j = bi * 32 + tx;
            if (i < n && j < n) dst[(long long)i * ldd + j] = tile[tx][r];
        }
    }
}

// out[i][j] = sgn * Y[perm[i]][j]  (P Y, with the S2 sign): one row per block iteration, 16-byte
// accesses (ld even, rows 16-byte aligned: workspace matrices)
__global__ void __launch_bounds__(256) gather_rows_signed_kernel(const double *__restrict__ Y, long long ld,
                                                                 const int *__restrict__ perm, double sgn, int n,
                                                                 double *__restrict__ out) {
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const double2 *src = reinterpret_cast<const double2 *>(Y + (long long)perm[i] * ld);
        double2 *dst = reinterpret_cast<double2 *>(out + (long long)i * ld);
        for (int c = threadIdx.x; c < n / 2; c += blockDim.x) {
            const double2 v = src[c];
            dst[c] = make_double2(sgn * v.x, sgn * v.y);
        }
        if ((n & 1) && threadIdx.x == 0) out[(long long)i * ld + n - 1] = sgn * Y[(long long)perm[i] * ld + n - 1];
    }
}
static int gather_blocks(int n) { return std::min(n, 148 * 8); }

// ||X^{-1}||_inf for NEXT-1, which never forms X^{-1} (R1'): the Hager-Higham estimate (LAPACK
// dlacon's iteration, at most 5 steps) of ||B||_1 for B = X^{-T} = P^T L^{-T} U^{-T}, by blocked
// solves with the factors (U, L: diagonal blocks inverted) and their transposes (Ut = U^T lower,
// Lt = L^T upper); perm: (P Y)[i] = Y[perm[i]].  A lower bound of the exact norm (exact for most
// matrices); synchronises per step.
static frob_status inv_norm_estimate(int n, const double *U, const double *L, const double *Ut, const double *Lt,
                                     long long ld, const int *perm, double *vec, cudaStream_t s, double *out) {
    const long long lv = ld_of(n);
    double *v0 = vec, *v1 = vec + lv, *v2 = vec + 2 * lv;
    std::vector<int> hp(n);
    std::vector<double> x(n, 1.0 / n), y(n), t(n), z(n);
    FROB_CUDA(cudaMemcpyAsync(hp.data(), perm, n * sizeof(int), cudaMemcpyDeviceToHost, s));
    GemmTag tag("gemm:inv_norm_est");
    auto apply_B = [&](const std::vector<double> &in, std::vector<double> &o) -> frob_status {  // o = X^{-T} in
        FROB_CUDA(cudaMemcpyAsync(v0, in.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
        FROB_CUDA(trsm_blocked(n, 1, Ut, ld, true, v0, 1, v1, 1, s));    // U^T w = in
        FROB_CUDA(trsm_blocked(n, 1, Lt, ld, false, v1, 1, v2, 1, s));   // L^T v = w
        FROB_CUDA(cudaMemcpyAsync(t.data(), v2, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < n; ++i) o[hp[i]] = t[i];  // P^T
        return FROB_OK;
    };
    auto apply_BT = [&](const std::vector<double> &in, std::vector<double> &o) -> frob_status {  // o = X^{-1} in
        for (int i = 0; i < n; ++i) t[i] = in[hp[i]];  // P in
        FROB_CUDA(cudaMemcpyAsync(v0, t.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
        FROB_CUDA(trsm_blocked(n, 1, L, ld, true, v0, 1, v1, 1, s));
        FROB_CUDA(trsm_blocked(n, 1, U, ld, false, v1, 1, v2, 1, s));
        FROB_CUDA(cudaMemcpyAsync(o.data(), v2, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaStreamSynchronize(s));
        return FROB_OK;
    };
    double est = 0.0;
    int jlast = -1;
    for (int it = 0; it < 5; ++it) {
        frob_status st = apply_B(x, y);
        if (st != FROB_OK) return st;
        double e1 = 0.0;
        for (int i = 0; i < n; ++i) e1 += std::fabs(y[i]);
        if (it > 0 && e1 <= est) break;  // no increase: converged
        est = e1;
        std::vector<double> xi(n);
        for (int i = 0; i < n; ++i) xi[i] = (y[i] >= 0.0) ? 1.0 : -1.0;
        if ((st = apply_BT(xi, z)) != FROB_OK) return st;
        int j = 0;
        double zx = 0.0;
        for (int i = 0; i < n; ++i) {
            if (std::fabs(z[i]) > std::fabs(z[j])) j = i;
            zx += z[i] * x[i];
        }
        if (std::fabs(z[j]) <= zx || j == jlast) break;
        jlast = j;
        std::fill(x.begin(), x.end(), 0.0);
        x[j] = 1.0;
    }
    // Higham's safeguard vector: x_i = (-1)^i (1 + i / (n - 1))
    std::vector<double> xa(n);
    for (int i = 0; i < n; ++i) xa[i] = ((i & 1) ? -1.0 : 1.0) * (1.0 + (n > 1 ? (double)i / (n - 1) : 0.0));
    frob_status st = apply_B(xa, y);
    if (st != FROB_OK) return st;
    double ea = 0.0;
    for (int i = 0; i < n; ++i) ea += std::fabs(y[i]);
    *out = std::max(est, 2.0 * ea / (3.0 * n));
    return FROB_OK;
}

static frob_status frob_inv_impl(int n, const double *Z, long long ldz, double *X, long long ldx,
                                 int branch, void *ws, size_t ws_bytes, cudaStream_t s,
                                 frob_info *host_info, double mu = 0.0, bool fused = false,
                                 bool dev_auto = false, StatusOut so = StatusOut(), OutChunks oc = OutChunks()) {
    if (n < 1 || !Z || !X || ldz < n || ldx < n || branch < 0 || branch > 2) return FROB_ERR_INVALID_ARG;
    if (dev_auto && (branch != FROB_BRANCH_AUTO || fused)) return FROB_ERR_INVALID_ARG;
    if (overlap(Z, (size_t)((n - 1) * ldz + n) * 16, X, (size_t)((n - 1) * ldx + n) * 16))
        return FROB_ERR_INVALID_ARG;
    FrobWs w = carve_frob(nullptr, n);
    if (!ws || ws_bytes < w.bytes) return FROB_ERR_WORKSPACE;
    w = carve_frob(ws, n);
    const long long ld = ld_of(n);
    const long long mat = (long long)n * ld;
    const double2 *Zc = reinterpret_cast<const double2 *>(Z);
    const bool small = n <= lu2_max_n();  // latency-oriented LU (lu2.cu), factors come out split (U, L)
    const bool autob = branch == FROB_BRANCH_AUTO;

    FROB_CUDA(cudaMemsetAsync(w.flags, 0, 64 * sizeof(int), s));
    // a0: ingest (W1 = copy of the first branch matrix for its LU)
    count_launch();
    // (the literal path factors B from W5, NEXT-1 every part from W1)
    split_kernel<<<ew_blocks((long long)n * n), 256, 0, s>>>(Zc, ldz, n, w.A, w.B,
                                                             (!fused && branch == FROB_BRANCH_B) ? w.W5 : w.W1,
                                                             branch == FROB_BRANCH_B ? 2 : 1, ld, w.flags, mu);
    FROB_CUDA(cudaGetLastError());

    int use = (branch == FROB_BRANCH_B) ? 2 : 1;
    int factored = 0;                 // bit 0: LU(A) ran, bit 1: LU(B) ran
    int *perm = w.perm_x;             // perm of the chosen part's LU
    double *Xinv = w.W4;              // a2 output: Xinv' = U^{-1} L^{-1} (X^{-1} = Xinv' P)
    double *Uf = w.W2, *Lf = w.W3;    // NEXT-1: U^{-1}, L^{-1} of the chosen part

    // a1 + a2 for part u (1 = A, 2 = B) of the literal path: LU, then Xinv' into `out`.
    //   u = 1: LU input W1 (written by split), lu2 ping-pong W4 -> (W2, W3) | getrf in place W1;
    //          inverse into W4 (scratch W1 | W2, W3)
    //   u = 2: LU input W5 (copy of B), lu2 ping-pong W1 -> (W6, W7) | getrf in place W5;
    //          inverse into W1 (scratch W5 | W2, W3)
    auto lit_part = [&](int u, bool copy_in) -> frob_status {
        double *in = (u == 1) ? w.W1 : w.W5;
        int *pm = (u == 1) ? w.perm_x : w.perm_b;
        if (copy_in) {
            count_launch();
            copy2d_kernel<double><<<ew_blocks((long long)n * n), 256, 0, s>>>(u == 1 ? w.A : w.B, ld, in, ld, n,
                                                                              nullptr);
            FROB_CUDA(cudaGetLastError());
        }
        // EarlyInv scratch: a buffer idle from the LU's start to the end of the inverse (W5 before
        // part 2 copies B there; W2 holds only part 1's spent factors then)
        EarlyInv ei;
        ei.h = small ? early_inv_h(n) : 0;
        ei.vbuf = (u == 1) ? w.W5 : w.W2;
        if (!small && getrf_early_ok(n) && u == 1) {  // getrf's EarlyInv: the split factors go to W2, W3
            ei.vbuf = w.W5;  // (part 2 has no idle matrix: A's inverse in W4 may still be the one kept)
            ei.U = w.W2;
            ei.L = w.W3;
        }
        {
            ProfScope ps("step:lu", s);
            if (small) FROB_CUDA(lu2_factor<double>(n, in, u == 1 ? w.W4 : w.W1, ld, u == 1 ? w.W2 : w.W6,
                                                    u == 1 ? w.W3 : w.W7, ld, pm, w.iw, w.diag, &w.stats[u - 1], s,
                                                    &ei));
            else FROB_CUDA(getrf<double>(n, in, ld, pm, w.mv, w.diag, &w.stats[u - 1], w.work, s, &ei));
        }
        factored |= u;
        ProfScope ps("step:inv_from_lu", s);
        if (small) {
            if (u == 1) FROB_CUDA(inv_from_ul<double>(n, w.W2, w.W3, ld, w.W1, w.W4, ld, nullptr, w.flags + 2, s, &ei));
            else FROB_CUDA(inv_from_ul<double>(n, w.W6, w.W7, ld, w.W5, w.W1, ld, nullptr, w.flags + 2, s, &ei));
        } else {
            FROB_CUDA(inv_from_lu<double>(n, in, ld, w.W2, w.W3, u == 1 ? w.W4 : w.W1, ld, nullptr, w.flags + 2, s,
                                          &ei));
        }
        return FROB_OK;
    };
    // NEXT-1 a1 + triangular inverses of part u into (W2, W3), perm_x (the same slots for both
    // parts: a switch recomputes)
    auto fused_part = [&](int u, bool copy_in) -> frob_status {
        if (copy_in) {
            count_launch();
            copy2d_kernel<double><<<ew_blocks((long long)n * n), 256, 0, s>>>(u == 1 ? w.A : w.B, ld, w.W1, ld, n,
                                                                              nullptr);
            FROB_CUDA(cudaGetLastError());
        }
        {
            ProfScope ps("step:lu", s);
            if (small) FROB_CUDA(lu2_factor<double>(n, w.W1, w.W4, ld, w.W2, w.W3, ld, w.perm_x, w.iw, w.diag,
                                                    &w.stats[u - 1], s));
            else {
                FROB_CUDA(getrf<double>(n, w.W1, ld, w.perm_x, w.mv, w.diag, &w.stats[u - 1], w.work, s));
                FROB_CUDA(extract_ul<double>(n, w.W1, ld, w.W2, w.W3, s));
            }
        }
        factored |= u;
        FROB_CUDA(block_diag_invert(n, w.W2, w.W3, ld, w.W1, s));
        return FROB_OK;
    };
    // norms of part u for kappa_inf (R1'): ||X|| and ||Xinv'|| (literal) or ||U^-1||, ||L^-1|| (NEXT-1)
    auto part_norms = [&](int u, const double *xinv) -> frob_status {
        const int o = (u == 1) ? 0 : 3;
        FROB_CUDA(norm_inf(u == 1 ? w.A : w.B, ld, n, w.nrm + NRM_A + o, s));
        if (!fused) {
            FROB_CUDA(norm_inf(xinv, ld, n, w.nrm + NRM_AINV + o, s));
        } else {
            // NEXT-1: the Hager-Higham estimate of ||X^{-1}||_inf from U^{-1}, L^{-1} (host loop),
            // written into the same slot (bit pattern of a non-negative double)
            double e = 0.0;
            count_launch(2);
            const int tb = (int)std::min<long long>((long long)((n + 31) / 32) * ((n + 31) / 32), 148LL * 8);
            transpose_d_kernel<<<tb, 256, 0, s>>>(w.W2, ld, w.W4, ld, n);  // U^T (lower)
            transpose_d_kernel<<<tb, 256, 0, s>>>(w.W3, ld, w.W5, ld, n);  // L^T (upper)
            FROB_CUDA(cudaGetLastError());
            const frob_status st = inv_norm_estimate(n, w.W2, w.W3, w.W4, w.W5, ld, w.perm_x, w.vec, s, &e);
            if (st != FROB_OK) return st;
            unsigned long long bits;
            std::memcpy(&bits, &e, sizeof(bits));
            FROB_CUDA(cudaMemcpyAsync(w.nrm + NRM_AINV + o, &bits, sizeof(bits), cudaMemcpyHostToDevice, s));
            FROB_CUDA(cudaStreamSynchronize(s));  // `bits` lives on this stack frame
        }
        return FROB_OK;
    };
    auto part = [&](int u, bool copy_in) { return fused ? fused_part(u, copy_in) : lit_part(u, copy_in); };
#define FROB_ST(x) do { const frob_status _s = (x); if (_s != FROB_OK) return _s; } while (0)

    FROB_ST(part(use, false));
    if (use == 2 && !fused) {  // forced S2: B's inverse and permutation
        perm = w.perm_b;
        Xinv = w.W1;
    }
    LuStats hs[3];
    for (auto &h : hs) { h.rho = NAN; h.umax = 0; h.info = 0; h.nonfinite = 0; }
    int hflags[2] = {0, 0};
    unsigned long long hn[NRM_SLOTS] = {0};
    double kap[2] = {NAN, NAN};
    auto kappa_host = [&](int u) {
        const int o = (u == 1) ? 0 : 3;
        if (hs[u - 1].info) return (double)INFINITY;
        return nrm_val(hn[NRM_A + o]) * nrm_val(hn[NRM_AINV + o]);
    };
    if (autob && !dev_auto) {
        // a1' (reading R1'): kappa_inf(A) from the computed inverse (or NEXT-1's triangular inverses),
        // one small device->host read
        FROB_ST(part_norms(1, w.W4));
        FROB_CUDA(cudaMemcpyAsync(&hs[0], &w.stats[0], sizeof(LuStats), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaMemcpyAsync(hflags, w.flags, sizeof(int), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaMemcpyAsync(hn, w.nrm, sizeof(hn), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaStreamSynchronize(s));
        if (hflags[0]) {
            if (host_info) { host_info->info = 0; host_info->branch_used = 0; }
            FROB_CUDA(finalize_status(w, 1, factored, false, FROB_ERR_NONFINITE, so, s));
            return FROB_ERR_NONFINITE;
        }
        kap[0] = kappa_host(1);
        if (hs[0].info != 0 || !(kap[0] <= kappa_switch(n))) {
            FROB_ST(part(2, true));
            FROB_ST(part_norms(2, w.W1));
            FROB_CUDA(cudaMemcpyAsync(&hs[1], &w.stats[1], sizeof(LuStats), cudaMemcpyDeviceToHost, s));
            FROB_CUDA(cudaMemcpyAsync(hn, w.nrm, sizeof(hn), cudaMemcpyDeviceToHost, s));
            FROB_CUDA(cudaStreamSynchronize(s));
            kap[1] = kappa_host(2);
            const bool sa = hs[0].info != 0, sb = hs[1].info != 0;
            if (sa && sb) {
                if (host_info) {
                    host_info->info = hs[0].info; host_info->branch_used = 0;
                    host_info->rho_a = hs[0].rho; host_info->rho_b = hs[1].rho; host_info->rho_m = NAN;
                    host_info->kappa_a = kap[0]; host_info->kappa_b = kap[1];
                }
                FROB_CUDA(finalize_status(w, 1, factored, false, FROB_ERR_BOTH_SINGULAR, so, s));
                return FROB_ERR_BOTH_SINGULAR;
            }
            if (sa || (!sb && kap[1] < kap[0])) {
                use = 2;
                perm = w.perm_b;
                Xinv = w.W1;
            } else if (fused) {
                FROB_ST(part(1, true));  // NEXT-1 keeps one set of slots: back to A
            }
        }
    } else if (dev_auto) {
        // a1' on the device: both parts factored and inverted, the decision in a one-thread kernel,
        // B's inverse / permutation and the rotated parts (B, -A) moved into the S1 slots by
        // predicated kernels (no host read)
        FROB_ST(part_norms(1, w.W4));
        FROB_ST(part(2, true));
        FROB_ST(part_norms(2, w.W1));
        count_launch(4);
        auto_select_kernel<<<1, 32, 0, s>>>(w.stats, w.nrm, n, w.flags);
        cond_copy_kernel<double><<<ew_blocks(mat), 256, 0, s>>>(w.W1, w.W4, mat, w.flags);
        cond_copy_kernel<int><<<ew_blocks(n), 256, 0, s>>>(w.perm_b, w.perm_x, n, w.flags);
        branch_rotate_kernel<<<ew_blocks((long long)n * n), 256, 0, s>>>(w.A, w.B, ld, n, w.flags);
        FROB_CUDA(cudaGetLastError());
    } else if (so.any() || host_info) {
        FROB_ST(part_norms(use, Xinv));  // kappa of the forced part (reported only)
    }
    const double *Xm = (use == 1) ? w.A : w.B;   // X of Alg 1
    const double *Ym = (use == 1) ? w.B : w.A;   // Y of Alg 1 (S2 uses Y = -A via sgn)
    const double sgn = (use == 1) ? 1.0 : -1.0;

    double *Cb;  // C = X^{-1} Y
    if (!fused) {
        // a3: C = X^{-1} Y = Xinv' (P Y): P Y gathered into W5 first (free here in every branch) --
        // a plain GEMM instead of a per-stage row lookup (n = 16384: 32.4 -> 34.2 TF/s)
        Cb = w.W2;
        count_launch();
        gather_rows_signed_kernel<<<gather_blocks(n), 256, 0, s>>>(Ym, ld, perm, sgn, n, w.W5);
        FROB_CUDA(cudaGetLastError());
        auto p = gemm_params<double>(n, n, n, 1.0, Xinv, ld, w.W5, ld, 0.0, nullptr, ld, Cb, ld);
        GemmTag tag("gemm:frob_C");
        FROB_CUDA(gemm_launch<double>(p, 1, s));
    } else {
        // a2+a3 fused (NEXT-1): L G = P Y, U C = G by blocked substitution; X^{-1} is
        // never formed (W4 = sgn P Y, G -> W5, C -> W1)
        count_launch();
        gather_rows_signed_kernel<<<gather_blocks(n), 256, 0, s>>>(Ym, ld, w.perm_x, sgn, n, w.W4);
        FROB_CUDA(cudaGetLastError());
        GemmTag tag("gemm:frob_trsm");
        FROB_CUDA(trsm_blocked(n, n, Lf, ld, true, w.W4, ld, w.W5, ld, s));
        Cb = w.W1;
        FROB_CUDA(trsm_blocked(n, n, Uf, ld, false, w.W5, ld, Cb, ld, s));
    }
    // a4: M = X + Y C
    {
        auto p = gemm_params<double>(n, n, n, sgn, Ym, ld, Cb, ld, 1.0, Xm, ld, w.W3, ld);
        GemmTag tag("gemm:frob_M");
        FROB_CUDA(gemm_launch<double>(p, 1, s));
    }
    // a5: Re' = M^{-1} (un-permuted); scratch: the two buffers not holding C
    double *Re = (use == 1) ? w.A : w.B;  // X buffer is free now
    double *Sa = fused ? w.W2 : w.W1;
    if (small) {
        EarlyInv ei;  // scratch: Re (X's buffer, idle until the product writes it)
        ei.h = early_inv_h(n);
        ei.vbuf = Re;
        {
            ProfScope ps("step:lu", s);
            FROB_CUDA(lu2_factor<double>(n, w.W3, Sa, ld, w.W4, w.W5, ld, w.perm_m, w.iw, w.diag, &w.stats[2], s,
                                         &ei));
        }
        ProfScope ps("step:inv_from_lu", s);
        FROB_CUDA(inv_from_ul<double>(n, w.W4, w.W5, ld, w.W3, Re, ld, nullptr, w.flags + 2, s, &ei));
    } else {
        EarlyInv ei;  // getrf's EarlyInv (4096 < n <= 8192): scratch Re, split factors Sa / W4
        if (getrf_early_ok(n)) {
            ei.vbuf = Re;
            ei.U = Sa;
            ei.L = w.W4;
        }
        {
            ProfScope ps("step:lu", s);
            FROB_CUDA(getrf<double>(n, w.W3, ld, w.perm_m, w.mv, w.diag, &w.stats[2], w.work, s, &ei));
        }
        ProfScope ps("step:inv_from_lu", s);
        FROB_CUDA(inv_from_lu<double>(n, w.W3, ld, Sa, w.W4, Re, ld, nullptr, w.flags + 2, s, &ei));
    }
    // a6/a7: Im' = -C Re', fused with the column interchanges and the interleaved store
    {
        const int per = (oc.k > 1) ? (int)(((long long)n + oc.k - 1) / oc.k + 63) / 64 * 64 : n;
        for (int r0 = 0, c = 0; r0 < n; r0 += per, ++c) {
            const int rc = std::min(per, n - r0);
            auto p = gemm_params<double>(rc, n, n, -1.0, Cb + (long long)r0 * ld, ld, Re, ld, 0.0,
                                         Re + (long long)r0 * ld, ld, X + 2 * (long long)r0 * ldx, ldx);
            p.epi = (use == 1) ? EPI_FROB_A : EPI_FROB_B;
            p.dbranch = dev_auto ? w.flags + 1 : nullptr;
            p.colperm = w.perm_m;
            p.mu = mu;  // Alg 5 line 5: Z^{-1} = (1 + mu i) W
            GemmTag tag("gemm:frob_Im");
            FROB_CUDA(gemm_launch<double>(p, 1, s));
            if (oc.ev && c < oc.k) FROB_CUDA(cudaEventRecord(oc.ev[c], s));
        }
    }
    FROB_CUDA(finalize_status(w, dev_auto ? 0 : use, factored, false, 0, so, s));
    if (host_info) {
        FROB_CUDA(cudaMemcpyAsync(hs, w.stats, 3 * sizeof(LuStats), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaMemcpyAsync(hflags, w.flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaMemcpyAsync(hn, w.nrm, sizeof(hn), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaStreamSynchronize(s));
        if (dev_auto) use = hflags[1];
        if (hflags[0]) {
            host_info->info = 0;
            host_info->branch_used = 0;
            return FROB_ERR_NONFINITE;
        }
        host_info->rho_a = (factored & 1) ? hs[0].rho : NAN;
        host_info->rho_b = (factored & 2) ? hs[1].rho : NAN;
        host_info->kappa_a = (factored & 1) ? kappa_host(1) : NAN;
        host_info->kappa_b = (factored & 2) ? kappa_host(2) : NAN;
        if (use == 0) {
            host_info->info = hs[0].info;
            host_info->branch_used = 0;
            host_info->rho_m = NAN;
            return FROB_ERR_BOTH_SINGULAR;
        }
        host_info->branch_used = use;
        host_info->rho_m = hs[2].rho;
        const int ix = (use == 1) ? hs[0].info : hs[1].info;
        host_info->info = ix ? ix : hs[2].info;
        if (host_info->info) return FROB_ERR_SINGULAR;
    }
    return FROB_OK;
#undef FROB_ST
}

// ---------------------------------------------------------------------- zinv_lu
static frob_status zinv_lu_impl(int n, const double *Z, long long ldz, double *X, long long ldx,
                                void *ws, size_t ws_bytes, cudaStream_t s, int *host_info) {
    if (n < 1 || !Z || !X || ldz < n || ldx < n) return FROB_ERR_INVALID_ARG;
    if (overlap(Z, (size_t)((n - 1) * ldz + n) * 16, X, (size_t)((n - 1) * ldx + n) * 16))
        return FROB_ERR_INVALID_ARG;
    ZluWs w = carve_zlu(nullptr, n);
    if (!ws || ws_bytes < w.bytes) return FROB_ERR_WORKSPACE;
    w = carve_zlu(ws, n);
    const long long ld = ld_of(n);
    FROB_CUDA(cudaMemsetAsync(w.flags, 0, 4 * sizeof(int), s));
    count_launch();
    copy2d_kernel<double2><<<ew_blocks((long long)n * n), 256, 0, s>>>(
        reinterpret_cast<const double2 *>(Z), ldz, w.W, ld, n, w.flags);
    FROB_CUDA(cudaGetLastError());
    if (n <= lu2_max_n()) {
        FROB_CUDA(lu2_factor<double2>(n, w.W, w.W2, ld, w.U, w.L, ld, w.perm, w.iw, w.diag, w.stats, s));
        FROB_CUDA(inv_from_ul<double2>(n, w.U, w.L, ld, w.W, reinterpret_cast<double2 *>(X), ldx, w.perm, w.flags + 2, s));
    } else {
        FROB_CUDA(getrf<double2>(n, w.W, ld, w.perm, w.mv, w.diag, w.stats, w.work, s));
        FROB_CUDA(inv_from_lu<double2>(n, w.W, ld, w.U, w.L, reinterpret_cast<double2 *>(X), ldx, w.perm, w.flags + 2, s));
    }
    if (host_info) {
        LuStats hs;
        int hf = 0;
        FROB_CUDA(cudaMemcpyAsync(&hs, w.stats, sizeof(LuStats), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaMemcpyAsync(&hf, w.flags, sizeof(int), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaStreamSynchronize(s));
        *host_info = hs.info;
        if (hf) return FROB_ERR_NONFINITE;
        if (hs.info) return FROB_ERR_SINGULAR;
    }
    return FROB_OK;
}

// ---------------------------------------------------------------------- real inverse
struct DinvWs {
    double *W, *U, *L, *W2, *diag, *work;  // W2: n <= LU2_MAX_N only
    double *V;                             // EarlyInv scratch (early_inv_h(n) > 0 only)
    int *perm, *mv, *iw;
    LuStats *stats;
    int *flags;
    size_t bytes;
};
static DinvWs carve_dinv(void *ws, int n) {
    const long long ld = ld_of(n);
    Carve c{reinterpret_cast<unsigned char *>(ws), 0, 0};
    DinvWs w{};
    w.W = c.take<double>((size_t)n * ld);
    w.U = c.take<double>((size_t)n * ld);
    w.L = c.take<double>((size_t)n * ld);
    const bool small = n <= lu2_max_n();
    w.W2 = small ? c.take<double>((size_t)n * ld) : nullptr;
    w.V = (small && early_inv_h(n) > 0) ? c.take<double>((size_t)n * ld) : nullptr;
    w.diag = c.take<double>((size_t)n);
    w.work = c.take<double>(getrf_work_elems<double>(n));
    w.perm = c.take<int>((size_t)n);
    w.mv = c.take<int>(lu_mv_ints(n));
    w.iw = small ? c.take<int>(lu2_int_elems(n)) : nullptr;
    w.stats = c.take<LuStats>(1);
    w.flags = c.take<int>(4);
    w.bytes = c.off;
    return w;
}

// ---------------------------------------------------------------------- Newton
// X <- (X + Y^op)/2 where Y^op = Y (sign) or conj(Y)^T (polar); per-block partial sums
// of |Xnew - Xold|^2 and |Xnew|^2 (deterministic two-pass reduction).
template <bool POLAR>
__global__ void __launch_bounds__(256) newton_update_kernel(double2 *__restrict__ X, const double2 *__restrict__ Y,
                                                            int n, double *__restrict__ partial) {
    __shared__ double2 tile[32][33];
    __shared__ double rs[8][2];
    const int tiles = (n + 31) / 32;
    double s_d = 0.0, s_x = 0.0;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int tb = blockIdx.x; tb < tiles * tiles; tb += gridDim.x) {
        const int bi = tb / tiles, bj = tb - bi * tiles;
        if (POLAR) {
            // load Y block (bj, bi) transposed
            __syncthreads();
            for (int r = ty; r < 32; r += 8) {
                const int gi = bj * 32 + r, gj = bi * 32 + tx;
                if (gi < n && gj < n) tile[r][tx] = Y[(long long)gi * n + gj];
            }
            __syncthreads();
        }
        for (int r = ty; r < 32; r += 8) {
            const int gi = bi * 32 + r, gj = bj * 32 + tx;
            if (gi >= n || gj >= n) continue;
            double2 y;
            if (POLAR) {
                const double2 t = tile[tx][r];
                y = make_double2(t.x, -t.y);
            } else {
                y = Y[(long long)gi * n + gj];
            }
            const double2 x = X[(long long)gi * n + gj];
            const double2 xn = make_double2(0.5 * (x.x + y.x), 0.5 * (x.y + y.y));
            const double dx = xn.x - x.x, dy = xn.y - x.y;
            s_d = fma(dx, dx, fma(dy, dy, s_d));
            s_x = fma(xn.x, xn.x, fma(xn.y, xn.y, s_x));
            X[(long long)gi * n + gj] = xn;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s_d += __shfl_xor_sync(0xffffffffu, s_d, o);
        s_x += __shfl_xor_sync(0xffffffffu, s_x, o);
    }
    if (tx == 0) { rs[ty][0] = s_d; rs[ty][1] = s_x; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0, b = 0;
        for (int i = 0; i < 8; ++i) { a += rs[i][0]; b += rs[i][1]; }
        partial[2 * blockIdx.x] = a;
        partial[2 * blockIdx.x + 1] = b;
    }
}

__global__ void reduce_pairs_kernel(const double *__restrict__ partial, int nb, double *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double a = 0, b = 0;
        for (int i = 0; i < nb; ++i) { a += partial[2 * i]; b += partial[2 * i + 1]; }
        out[0] = a;
        out[1] = b;
    }
}

// H = (W + W^H)/2
__global__ void herm_sym_kernel(const double2 *__restrict__ W, double2 *__restrict__ H, int n) {
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const double2 a = W[(long long)i * n + j], b = W[(long long)j * n + i];
        H[idx] = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
    }
}
// V = U^H
__global__ void conj_transpose_kernel(const double2 *__restrict__ U, double2 *__restrict__ V, int n) {
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const double2 a = U[(long long)j * n + i];
        V[idx] = make_double2(a.x, -a.y);
    }
}

constexpr int NEWTON_BLOCKS = 296;

static size_t inv_ws_bytes(int n, int method) {
    return method == FROB_INV_ZLU ? carve_zlu(nullptr, n).bytes : carve_frob(nullptr, n).bytes;
}

static size_t newton_ws_bytes(int n, int method) {
    return align256(inv_ws_bytes(n, method)) + align256((size_t)n * n * 16) * 2 +
           align256(NEWTON_BLOCKS * 2 * sizeof(double)) + align256(2 * sizeof(double));
}

static frob_status newton_impl(bool polar, int n, const double *Z, double *S, double *Hout, double tol,
                               int max_iter, int method, void *ws, size_t ws_bytes, cudaStream_t s,
                               int *iters, double *final_delta, double *trace) {
    if (n < 1 || !Z || !S || max_iter < 1 || !(tol > 0) || !iters || !final_delta ||
        (method != FROB_INV_FROBENIUS && method != FROB_INV_ZLU) || (polar && !Hout))
        return FROB_ERR_INVALID_ARG;
    if (overlap(Z, (size_t)n * n * 16, S, (size_t)n * n * 16)) return FROB_ERR_INVALID_ARG;
    if (!ws || ws_bytes < newton_ws_bytes(n, method)) return FROB_ERR_WORKSPACE;
    unsigned char *b = reinterpret_cast<unsigned char *>(ws);
    const size_t ib = align256(inv_ws_bytes(n, method));
    void *iws = b;
    double *Yinv = reinterpret_cast<double *>(b + ib);
    double *Tmp = reinterpret_cast<double *>(b + ib + align256((size_t)n * n * 16));
    double *partial = reinterpret_cast<double *>(b + ib + 2 * align256((size_t)n * n * 16));
    double *sums = partial + align256(NEWTON_BLOCKS * 2 * sizeof(double)) / sizeof(double);

    FROB_CUDA(cudaMemcpyAsync(S, Z, (size_t)n * n * 16, cudaMemcpyDeviceToDevice, s));
    const int tiles = (n + 31) / 32;
    const int nb = std::min(NEWTON_BLOCKS, tiles * tiles);
    double delta = INFINITY;
    int it = 0;
    frob_status st = FROB_OK;
    for (it = 0; it < max_iter;) {
        if (method == FROB_INV_ZLU) st = zinv_lu_impl(n, S, n, Yinv, n, iws, ib, s, nullptr);
        else st = frob_inv_impl(n, S, n, Yinv, n, FROB_BRANCH_AUTO, iws, ib, s, nullptr);
        if (st != FROB_OK) return st;
        count_launch();
        if (polar)
            newton_update_kernel<true><<<nb, 256, 0, s>>>(reinterpret_cast<double2 *>(S),
                                                           reinterpret_cast<const double2 *>(Yinv), n, partial);
        else
            newton_update_kernel<false><<<nb, 256, 0, s>>>(reinterpret_cast<double2 *>(S),
                                                            reinterpret_cast<const double2 *>(Yinv), n, partial);
        FROB_CUDA(cudaGetLastError());
        count_launch();
        reduce_pairs_kernel<<<1, 32, 0, s>>>(partial, nb, sums);
        FROB_CUDA(cudaGetLastError());
        double h[2];
        FROB_CUDA(cudaMemcpyAsync(h, sums, sizeof(h), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaStreamSynchronize(s));
        delta = std::sqrt(h[0]) / std::sqrt(h[1]);
        if (trace) trace[it] = delta;
        ++it;
        if (delta < tol) break;
    }
    *iters = it;
    *final_delta = delta;
    if (polar) {
        // H = (U^H A + (U^H A)^H) / 2
        const double2 *U2 = reinterpret_cast<const double2 *>(S);
        count_launch();
        conj_transpose_kernel<<<ew_blocks((long long)n * n), 256, 0, s>>>(U2, reinterpret_cast<double2 *>(Yinv), n);
        FROB_CUDA(cudaGetLastError());
        auto p = gemm_params<double2>(n, n, n, 1.0, reinterpret_cast<const double2 *>(Yinv), n,
                                      reinterpret_cast<const double2 *>(Z), n, 0.0, nullptr, n,
                                      reinterpret_cast<double2 *>(Tmp), n);
        FROB_CUDA(gemm_launch<double2>(p, 1, s));
        count_launch();
        herm_sym_kernel<<<ew_blocks((long long)n * n), 256, 0, s>>>(reinterpret_cast<const double2 *>(Tmp),
                                                                     reinterpret_cast<double2 *>(Hout), n);
        FROB_CUDA(cudaGetLastError());
        FROB_CUDA(cudaStreamSynchronize(s));
    }
    return (delta < tol) ? FROB_OK : FROB_ERR_NOT_CONVERGED;
}

// ---------------------------------------------------------------------- Sylvester (NEXT-3)
// T = [[A, -C], [0, -B]] (order m + n) from dense row-major A (m x m), B (n x n), C (m x n);
// lyap != 0: B = A^H (B pointer ignored)
__global__ void sylv_assemble_kernel(const double2 *__restrict__ A, const double2 *__restrict__ B,
                                     const double2 *__restrict__ C, int m, int n, int lyap, double2 *__restrict__ T) {
    const int N = m + n;
    const long long total = (long long)N * N;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / N), j = (int)(idx - (long long)i * N);
        double2 v = make_double2(0.0, 0.0);
        if (i < m && j < m) v = A[(long long)i * m + j];
        else if (i < m) { const double2 c = C[(long long)i * n + (j - m)]; v = make_double2(-c.x, -c.y); }
        else if (j >= m) {
            const int bi = i - m, bj = j - m;
            if (lyap) { const double2 a = A[(long long)bj * m + bi]; v = make_double2(-a.x, a.y); }  // -(A^H)
            else { const double2 b = B[(long long)bi * n + bj]; v = make_double2(-b.x, -b.y); }
        }
        T[idx] = v;
    }
}
// X = -S_12 / 2
__global__ void sylv_extract_kernel(const double2 *__restrict__ S, int m, int n, double2 *__restrict__ X) {
    const int N = m + n;
    const long long total = (long long)m * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const double2 v = S[(long long)i * N + m + j];
        X[idx] = make_double2(-0.5 * v.x, -0.5 * v.y);
    }
}

static size_t sylv_ws_bytes(int m, int n, int method) {
    const int N = m + n;
    return align256(newton_ws_bytes(N, method)) + 2 * align256((size_t)N * N * 16);
}

static frob_status sylvester_impl(int m, int n, const double *A, const double *B, const double *C, double *X,
                                  int lyap, double tol, int max_iter, int method, void *ws, size_t ws_bytes,
                                  cudaStream_t s, int *iters, double *final_delta) {
    if (m < 1 || n < 1 || !A || !C || !X || (!lyap && !B) || !iters || !final_delta) return FROB_ERR_INVALID_ARG;
    if (lyap && m != n) return FROB_ERR_INVALID_ARG;
    if (!ws || ws_bytes < sylv_ws_bytes(m, n, method)) return FROB_ERR_WORKSPACE;
    const int N = m + n;
    unsigned char *b = reinterpret_cast<unsigned char *>(ws);
    const size_t nb = align256(newton_ws_bytes(N, method));
    double2 *T = reinterpret_cast<double2 *>(b + nb);
    double2 *S = reinterpret_cast<double2 *>(b + nb + align256((size_t)N * N * 16));
    count_launch();
    sylv_assemble_kernel<<<ew_blocks((long long)N * N), 256, 0, s>>>(
        reinterpret_cast<const double2 *>(A), reinterpret_cast<const double2 *>(B), reinterpret_cast<const double2 *>(C),
        m, n, lyap, T);
    FROB_CUDA(cudaGetLastError());
    frob_status st = newton_impl(false, N, reinterpret_cast<const double *>(T), reinterpret_cast<double *>(S), nullptr,
                                 tol, max_iter, method, ws, nb, s, iters, final_delta, nullptr);
    if (st != FROB_OK && st != FROB_ERR_NOT_CONVERGED) return st;
    count_launch();
    sylv_extract_kernel<<<ew_blocks((long long)m * n), 256, 0, s>>>(S, m, n, reinterpret_cast<double2 *>(X));
    FROB_CUDA(cudaGetLastError());
    FROB_CUDA(cudaStreamSynchronize(s));
    return st;
}

}  // namespace frob

// =====================================================================================
// C ABI
// =====================================================================================
using namespace frob;

extern "C" {

size_t frob_inv_workspace_bytes(int n) { return n < 1 ? 0 : carve_frob(nullptr, n).bytes; }

frob_status frob_inv(int n, const double *Z, long long ldz, double *X, long long ldx, int branch,
                     void *ws, size_t ws_bytes, void *stream, frob_info *host_info) {
    return frob_inv_impl(n, Z, ldz, X, ldx, branch, ws, ws_bytes, (cudaStream_t)stream, host_info);
}

frob_status frob_inv_rand(int n, const double *Z, long long ldz, double *X, long long ldx, double mu, void *ws,
                          size_t ws_bytes, void *stream, frob_info *host_info) {
    if (!(mu >= 0.0 && mu <= 1.0)) return FROB_ERR_INVALID_ARG;
    return frob_inv_impl(n, Z, ldz, X, ldx, FROB_BRANCH_AUTO, ws, ws_bytes, (cudaStream_t)stream, host_info, mu);
}

frob_status frob_inv_opts(int n, const double *Z, long long ldz, double *X, long long ldx, int branch, int options,
                          void *ws, size_t ws_bytes, void *stream, frob_info *host_info) {
    if (options & ~(FROB_OPT_FUSED_FIRST_STEP | FROB_OPT_DEVICE_AUTO)) return FROB_ERR_INVALID_ARG;
    return frob_inv_impl(n, Z, ldz, X, ldx, branch, ws, ws_bytes, (cudaStream_t)stream, host_info, 0.0,
                         (options & FROB_OPT_FUSED_FIRST_STEP) != 0, (options & FROB_OPT_DEVICE_AUTO) != 0);
}

frob_status frob_inv_dev(int n, const double *Z, long long ldz, double *X, long long ldx, int branch, int options,
                         frob_dev_status *d_status, void *ws, size_t ws_bytes, void *stream) {
    if (options & ~(FROB_OPT_FUSED_FIRST_STEP | FROB_OPT_DEVICE_AUTO)) return FROB_ERR_INVALID_ARG;
    StatusOut so;
    so.rec = d_status;
    return frob_inv_impl(n, Z, ldz, X, ldx, branch, ws, ws_bytes, (cudaStream_t)stream, nullptr, 0.0,
                         (options & FROB_OPT_FUSED_FIRST_STEP) != 0, (options & FROB_OPT_DEVICE_AUTO) != 0, so);
}

size_t frob_inv_host_workspace_bytes(int n) {
    return n < 1 ? 0 : align256(frob_inv_workspace_bytes(n)) + 2 * align256((size_t)n * n * 16) + 256;
}

size_t frob_inv_host_many_workspace_bytes(int n) {
    return n < 1 ? 0 : align256(frob_inv_workspace_bytes(n)) + 4 * align256((size_t)n * n * 16) + 2 * 256;
}

// per-device copy streams and events of the pipelined host entry point
constexpr int HOST_CHUNKS = 8;
struct HostPipe {
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t start, in[2], done[2], freed[2], fin, chunk[HOST_CHUNKS];
    bool ok = false;
    std::mutex mu;
};
static HostPipe &host_pipe(cudaError_t &err) {
    static HostPipe pipes[64];
    static std::mutex gmu;
    int dev = 0;
    cudaGetDevice(&dev);
    HostPipe &p = pipes[dev & 63];
    std::lock_guard<std::mutex> g(gmu);
    err = cudaSuccess;
    if (!p.ok) {
        err = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking);
        if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking);
        cudaEvent_t *evs[] = {&p.start, &p.in[0], &p.in[1], &p.done[0], &p.done[1], &p.freed[0], &p.freed[1], &p.fin};
        for (cudaEvent_t *e : evs)
            if (err == cudaSuccess) err = cudaEventCreateWithFlags(e, cudaEventDisableTiming);
        for (cudaEvent_t &e : p.chunk)
            if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        p.ok = (err == cudaSuccess);
    }
    return p;
}

// Join both copy streams into `s` and wait for everything (every exit path of the pipelined entry
// points: no copy into or out of the caller's host buffers is still in flight on return).
static cudaError_t host_pipe_join(HostPipe &hp, cudaStream_t s) {
    cudaError_t first = cudaEventRecord(hp.fin, hp.d2h);
    if (first == cudaSuccess) first = cudaStreamWaitEvent(s, hp.fin, 0);
    cudaError_t e = cudaEventRecord(hp.fin, hp.h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, hp.fin, 0);
    if (first == cudaSuccess) first = e;
    e = cudaStreamSynchronize(s);
    if (first == cudaSuccess) first = e;
    if (first != cudaSuccess) {  // a failed join: fall back to waiting on each stream
        cudaStreamSynchronize(hp.h2d);
        cudaStreamSynchronize(hp.d2h);
    }
    return first;
}

frob_status frob_inv_host(int n, const double *Z_host, double *X_host, int branch, void *ws,
                          size_t ws_bytes, void *stream, frob_info *host_info) {
    if (n < 1 || !Z_host || !X_host) return FROB_ERR_INVALID_ARG;
    if (!ws || ws_bytes < frob_inv_host_workspace_bytes(n)) return FROB_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned char *b = reinterpret_cast<unsigned char *>(ws);
    const size_t ib = align256(frob_inv_workspace_bytes(n));
    double *Zd = reinterpret_cast<double *>(b + ib);
    double *Xd = reinterpret_cast<double *>(b + ib + align256((size_t)n * n * 16));
    StatusOut so;
    so.code = reinterpret_cast<int *>(b + ib + 2 * align256((size_t)n * n * 16));
    // n >= 8192: the final GEMM runs in HOST_CHUNKS row blocks (>= 1024 rows: still several waves of
    // tiles, no split-K, so every element is computed exactly as in one launch) and each block is
    // copied out on a library-owned copy stream while the next one is computed
    const int K = (n >= 8192) ? HOST_CHUNKS : 1;
    cudaError_t ce = cudaSuccess;
    HostPipe &hp = host_pipe(ce);
    FROB_CUDA(ce);
    std::unique_lock<std::mutex> guard(hp.mu, std::defer_lock);
    OutChunks oc;
    if (K > 1) {
        guard.lock();
        oc.k = K;
        oc.ev = hp.chunk;
    }
    FROB_CUDA(cudaMemcpyAsync(Zd, Z_host, (size_t)n * n * 16, cudaMemcpyHostToDevice, s));
    frob_status st = frob_inv_impl(n, Zd, n, Xd, n, branch, ws, ib, s, host_info, 0.0, false, false, so, oc);
    int code = FROB_OK;
    cudaError_t err = cudaSuccess;
    if (st == FROB_OK && K > 1) {
        // (each copy waits only for its chunk's event, recorded on `stream` after that chunk's GEMM)
        const int per = (int)(((long long)n + K - 1) / K + 63) / 64 * 64;
        for (int r0 = 0, c = 0; r0 < n && err == cudaSuccess; r0 += per, ++c) {
            const int rc = std::min(per, n - r0);
            err = cudaStreamWaitEvent(hp.d2h, hp.chunk[c], 0);
            if (err == cudaSuccess)
                err = cudaMemcpyAsync(X_host + 2 * (size_t)r0 * n, Xd + 2 * (size_t)r0 * n, (size_t)rc * n * 16,
                                      cudaMemcpyDeviceToHost, hp.d2h);
        }
        if (err == cudaSuccess) err = cudaMemcpyAsync(&code, so.code, sizeof(int), cudaMemcpyDeviceToHost, s);
        const cudaError_t ej = host_pipe_join(hp, s);
        if (err == cudaSuccess) err = ej;
    } else if (st == FROB_OK) {
        err = cudaMemcpyAsync(X_host, Xd, (size_t)n * n * 16, cudaMemcpyDeviceToHost, s);
        if (err == cudaSuccess) err = cudaMemcpyAsync(&code, so.code, sizeof(int), cudaMemcpyDeviceToHost, s);
    }
    // every path waits for the copies that read / write the caller's host buffers
    const cudaError_t e = cudaStreamSynchronize(s);
    if (st != FROB_OK) return st;
    if (err != cudaSuccess) return cuda_fail(err);
    if (e != cudaSuccess) return cuda_fail(e);
    return (frob_status)code;
}

frob_status frob_inv_host_many(int n, int count, const double *Z_host, double *X_host, int branch, int *h_status,
                               void *ws, size_t ws_bytes, void *stream) {
    if (n < 1 || count < 0 || (count > 0 && (!Z_host || !X_host))) return FROB_ERR_INVALID_ARG;
    if (count == 0) return FROB_OK;
    if (!ws || ws_bytes < frob_inv_host_many_workspace_bytes(n)) return FROB_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t ce;
    HostPipe &hp = host_pipe(ce);
    FROB_CUDA(ce);
    std::lock_guard<std::mutex> guard(hp.mu);
    // per-matrix device status: the caller's array, else a pinned one of our own
    int *codes = h_status;
    if (!codes) FROB_CUDA(cudaHostAlloc(&codes, (size_t)count * sizeof(int), cudaHostAllocDefault));
    for (int i = 0; i < count; ++i) codes[i] = FROB_ERR_INVALID_ARG;  // "not computed"
    const size_t mb = (size_t)n * n * 16, md = (size_t)n * n * 2;  // bytes / doubles per matrix
    unsigned char *b = reinterpret_cast<unsigned char *>(ws);
    const size_t ib = align256(frob_inv_workspace_bytes(n));
    double *Zd[2], *Xd[2];
    int *Cd[2];
    for (int k = 0; k < 2; ++k) {
        Zd[k] = reinterpret_cast<double *>(b + ib + (2 * k) * align256(mb));
        Xd[k] = reinterpret_cast<double *>(b + ib + (2 * k + 1) * align256(mb));
        Cd[k] = reinterpret_cast<int *>(b + ib + 4 * align256(mb) + k * 256);
    }
    auto h2d = [&](int i) -> cudaError_t {
        const int k = i & 1;
        cudaError_t e = cudaSuccess;
        if (i >= 2) e = cudaStreamWaitEvent(hp.h2d, hp.done[k], 0);  // inversion i - 2 has read Zd[k]
        if (e == cudaSuccess) e = cudaMemcpyAsync(Zd[k], Z_host + (size_t)i * md, mb, cudaMemcpyHostToDevice, hp.h2d);
        if (e == cudaSuccess) e = cudaEventRecord(hp.in[k], hp.h2d);
        return e;
    };
    frob_status result = FROB_OK;
    cudaError_t err = cudaEventRecord(hp.start, s);  // the copy streams start after the work queued on `stream`
    if (err == cudaSuccess) err = cudaStreamWaitEvent(hp.h2d, hp.start, 0);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(hp.d2h, hp.start, 0);
    if (err == cudaSuccess) err = h2d(0);
    for (int i = 0; i < count && err == cudaSuccess; ++i) {
        const int k = i & 1;
        if (i + 1 < count && (err = h2d(i + 1)) != cudaSuccess) break;  // queued before inversion i
        if ((err = cudaStreamWaitEvent(s, hp.in[k], 0)) != cudaSuccess) break;
        if (i >= 2 && (err = cudaStreamWaitEvent(s, hp.freed[k], 0)) != cudaSuccess) break;  // X of i - 2 left Xd[k]
        StatusOut so;
        so.code = Cd[k];
        const frob_status st = frob_inv_impl(n, Zd[k], n, Xd[k], n, branch, ws, ib, s, nullptr, 0.0, false, false, so);
        if (st != FROB_OK) {
            result = st;
            codes[i] = st;
            break;
        }
        if ((err = cudaEventRecord(hp.done[k], s)) != cudaSuccess) break;
        if ((err = cudaStreamWaitEvent(hp.d2h, hp.done[k], 0)) != cudaSuccess) break;
        if ((err = cudaMemcpyAsync(X_host + (size_t)i * md, Xd[k], mb, cudaMemcpyDeviceToHost, hp.d2h)) != cudaSuccess) break;
        if ((err = cudaMemcpyAsync(codes + i, Cd[k], sizeof(int), cudaMemcpyDeviceToHost, hp.d2h)) != cudaSuccess) break;
        if ((err = cudaEventRecord(hp.freed[k], hp.d2h)) != cudaSuccess) break;
    }
    const cudaError_t ej = host_pipe_join(hp, s);
    if (err == cudaSuccess) err = ej;
    if (result == FROB_OK && err == cudaSuccess)
        for (int i = 0; i < count; ++i)
            if (codes[i] != FROB_OK) { result = (frob_status)codes[i]; break; }
    if (!h_status) cudaFreeHost(codes);
    if (err != cudaSuccess) return cuda_fail(err);
    return result;
}

size_t frob_inv_batched_host_workspace_bytes(int n, int chunk) {
    if (n < 1 || chunk < 1) return 0;
    const size_t mb = align256((size_t)chunk * n * n * 16), ib = align256((size_t)chunk * sizeof(int));
    return 4 * mb + 2 * ib + 2 * align256((size_t)chunk);
}

frob_status frob_inv_batched_host(int n, int batch, const double *Z_host, double *X_host, int branch, int *h_info,
                                  int chunk, void *ws, size_t ws_bytes, void *stream) {
    if (n < 1 || n > 128 || batch < 0 || chunk < 1 || (batch > 0 && (!Z_host || !X_host))) return FROB_ERR_INVALID_ARG;
    if (batch == 0) return FROB_OK;
    if (!ws || ws_bytes < frob_inv_batched_host_workspace_bytes(n, chunk)) return FROB_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t ce;
    HostPipe &hp = host_pipe(ce);
    FROB_CUDA(ce);
    std::lock_guard<std::mutex> guard(hp.mu);
    const size_t md = (size_t)n * n * 2;  // doubles per matrix
    const size_t mb = align256((size_t)chunk * n * n * 16), ib = align256((size_t)chunk * sizeof(int));
    unsigned char *b = reinterpret_cast<unsigned char *>(ws);
    double *Zd[2], *Xd[2];
    int *Id[2];
    unsigned char *Bu[2];
    for (int k = 0; k < 2; ++k) {
        Zd[k] = reinterpret_cast<double *>(b + (2 * k) * mb);
        Xd[k] = reinterpret_cast<double *>(b + (2 * k + 1) * mb);
        Id[k] = reinterpret_cast<int *>(b + 4 * mb + k * ib);
        Bu[k] = b + 4 * mb + 2 * ib + k * align256((size_t)chunk);
    }
    const int nch = (batch + chunk - 1) / chunk;
    auto cnt = [&](int j) { return std::min(chunk, batch - j * chunk); };
    auto h2d = [&](int j) -> cudaError_t {
        const int k = j & 1;
        cudaError_t e = cudaSuccess;
        if (j >= 2) e = cudaStreamWaitEvent(hp.h2d, hp.done[k], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(Zd[k], Z_host + (size_t)j * chunk * md, (size_t)cnt(j) * md * 8, cudaMemcpyHostToDevice,
                                hp.h2d);
        if (e == cudaSuccess) e = cudaEventRecord(hp.in[k], hp.h2d);
        return e;
    };
    frob_status result = FROB_OK;
    cudaError_t err = cudaEventRecord(hp.start, s);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(hp.h2d, hp.start, 0);
    if (err == cudaSuccess) err = cudaStreamWaitEvent(hp.d2h, hp.start, 0);
    if (err == cudaSuccess) err = h2d(0);
    for (int j = 0; j < nch && err == cudaSuccess; ++j) {
        const int k = j & 1, c = cnt(j);
        if (j + 1 < nch && (err = h2d(j + 1)) != cudaSuccess) break;
        if ((err = cudaStreamWaitEvent(s, hp.in[k], 0)) != cudaSuccess) break;
        if (j >= 2 && (err = cudaStreamWaitEvent(s, hp.freed[k], 0)) != cudaSuccess) break;
        const frob_status st = frob_inv_batched(n, c, Zd[k], (long long)n * n, Xd[k], (long long)n * n, branch, Id[k],
                                                Bu[k], nullptr, 0, s);
        if (st != FROB_OK) {
            result = st;
            break;
        }
        if ((err = cudaEventRecord(hp.done[k], s)) != cudaSuccess) break;
        if ((err = cudaStreamWaitEvent(hp.d2h, hp.done[k], 0)) != cudaSuccess) break;
        if ((err = cudaMemcpyAsync(X_host + (size_t)j * chunk * md, Xd[k], (size_t)c * md * 8, cudaMemcpyDeviceToHost,
                                   hp.d2h)) != cudaSuccess)
            break;
        if (h_info && (err = cudaMemcpyAsync(h_info + (size_t)j * chunk, Id[k], (size_t)c * sizeof(int),
                                             cudaMemcpyDeviceToHost, hp.d2h)) != cudaSuccess)
            break;
        if ((err = cudaEventRecord(hp.freed[k], hp.d2h)) != cudaSuccess) break;
    }
    const cudaError_t ej = host_pipe_join(hp, s);
    if (err == cudaSuccess) err = ej;
    if (err != cudaSuccess) return cuda_fail(err);
    return result;
}

size_t zinv_lu_workspace_bytes(int n) { return n < 1 ? 0 : carve_zlu(nullptr, n).bytes; }

frob_status zinv_lu(int n, const double *Z, long long ldz, double *X, long long ldx, void *ws,
                    size_t ws_bytes, void *stream, int *host_info) {
    return zinv_lu_impl(n, Z, ldz, X, ldx, ws, ws_bytes, (cudaStream_t)stream, host_info);
}

size_t frob_newton_workspace_bytes(int n, int method) { return n < 1 ? 0 : newton_ws_bytes(n, method); }

frob_status frob_sign_newton(int n, const double *Z, double *S, double tol, int max_iter, int method,
                             void *ws, size_t ws_bytes, void *stream, int *host_iters,
                             double *host_final_delta, double *host_trace) {
    return newton_impl(false, n, Z, S, nullptr, tol, max_iter, method, ws, ws_bytes, (cudaStream_t)stream,
                       host_iters, host_final_delta, host_trace);
}

frob_status frob_polar_newton(int n, const double *A, double *U, double *H, double tol, int max_iter,
                              int method, void *ws, size_t ws_bytes, void *stream, int *host_iters,
                              double *host_final_delta, double *host_trace) {
    if (H && (overlap(H, (size_t)n * n * 16, A, (size_t)n * n * 16) ||
              overlap(H, (size_t)n * n * 16, U, (size_t)n * n * 16)))
        return FROB_ERR_INVALID_ARG;
    return newton_impl(true, n, A, U, H, tol, max_iter, method, ws, ws_bytes, (cudaStream_t)stream,
                       host_iters, host_final_delta, host_trace);
}

size_t frob_sylvester_workspace_bytes(int m, int n, int method) {
    return (m < 1 || n < 1) ? 0 : sylv_ws_bytes(m, n, method);
}

frob_status frob_sylvester(int m, int n, const double *A, const double *B, const double *C, double *X, double tol,
                           int max_iter, int method, void *ws, size_t ws_bytes, void *stream, int *host_iters,
                           double *host_final_delta) {
    return sylvester_impl(m, n, A, B, C, X, 0, tol, max_iter, method, ws, ws_bytes, (cudaStream_t)stream, host_iters,
                          host_final_delta);
}

frob_status frob_lyapunov(int n, const double *A, const double *C, double *X, double tol, int max_iter, int method,
                          void *ws, size_t ws_bytes, void *stream, int *host_iters, double *host_final_delta) {
    return sylvester_impl(n, n, A, nullptr, C, X, 1, tol, max_iter, method, ws, ws_bytes, (cudaStream_t)stream,
                          host_iters, host_final_delta);
}

frob_status frob_dgemm(int m, int n, int k, double alpha, const double *A, long long lda, const double *B,
                       long long ldb, double beta, double *C, long long ldc, void *stream) {
    if (m < 0 || n < 0 || k < 0 || (m > 0 && n > 0 && (!C || ldc < n)) || (k > 0 && (!A || !B || lda < k || ldb < n)))
        return FROB_ERR_INVALID_ARG;
    auto p = gemm_params<double>(m, n, k, alpha, A, lda, B, ldb, beta, beta != 0.0 ? C : nullptr, ldc, C, ldc);
    FROB_CUDA(gemm_launch<double>(p, 1, (cudaStream_t)stream));
    return FROB_OK;
}

frob_status frob_dtrmm(int uplo, int n, int m, double alpha, const double *T, long long ldt, const double *B,
                       long long ldb, double *C, long long ldc, void *stream) {
    if ((uplo != TRI_UPPER && uplo != TRI_LOWER) || n < 0 || m < 0 ||
        (n > 0 && (!T || !B || !C || ldt < n || ldb < m || ldc < m)))
        return FROB_ERR_INVALID_ARG;
    if (n == 0 || m == 0) return FROB_OK;
    auto p = gemm_params<double>(n, m, n, alpha, T, ldt, B, ldb, 0.0, nullptr, ldc, C, ldc);
    p.triA = uplo;
    GemmTag tag("gemm:trmm");
    FROB_CUDA(gemm_launch<double>(p, 1, (cudaStream_t)stream));
    return FROB_OK;
}

size_t frob_dinv_workspace_bytes(int n) { return n < 1 ? 0 : carve_dinv(nullptr, n).bytes; }

frob_status frob_dinv(int n, const double *A, long long lda, double *Ainv, long long ldainv, void *ws,
                      size_t ws_bytes, void *stream, frob_info *host_info) {
    if (n < 1 || !A || !Ainv || lda < n || ldainv < n) return FROB_ERR_INVALID_ARG;
    if (overlap(A, (size_t)((n - 1) * lda + n) * 8, Ainv, (size_t)((n - 1) * ldainv + n) * 8))
        return FROB_ERR_INVALID_ARG;
    DinvWs w = carve_dinv(nullptr, n);
    if (!ws || ws_bytes < w.bytes) return FROB_ERR_WORKSPACE;
    w = carve_dinv(ws, n);
    cudaStream_t s = (cudaStream_t)stream;
    const long long ld = ld_of(n);
    count_launch();
    copy2d_kernel<double><<<ew_blocks((long long)n * n), 256, 0, s>>>(A, lda, w.W, ld, n, nullptr);
    FROB_CUDA(cudaGetLastError());
    if (n <= lu2_max_n()) {
        EarlyInv ei;  // the same inversion as frob_inv's (T_inv of the threshold analysis)
        ei.h = w.V ? early_inv_h(n) : 0;
        ei.vbuf = w.V;
        FROB_CUDA(lu2_factor<double>(n, w.W, w.W2, ld, w.U, w.L, ld, w.perm, w.iw, w.diag, w.stats, s, &ei));
        FROB_CUDA(inv_from_ul<double>(n, w.U, w.L, ld, w.W, Ainv, ldainv, w.perm, w.flags, s, &ei));
    } else {
        FROB_CUDA(getrf<double>(n, w.W, ld, w.perm, w.mv, w.diag, w.stats, w.work, s));
        FROB_CUDA(inv_from_lu<double>(n, w.W, ld, w.U, w.L, Ainv, ldainv, w.perm, w.flags, s));
    }
    if (host_info) {
        LuStats hs;
        FROB_CUDA(cudaMemcpyAsync(&hs, w.stats, sizeof(hs), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaStreamSynchronize(s));
        host_info->info = hs.info;
        host_info->branch_used = 0;
        host_info->rho_a = hs.rho;
        host_info->rho_b = NAN;
        host_info->rho_m = NAN;
        host_info->kappa_a = NAN;
        host_info->kappa_b = NAN;
        if (hs.info) return FROB_ERR_SINGULAR;
    }
    return FROB_OK;
}

size_t frob_dgetrf_workspace_bytes(int n) {
    if (n < 1) return 0;
    Carve c{nullptr, 0, 0};
    c.take<double>((size_t)n);
    c.take<double>(getrf_work_elems<double>(n));
    c.take<int>(lu_mv_ints(n));
    c.take<LuStats>(1);
    return c.off;
}

frob_status frob_dgetrf(int n, double *A, long long lda, int *perm, void *ws, size_t ws_bytes, void *stream,
                        frob_info *host_info) {
    if (n < 1 || !A || !perm || lda < n) return FROB_ERR_INVALID_ARG;
    if (!ws || ws_bytes < frob_dgetrf_workspace_bytes(n)) return FROB_ERR_WORKSPACE;
    Carve c{reinterpret_cast<unsigned char *>(ws), 0, 0};
    double *diag = c.take<double>((size_t)n);
    double *work = c.take<double>(getrf_work_elems<double>(n));
    int *mv = c.take<int>(lu_mv_ints(n));
    LuStats *st = c.take<LuStats>(1);
    cudaStream_t s = (cudaStream_t)stream;
    FROB_CUDA(getrf<double>(n, A, lda, perm, mv, diag, st, work, s));
    if (host_info) {
        LuStats hs;
        FROB_CUDA(cudaMemcpyAsync(&hs, st, sizeof(hs), cudaMemcpyDeviceToHost, s));
        FROB_CUDA(cudaStreamSynchronize(s));
        host_info->info = hs.info;
        host_info->branch_used = 0;
        host_info->rho_a = hs.rho;
        host_info->rho_b = NAN;
        host_info->rho_m = NAN;
        host_info->kappa_a = NAN;
        host_info->kappa_b = NAN;
        if (hs.info) return FROB_ERR_SINGULAR;
    }
    return FROB_OK;
}

const char *frob_status_string(int status) {
    switch (status) {
        case FROB_OK: return "ok";
        case FROB_ERR_SINGULAR: return "singular pivot";
        case FROB_ERR_BOTH_SINGULAR: return "both real and imaginary parts singular";
        case FROB_ERR_NOT_CONVERGED: return "Newton iteration did not converge";
        case FROB_ERR_INVALID_ARG: return "invalid argument";
        case FROB_ERR_NONFINITE: return "non-finite input";
        case FROB_ERR_WORKSPACE: return "workspace too small";
        case FROB_ERR_CUDA: return "CUDA error";
        default: return "unknown status";
    }
}

const char *frob_last_cuda_error(void) { return g_last_cuda; }

void frob_profile_enable(int on) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (auto &r : g_prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto &r : g_prof_open) cudaEventDestroy(r.e);
    g_prof.clear();
    g_prof_open.clear();
    g_prof_on = on != 0;
}

int frob_profile_read(char *buf, size_t len) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    struct Agg { long long cnt = 0; double ms = 0.0, work = 0.0; };
    std::map<std::string, Agg> agg;
    for (auto &r : g_prof) {
        if (cudaEventSynchronize(r.b) != cudaSuccess) return -1;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) return -1;
        auto &a = agg[r.name];
        a.cnt += 1;
        a.ms += ms;
        a.work += r.work;
    }
    std::string out = "{";
    bool first = true;
    for (auto &kv : agg) {
        char tmp[320];
        snprintf(tmp, sizeof(tmp), "%s\"%s\": {\"launches\": %lld, \"total_ms\": %.6f, \"flops\": %.6e}",
                 first ? "" : ", ", kv.first.c_str(), kv.second.cnt, kv.second.ms, kv.second.work);
        out += tmp;
        first = false;
    }
    out += "}";
    if (buf && len > 0) {
        snprintf(buf, len, "%s", out.c_str());
    }
    return (int)out.size();
}

unsigned long long frob_launch_count(void) { return frob::launch_counter(); }

int frob_version(void) { return 1; }

}  // extern "C"
