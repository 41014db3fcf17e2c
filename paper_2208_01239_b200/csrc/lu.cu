// lu.cu -- LU panel / swap+TRSM / diagnostics kernels, the triangular-inverse
// recursion and the GEMM launcher.  See lu.cuh and DESIGN.md section "Kernels".
#include <cooperative_groups.h>
#include <climits>
#include <cstdio>
#include "lu.cuh"

namespace cg = cooperative_groups;

namespace frob {

// =====================================================================================
// GEMM launcher
// =====================================================================================
template <typename T, bool VEC>
static cudaError_t gemm_launch_impl(const GemmParams<T> &p, int batch, cudaStream_t s) {
    using Cf = GemmCfg<T>;
    constexpr size_t smem = gemm_smem_bytes<T>();
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(gemm_kernel<T, VEC>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    dim3 grid((p.N + Cf::BN - 1) / Cf::BN, (p.M + Cf::BM - 1) / Cf::BM, batch);
    count_launch();
    gemm_kernel<T, VEC><<<grid, Cf::WGM * Cf::WGN * 32, smem, s>>>(p);
    return cudaGetLastError();
}

static bool aligned16(const void *ptr) { return ((uintptr_t)ptr & 15u) == 0; }

template <typename T>
cudaError_t gemm_launch(const GemmParams<T> &p, int batch, cudaStream_t s) {
    if (p.M <= 0 || p.N <= 0 || batch <= 0) return cudaSuccess;
    constexpr int E = 16 / sizeof(T);
    bool vec = aligned16(p.A) && aligned16(p.B) && (p.lda % E == 0) && (p.ldb % E == 0) &&
               (batch == 1 || ((p.sA % E == 0) && (p.sB % E == 0)));
    return vec ? gemm_launch_impl<T, true>(p, batch, s) : gemm_launch_impl<T, false>(p, batch, s);
}
template cudaError_t gemm_launch<double>(const GemmParams<double> &, int, cudaStream_t);
template cudaError_t gemm_launch<double2>(const GemmParams<double2> &, int, cudaStream_t);

// =====================================================================================
// Panel factorisation (cluster, DSMEM argmax)
// =====================================================================================
constexpr int PANEL_THREADS = 256;
constexpr int PANEL_WARPS = PANEL_THREADS / 32;

template <typename T, int PW>
struct PanelShared {
    // fixed part (after the row tile and per-row ints)
    double wred_v[2][PANEL_WARPS];
    int wred_i[2][PANEL_WARPS];
    double pub_v[2];
    int pub_i[2];
    T pubrow[2][PW];
    T wpiv[PANEL_WARPS][PW];
    int pivrows[PW];
    T pvals[PW];
    int vac[PW];
    unsigned evmask;
};

template <typename T, int PW>
static size_t panel_smem_bytes(int rpc) {
    size_t tile = (size_t)rpc * (PW + 1) * sizeof(T);
    size_t ints = (size_t)rpc * sizeof(int);
    size_t off = (tile + ints + 15) & ~(size_t)15;
    return off + sizeof(PanelShared<T, PW>);
}

// P: panel top-left (row k0, col k0); m = n - k0 panel rows; w <= PW columns.
template <typename T, int PW>
__global__ void __launch_bounds__(PANEL_THREADS)
lu_panel_kernel(T *__restrict__ P, long long lda, int m, int w, int rpc, int CS, int k0,
                int *__restrict__ mv, T *__restrict__ diag) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *tile = reinterpret_cast<T *>(smem_raw);
    int *rowpiv = reinterpret_cast<int *>(smem_raw + (size_t)rpc * (PW + 1) * sizeof(T));
    size_t off = ((size_t)rpc * (PW + 1) * sizeof(T) + (size_t)rpc * sizeof(int) + 15) & ~(size_t)15;
    PanelShared<T, PW> &sh = *reinterpret_cast<PanelShared<T, PW> *>(smem_raw + off);
    constexpr int TS = PW + 1;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int crank = 0;
    if (CS > 1) crank = (int)cg::this_cluster().block_rank();
    const int rbeg = crank * rpc;
    const int nrows = max(0, min(rpc, m - rbeg));

    for (int idx = tid; idx < nrows * w; idx += PANEL_THREADS) {
        const int r = idx / w, c = idx - r * w;
        tile[r * TS + c] = P[(long long)(rbeg + r) * lda + c];
    }
    for (int r = tid; r < nrows; r += PANEL_THREADS) rowpiv[r] = -1;
    __syncthreads();

    for (int j = 0; j < w; ++j) {
        const int par = j & 1;
        double bv = -1.0;
        int bi = INT_MAX;
        for (int r = tid; r < nrows; r += PANEL_THREADS) {
            if (rowpiv[r] < 0) {
                const double v = pkey(tile[r * TS + j]);
                if (better(v, rbeg + r, bv, bi)) { bv = v; bi = rbeg + r; }
            }
        }
        ArgMax wa = warp_argmax(bv, bi);
        if (lane == 0) { sh.wred_v[par][warp] = wa.v; sh.wred_i[par][warp] = wa.i; }
        __syncthreads();
        ArgMax ca = warp_argmax(lane < PANEL_WARPS ? sh.wred_v[par][lane] : -1.0,
                                lane < PANEL_WARPS ? sh.wred_i[par][lane] : INT_MAX);
        int gp;
        T pv = zero_of(T());
        if (CS == 1) {
            gp = ca.i;
            if (lane < w) pv = tile[(gp - rbeg) * TS + lane];
        } else {
            cg::cluster_group cl = cg::this_cluster();
            if (warp == 0) {
                if (lane == 0) { sh.pub_v[par] = ca.v; sh.pub_i[par] = ca.i; }
                if (lane < w && ca.i != INT_MAX) sh.pubrow[par][lane] = tile[(ca.i - rbeg) * TS + lane];
            }
            cl.sync();
            double qv = -1.0;
            int qi = INT_MAX;
            if (lane < CS) {
                qv = *cl.map_shared_rank(&sh.pub_v[par], lane);
                qi = *cl.map_shared_rank(&sh.pub_i[par], lane);
            }
            ArgMax ga = warp_argmax(qv, qi);
            gp = ga.i;
            const int owner = gp / rpc;
            if (lane < w) pv = *cl.map_shared_rank(&sh.pubrow[par][lane], owner);
        }
        if (lane < PW) sh.wpiv[warp][lane] = pv;
        __syncwarp();
        const T piv = sh.wpiv[warp][j];
        const bool zp = is_zero(piv);
        const T ip = zp ? zero_of(T()) : recip(piv);
        if (tid == 0) { sh.pivrows[j] = gp; sh.pvals[j] = piv; }
        for (int r = tid; r < nrows; r += PANEL_THREADS) {
            if (rowpiv[r] >= 0) continue;
            if (rbeg + r == gp) { rowpiv[r] = j; continue; }
            if (zp) continue;
            T *row = tile + r * TS;
            const T l = mul(row[j], ip);
            row[j] = l;
            for (int c = j + 1; c < w; ++c) row[c] = msub(row[c], l, sh.wpiv[warp][c]);
        }
    }
    __syncthreads();

    // final positions: pivot j -> row j; evicted rows (< w, not pivots) fill the rows
    // vacated by pivots that came from below (>= w), in pivot order.
    if (warp == 0) {
        bool rp = false;
        if (lane < w)
            for (int q = 0; q < w; ++q) rp |= (sh.pivrows[q] == lane);
        const unsigned pivmask = __ballot_sync(0xffffffffu, rp);
        const unsigned wmask = (w >= 32) ? 0xffffffffu : ((1u << w) - 1u);
        const unsigned evmask = wmask & ~pivmask;
        const int gpj = lane < w ? sh.pivrows[lane] : -1;
        const bool isv = lane < w && gpj >= w;
        const unsigned vb = __ballot_sync(0xffffffffu, isv);
        if (isv) sh.vac[__popc(vb & ((1u << lane) - 1u))] = gpj;
        if (lane == 0) sh.evmask = evmask;
        __syncwarp();
        if (crank == 0) {
            // movement list for the other columns (global row indices)
            const bool moved = lane < w && gpj != lane;
            const unsigned mb = __ballot_sync(0xffffffffu, moved);
            const int nm = __popc(mb);
            if (moved) {
                const int q = __popc(mb & ((1u << lane) - 1u));
                mv[1 + q] = k0 + lane;
                mv[1 + 2 * PW_MAX + q] = k0 + gpj;
            }
            const bool ev = (evmask >> lane) & 1u;
            if (ev) {
                const int q = nm + __popc(evmask & ((1u << lane) - 1u));
                mv[1 + q] = k0 + sh.vac[__popc(evmask & ((1u << lane) - 1u))];
                mv[1 + 2 * PW_MAX + q] = k0 + lane;
            }
            if (lane == 0) mv[0] = nm + __popc(evmask);
            if (lane < w) diag[k0 + lane] = sh.pvals[lane];
        }
    }
    __syncthreads();
    for (int r = tid; r < nrows; r += PANEL_THREADS) {
        const int g = rbeg + r;
        int dst;
        if (rowpiv[r] >= 0) dst = rowpiv[r];
        else if (g < w) dst = sh.vac[__popc(sh.evmask & ((1u << g) - 1u))];
        else dst = g;
        rowpiv[r] = dst;
    }
    __syncthreads();
    for (int idx = tid; idx < nrows * w; idx += PANEL_THREADS) {
        const int r = idx / w, c = idx - r * w;
        P[(long long)rowpiv[r] * lda + c] = tile[r * TS + c];
    }
}

// =====================================================================================
// Row movement on the other columns + U12 = L11^{-1} A12 (unit lower forward solve)
// =====================================================================================
constexpr int SWP_COLS = 64;

template <typename T, int PW>
__global__ void __launch_bounds__(SWP_COLS)
lu_swap_trsm_kernel(T *__restrict__ A, long long lda, int n, int k0, int w,
                    const int *__restrict__ mv, int *__restrict__ perm) {
    __shared__ T Ls[PW][PW + 1];
    __shared__ T buf[2 * PW][SWP_COLS];
    __shared__ int ptmp[2 * PW];
    const int tid = threadIdx.x;
    const int cnt = mv[0];
    const int *dst = mv + 1, *src = mv + 1 + 2 * PW_MAX;
    if (blockIdx.x == 0) {
        for (int q = tid; q < cnt; q += SWP_COLS) ptmp[q] = perm[src[q]];
        __syncthreads();
        for (int q = tid; q < cnt; q += SWP_COLS) perm[dst[q]] = ptmp[q];
    }
    for (int idx = tid; idx < w * w; idx += SWP_COLS) {
        const int i = idx / w, q = idx - i * w;
        Ls[i][q] = A[(long long)(k0 + i) * lda + k0 + q];
    }
    __syncthreads();
    const int v = blockIdx.x * SWP_COLS + tid;
    if (v >= n - w) return;
    const int c = (v < k0) ? v : v + w;
    for (int q = 0; q < cnt; ++q) buf[q][tid] = A[(long long)src[q] * lda + c];
    for (int q = 0; q < cnt; ++q) A[(long long)dst[q] * lda + c] = buf[q][tid];
    if (c < k0 + w) return;
    T x[PW];
#pragma unroll
    for (int i = 0; i < PW; ++i) x[i] = (i < w) ? A[(long long)(k0 + i) * lda + c] : zero_of(T());
#pragma unroll
    for (int i = 1; i < PW; ++i) {
        if (i < w) {
            T acc = x[i];
#pragma unroll
            for (int q = 0; q < i; ++q) acc = msub(acc, Ls[i][q], x[q]);
            x[i] = acc;
        }
    }
#pragma unroll
    for (int i = 0; i < PW; ++i)
        if (i < w) A[(long long)(k0 + i) * lda + c] = x[i];
}

// =====================================================================================
// Pivot diagnostics (reading R2): rho, singular column, non-finite
// =====================================================================================
template <typename T>
__global__ void __launch_bounds__(1024) lu_stats_kernel(const T *__restrict__ diag, int n, LuStats *st) {
    __shared__ double smax[32], smin[32];
    __shared__ int snf[32], sidx[32];
    __shared__ double thr_s;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double mx = 0.0, mn = INFINITY;
    int nf = 0;
    for (int i = tid; i < n; i += blockDim.x) {
        const T d = diag[i];
        if (!finite_of(d)) nf = 1;
        const double a = pmag(d);
        mx = fmax(mx, a);
        mn = fmin(mn, a);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        nf |= __shfl_xor_sync(0xffffffffu, nf, o);
    }
    if (lane == 0) { smax[warp] = mx; smin[warp] = mn; snf[warp] = nf; }
    __syncthreads();
    const int nw = blockDim.x / 32;
    if (warp == 0) {
        mx = lane < nw ? smax[lane] : 0.0;
        mn = lane < nw ? smin[lane] : INFINITY;
        nf = lane < nw ? snf[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            nf |= __shfl_xor_sync(0xffffffffu, nf, o);
        }
        if (lane == 0) {
            thr_s = 100.0 * (double)n * 1.1102230246251565e-16 * mx;
            st->rho = (mn > 0.0) ? mx / mn : INFINITY;
            st->umax = mx;
            st->nonfinite = nf;
        }
    }
    __syncthreads();
    // first singular pivot column: |u_kk| < thr (or zero)
    int first = INT_MAX;
    for (int i = tid; i < n; i += blockDim.x) {
        const double a = pmag(diag[i]);
        if (!(a >= thr_s) || a == 0.0) { first = i; break; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
    if (lane == 0) sidx[warp] = first;
    __syncthreads();
    if (warp == 0) {
        first = lane < nw ? sidx[lane] : INT_MAX;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
        if (lane == 0) st->info = (first == INT_MAX) ? 0 : first + 1;
    }
}

__global__ void iota_kernel(int *p, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

// =====================================================================================
// getrf driver
// =====================================================================================
template <typename T, int PW>
static cudaError_t launch_panel(T *P, long long lda, int m, int w, int k0, int *mv, T *diag,
                                cudaStream_t s) {
    // rows per CTA so that the tile fits in ~200 KB of shared memory
    const size_t row_bytes = (size_t)(PW + 1) * sizeof(T) + sizeof(int);
    const int maxrows = (int)((200 * 1024 - sizeof(PanelShared<T, PW>) - 64) / row_bytes);
    int CS = (m + maxrows - 1) / maxrows;
    if (CS < 1) CS = 1;
    int rpc = (m + CS - 1) / CS;
    const size_t smem = panel_smem_bytes<T, PW>(rpc);
    auto kern = lu_panel_kernel<T, PW>;
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3(CS, 1, 1);
    cfg.blockDim = dim3(PANEL_THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (CS > 1) ? 1 : 0;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kern, P, lda, m, w, rpc, CS, k0, mv, diag);
}

// Largest panel width whose cluster stays <= 16 CTAs.
template <typename T>
static int choose_pw(int n) {
    const int rows32 = (int)((200 * 1024 - 2048) / ((32 + 1) * sizeof(T) + 4));
    const int rows16 = (int)((200 * 1024 - 2048) / ((16 + 1) * sizeof(T) + 4));
    if (sizeof(T) == 8) {
        if ((n + rows32 - 1) / rows32 <= 8) return 32;
        if ((n + rows16 - 1) / rows16 <= 16) return 16;
        return 8;
    }
    if ((n + rows16 - 1) / rows16 <= 8) return 16;
    return 8;
}

template <typename T, int PW>
static cudaError_t getrf_pw(int n, T *A, long long lda, int *perm, int *mv, T *diag, cudaStream_t s) {
    cudaError_t e;
    for (int k0 = 0; k0 < n; k0 += PW) {
        const int w = min(PW, n - k0), m = n - k0;
        e = launch_panel<T, PW>(A + (long long)k0 * lda + k0, lda, m, w, k0, mv, diag, s);
        if (e != cudaSuccess) return e;
        const int ncols = n - w;
        const int nb = max(1, (ncols + SWP_COLS - 1) / SWP_COLS);
        count_launch();
        lu_swap_trsm_kernel<T, PW><<<nb, SWP_COLS, 0, s>>>(A, lda, n, k0, w, mv, perm);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        const int rest = n - k0 - w;
        if (rest > 0) {
            T *a21 = A + (long long)(k0 + w) * lda + k0;
            T *a12 = A + (long long)k0 * lda + k0 + w;
            T *a22 = A + (long long)(k0 + w) * lda + k0 + w;
            auto p = gemm_params<T>(rest, rest, w, -1.0, a21, lda, a12, lda, 1.0, a22, lda, a22, lda);
            if ((e = gemm_launch<T>(p, 1, s)) != cudaSuccess) return e;
        }
    }
    return cudaSuccess;
}

template <typename T>
cudaError_t getrf(int n, T *A, long long lda, int *perm, int *mv, T *diag, LuStats *stats,
                  cudaStream_t s) {
    count_launch();
    iota_kernel<<<(n + 255) / 256, 256, 0, s>>>(perm, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int pw = choose_pw<T>(n);
    if constexpr (sizeof(T) == 8) {
        if (pw == 32) e = getrf_pw<T, 32>(n, A, lda, perm, mv, diag, s);
        else if (pw == 16) e = getrf_pw<T, 16>(n, A, lda, perm, mv, diag, s);
        else e = getrf_pw<T, 8>(n, A, lda, perm, mv, diag, s);
    } else {
        if (pw == 16) e = getrf_pw<T, 16>(n, A, lda, perm, mv, diag, s);
        else e = getrf_pw<T, 8>(n, A, lda, perm, mv, diag, s);
    }
    if (e != cudaSuccess) return e;
    if (stats) {
        count_launch();
        lu_stats_kernel<T><<<1, 1024, 0, s>>>(diag, n, stats);
        e = cudaGetLastError();
    }
    return e;
}
template cudaError_t getrf<double>(int, double *, long long, int *, int *, double *, LuStats *, cudaStream_t);
template cudaError_t getrf<double2>(int, double2 *, long long, int *, int *, double2 *, LuStats *, cudaStream_t);

// =====================================================================================
// Triangular inverses: U^{-1} (non-unit upper) and L^{-1} (unit lower)
// =====================================================================================
constexpr int TRI_LEAF = 32;

// U = triu(lu) (zeros below), L = tril(lu, -1) + I (zeros above)
template <typename T>
__global__ void extract_ul_kernel(const T *__restrict__ lu, long long ld, int n, T *__restrict__ U,
                                  T *__restrict__ L) {
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), j = (int)(idx - (long long)i * n);
        const T v = lu[(long long)i * ld + j];
        const T z = zero_of(T());
        U[(long long)i * ld + j] = (j >= i) ? v : z;
        L[(long long)i * ld + j] = (j < i) ? v : ((j == i) ? one_of(T()) : z);
    }
}

// blockIdx.y == 0: invert upper diagonal blocks of U in place; == 1: unit-lower blocks of L
template <typename T>
__global__ void __launch_bounds__(TRI_LEAF) tri_leaf_kernel(T *__restrict__ U, T *__restrict__ L,
                                                            long long ld, int n) {
    __shared__ T S[TRI_LEAF][TRI_LEAF + 1];
    __shared__ T X[TRI_LEAF][TRI_LEAF + 1];
    const int b0 = blockIdx.x * TRI_LEAF;
    const int sz = min(TRI_LEAF, n - b0);
    const bool upper = (blockIdx.y == 0);
    T *M = upper ? U : L;
    const int tid = threadIdx.x;
    for (int i = 0; i < sz; ++i)
        if (tid < sz) S[i][tid] = M[(long long)(b0 + i) * ld + b0 + tid];
    __syncthreads();
    if (tid < sz) {
        if (upper) {
            // row i = tid of U^{-1}: X[i][i] = 1/u_ii; X[i][j] = -(sum_{k=i}^{j-1} X[i][k] u_kj)/u_jj
            const int i = tid;
            for (int j = 0; j < i; ++j) X[i][j] = zero_of(T());
            X[i][i] = recip(S[i][i]);
            for (int j = i + 1; j < sz; ++j) {
                T acc = zero_of(T());
                for (int k = i; k < j; ++k) acc = madd(acc, X[i][k], S[k][j]);
                X[i][j] = neg(mul(acc, recip(S[j][j])));
            }
        } else {
            // column j = tid of L^{-1}: Y[j][j] = 1; Y[i][j] = -sum_{k=j}^{i-1} l_ik Y[k][j]
            const int j = tid;
            for (int i = 0; i < j; ++i) X[i][j] = zero_of(T());
            X[j][j] = one_of(T());
            for (int i = j + 1; i < sz; ++i) {
                T acc = zero_of(T());
                for (int k = j; k < i; ++k) acc = madd(acc, S[i][k], X[k][j]);
                X[i][j] = neg(acc);
            }
        }
    }
    __syncthreads();
    for (int i = 0; i < sz; ++i)
        if (tid < sz) M[(long long)(b0 + i) * ld + b0 + tid] = X[i][tid];
}

// One recursion level of size s: blocks [o, o+s) x [o+s, o+s+s2) for o = p*2s.
template <typename T>
static cudaError_t tri_level(T *U, T *L, T *tmp, long long ld, int s, int o, int s2, int batch,
                             cudaStream_t st) {
    const long long stride = 2LL * s * (ld + 1);
    cudaError_t e;
    // upper: W = U12 * inv(U22);  U12 <- -inv(U11) * W
    {
        auto p = gemm_params<T>(s, s2, s2, 1.0, U + (long long)o * ld + o + s, ld,
                                U + (long long)(o + s) * ld + o + s, ld, 0.0, nullptr, ld,
                                tmp + (long long)o * ld + o + s, ld);
        p.triB = TRI_UPPER; p.sA = p.sB = p.sC = stride; p.sD = 0;
        if ((e = gemm_launch<T>(p, batch, st)) != cudaSuccess) return e;
        auto q = gemm_params<T>(s, s2, s, -1.0, U + (long long)o * ld + o, ld,
                                tmp + (long long)o * ld + o + s, ld, 0.0, nullptr, ld,
                                U + (long long)o * ld + o + s, ld);
        q.triA = TRI_UPPER; q.sA = q.sB = q.sC = stride; q.sD = 0;
        if ((e = gemm_launch<T>(q, batch, st)) != cudaSuccess) return e;
    }
    // lower: W = L21 * inv(L11);  L21 <- -inv(L22) * W
    {
        auto p = gemm_params<T>(s2, s, s, 1.0, L + (long long)(o + s) * ld + o, ld,
                                L + (long long)o * ld + o, ld, 0.0, nullptr, ld,
                                tmp + (long long)(o + s) * ld + o, ld);
        p.triB = TRI_LOWER; p.sA = p.sB = p.sC = stride; p.sD = 0;
        if ((e = gemm_launch<T>(p, batch, st)) != cudaSuccess) return e;
        auto q = gemm_params<T>(s2, s, s2, -1.0, L + (long long)(o + s) * ld + o + s, ld,
                                tmp + (long long)(o + s) * ld + o, ld, 0.0, nullptr, ld,
                                L + (long long)(o + s) * ld + o, ld);
        q.triA = TRI_LOWER; q.sA = q.sB = q.sC = stride; q.sD = 0;
        if ((e = gemm_launch<T>(q, batch, st)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

template <typename T>
cudaError_t inv_from_lu(int n, T *lu, long long ld, T *U, T *L, T *out, long long ldo,
                        const int *colperm, cudaStream_t s) {
    cudaError_t e;
    {
        long long total = (long long)n * n;
        long long nb = (total + 255) / 256; int blocks = (int)(nb < 148LL * 16 ? nb : 148LL * 16);
        count_launch();
        extract_ul_kernel<T><<<blocks, 256, 0, s>>>(lu, ld, n, U, L);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    count_launch();
    tri_leaf_kernel<T><<<dim3((n + TRI_LEAF - 1) / TRI_LEAF, 2), TRI_LEAF, 0, s>>>(U, L, ld, n);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    T *tmp = lu;  // the LU factors are no longer needed
    for (int sz = TRI_LEAF; sz < n; sz *= 2) {
        const int full = n / (2 * sz);
        if (full > 0 && (e = tri_level<T>(U, L, tmp, ld, sz, 0, sz, full, s)) != cudaSuccess) return e;
        const int o = full * 2 * sz;
        if (o + sz < n) {
            if ((e = tri_level<T>(U, L, tmp, ld, sz, o, n - o - sz, 1, s)) != cudaSuccess) return e;
        }
    }
    // X = U^{-1} L^{-1}: (upper) x (lower) -> k from max(row0, col0)
    auto p = gemm_params<T>(n, n, n, 1.0, U, ld, L, ld, 0.0, nullptr, ld, out, ldo);
    p.triA = TRI_UPPER;
    p.triB = TRI_LOWER;
    p.colperm = colperm;
    return gemm_launch<T>(p, 1, s);
}
template cudaError_t inv_from_lu<double>(int, double *, long long, double *, double *, double *, long long, const int *, cudaStream_t);
template cudaError_t inv_from_lu<double2>(int, double2 *, long long, double2 *, double2 *, double2 *, long long, const int *, cudaStream_t);

}  // namespace frob
