// lu3_experiment.cu -- EXPERIMENT (not built into libfrobinv.so; kept for tools/lu2_probe.cu): persistent LU with partial pivoting (Alg 3 line 1) for the inversion
// path, orders n <= LU3_MAX_N (1024), real (PW = 16) and complex (PW = 8).
//
// ONE cooperative launch per factorisation (one 1024-thread CTA per SM, all co-resident).
// The first CTA to start takes the PANEL role, every other CTA runs four 256-thread WORKERS:
//
//   panel CTA  owns the pivot chain.  Thread t keeps original row t in registers for the
//              current PW-column block.  Per column: warp argmax (REDUX), the warp winner
//              publishes its row + reciprocal in shared memory, ONE __syncthreads, block
//              argmax over the 32 warp candidates, rank-1 update of the own row.  (A thread-
//              block cluster was measured first: a DSMEM st.async + mbarrier round trip costs
//              ~520 cycles per column against 36 for __syncthreads -- tools/dsmem_probe.cu.)
//              Before each block it applies the previous block's update to it itself
//              (look-ahead: U12 = L11^{-1} X, a -= l21 U12, l21 kept in shared memory).
//   workers    take tasks (step k, column group g, row tile r) from an atomic ticket in
//              dependency order and apply U12 = L11^{-1} X, A22 -= L21 U12 to the column
//              groups >= k+2 (flags in global memory, acquire/release; bounded spins trap).
//
// Rows are never moved: a row keeps its original index; the pivot of column k0+j gets
// position k0+j (perm[k0+j] = its original row).  U is written straight to its final
// position (U[k0+j][.]), L multipliers stay in the rows of A; lu3_assemble_kernel writes
// the split L (and zeroes U below the diagonal) in final row order.
#include <climits>
#include <cstdio>
#include <utility>
#include <algorithm>
#include <cooperative_groups.h>
#include "../paper_2208_01239_b200/csrc/lu.cuh"

namespace cg = cooperative_groups;

namespace frob {

// Persistent LU (this file; experiment, not built into the library) for n <= LU3_MAX_N: A (n x ld) is destroyed (it keeps the
// L multipliers by original row), U and L come out split in final row order (ld);
// iw = lu3_int_elems(n) ints.
constexpr int LU3_MAX_N = 1024;
size_t lu3_int_elems(int n);
template <typename T>
cudaError_t lu3_factor(int n, T *A, long long ld, T *U, T *L, int *perm, int *iw, T *diag, LuStats *stats,
                       cudaStream_t s);

constexpr int LU3_T = 1024;      // threads per CTA (panel: one row per thread)
constexpr int LU3_W = LU3_T / 32;
constexpr int LU3_ST = 256;      // threads per worker
constexpr int LU3_NSUB = LU3_T / LU3_ST;
constexpr int LU3_TR = 64;       // worker row tile
constexpr int LU3_G = 4;         // worker column group: LU3_G blocks of PW columns

template <typename T> struct Lu3W { static constexpr int PW = 16; };
template <> struct Lu3W<double2> { static constexpr int PW = 8; };

template <typename T>
struct Lu3Params {
    T *A;            // n x ld, input; L multipliers are left in place (original rows)
    T *U;            // n x ld, U in final row order (rows k0+j), upper part written here
    long long ld;
    int n, nb, ngroups, nrt;
    int *perm;       // [n] position -> original row
    int *prow;       // [nb * PW] pivot original rows per step
    int *pstep;      // [n] step at which an original row became a pivot (INT_MAX before)
    T *diag;         // [n] pivot values in position order
    int *flags;      // [0] cluster ticket, [1] task ticket, [2..2+nb) panel done, then done[nb][ngroups]
    long long ntasks;
};

// ------------------------------------------------------------------ sync helpers
FROB_DEV int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
FROB_DEV void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
FROB_DEV void red_release_add(int *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// bounded spin: a dependency that never resolves traps instead of hanging the GPU
FROB_DEV void wait_geq(const int *p, int target) {
    long long it = 0;
    while (ld_acquire(p) < target) {
        __nanosleep(64);
        if (++it > (1LL << 26)) __trap();
    }
}
FROB_DEV void st_async16(unsigned raddr, const uint4 v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
                 : "memory");
}
FROB_DEV void mbar_arrive_expect(unsigned addr, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(tx) : "memory");
}
FROB_DEV void mbar_wait_cluster(unsigned addr, unsigned parity) {
    long long it = 0;
    unsigned ok = 0;
    while (true) {
        asm volatile(
            "{\n.reg .pred p;\n"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            "selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(addr), "r"(parity)
            : "memory");
        if (ok) break;
        if (++it > (1LL << 24)) __trap();
    }
}

#ifdef FROB_L3_TRACE
__device__ long long g_l3_trace[16];
#define L3T(v) long long v = 0; if (threadIdx.x == 0 && crank == 0) v = clock64();
#define L3ACC(i, a, b) do { if (threadIdx.x == 0 && crank == 0) g_l3_trace[i] += (b) - (a); } while (0)
#define L3C(i) do { if (threadIdx.x == 0 && crank == 0 && k == 10 && J == 5) g_l3_trace[i] = clock64(); } while (0)
#else
#define L3C(i) do { } while (0)
#define L3T(v)
#define L3ACC(i, a, b) do { } while (0)
#endif

FROB_DEV double l3_rcp(double x) { return (x == 0.0) ? 0.0 : frcp(x); }
FROB_DEV double2 l3_rcp(double2 x) { return is_zero(x) ? make_double2(0.0, 0.0) : recip(x); }

template <typename T>
FROB_DEV T shfl_t(const T &v, int src) { return shfl(v, src); }

template <typename F, int... J>
FROB_DEV void static_for_l3_impl(F &&f, std::integer_sequence<int, J...>) {
    (f(std::integral_constant<int, J>{}), ...);
}
template <int N, typename F>
FROB_DEV void static_for_l3(F &&f) {
    static_for_l3_impl(f, std::make_integer_sequence<int, N>{});
}
template <typename T, int PW>
FROB_DEV void st_row_l3(T *dst, const T (&r)[PW]) {
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int c = 0; c < PW; c += 2) *reinterpret_cast<double2 *>(dst + c) = make_double2(r[c], r[c + 1]);
    } else {
#pragma unroll
        for (int c = 0; c < PW; ++c) dst[c] = r[c];
    }
}
template <typename T, int PW>
FROB_DEV void ld_row_smem_l3(T (&u)[PW], const T *src) {
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int c = 0; c < PW; c += 2) {
            const double2 v = *reinterpret_cast<const double2 *>(src + c);
            u[c] = v.x;
            u[c + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int c = 0; c < PW; ++c) u[c] = src[c];
    }
}

// ------------------------------------------------------------------ shared memory
template <typename T, int PW>
struct Lu3PanelSmem {
    __align__(16) T wrow[2][LU3_W][PW];   // each warp's candidate row
    T wrcp[2][LU3_W];
    unsigned long long ck[2][LU3_W];
    int ci[2][LU3_W];
    T upiv[PW][PW];                        // pivot rows of the current step (L11 | U11)
    T upiv_prev[PW][PW];
    int prow_s[PW], prow_prev[PW];
    __align__(16) T Xs[PW][PW];            // look-ahead: pivot rows' block values, then U12
    __align__(16) T Lsave[LU3_T][PW];      // multipliers of the previous step, one row per thread
};
template <typename T, int PW>
struct Lu3SubSmem {
    T L11[PW][PW + 1];
    __align__(16) T Us[PW][LU3_G * PW];
    T Ls[LU3_TR][PW + 1];
    int tprow[PW];
    long long task;
};
template <typename T, int PW>
struct Lu3Smem {
    union {
        Lu3PanelSmem<T, PW> panel;
        Lu3SubSmem<T, PW> sub[LU3_NSUB];
    };
    int role;
};

// ------------------------------------------------------------------ panel role
template <typename T, int PW>
FROB_DEV void lu3_panel(const Lu3Params<T> &p, Lu3PanelSmem<T, PW> &sm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = p.n;
    const long long ld = p.ld;
    bool act = tid < n;          // original row tid, not yet a pivot
    bool lpact = false;          // row has multipliers of the previous step in Lsave
    T a[PW];
    int *panel_done = p.flags + 2;
    const int *done = p.flags + 2 + p.nb;
    const int crank = 0;
    (void)crank;
    for (int k = 0; k < p.nb; ++k) {
        const int k0 = k * PW, w = min(PW, n - k0);
        L3T(t0);
        // ---------------- block k: load, then the look-ahead update with step k-1's factors
        if (k >= 2) {
            if (tid == 0) wait_geq(&done[(long long)(k - 2) * p.ngroups + k / LU3_G], p.nrt);
            __syncthreads();
        }
        L3T(t1);
        L3ACC(0, t0, t1);
        if (act) {
            const T *src = p.A + (long long)tid * ld + k0;
#pragma unroll
            for (int c = 0; c < PW; ++c) a[c] = (c < w) ? src[c] : zero_of(T());
        }
        if (k >= 1) {
            if (tid < PW * PW) {
                const int j = tid / PW, c = tid % PW;
                sm.Xs[j][c] = (c < w) ? p.A[(long long)sm.prow_prev[j] * ld + k0 + c] : zero_of(T());
            }
            __syncthreads();
            if (tid < PW) {
                T x[PW];
#pragma unroll
                for (int j = 0; j < PW; ++j) x[j] = sm.Xs[j][tid];
#pragma unroll
                for (int q = 0; q < PW; ++q)
#pragma unroll
                    for (int j = q + 1; j < PW; ++j) x[j] = msub(x[j], sm.upiv_prev[j][q], x[q]);
#pragma unroll
                for (int j = 0; j < PW; ++j) sm.Xs[j][tid] = x[j];
                if (tid < w) {
#pragma unroll
                    for (int j = 0; j < PW; ++j) p.U[(long long)(k0 - PW + j) * ld + k0 + tid] = x[j];
                }
            }
            __syncthreads();
            if (act && lpact) {
#pragma unroll
                for (int q = 0; q < PW; ++q) {
                    const T lq = sm.Lsave[tid][q];
#pragma unroll
                    for (int c = 0; c < PW; ++c) a[c] = msub(a[c], lq, sm.Xs[q][c]);
                }
            }
        }
        L3T(t2);
        L3ACC(1, t1, t2);
        // ---------------- the pivot chain of block k
        auto column = [&](auto Jc) {
            constexpr int J = decltype(Jc)::value;
            constexpr int s = J & 1;
            const unsigned long long kk = act ? pkey_bits(a[J]) : 0ull;
            const T myr = act ? l3_rcp(a[J]) : zero_of(T());
            const ArgMaxK wa = warp_argmax_key(kk, act ? tid : INT_MAX);
            if (lane == 0) { sm.ck[s][warp] = wa.k; sm.ci[s][warp] = wa.i; }
            if (act && tid == wa.i) {
                st_row_l3<T, PW>(sm.wrow[s][warp], a);
                sm.wrcp[s][warp] = myr;
            }
            __syncthreads();
            const ArgMaxK ca = warp_argmax_key(sm.ck[s][lane], sm.ci[s][lane]);
            const int gi = ca.i;
            const int ww = gi >> 5;
            const T *u = sm.wrow[s][ww];
            const T rc = sm.wrcp[s][ww];
            if (tid == 0) {
#pragma unroll
                for (int c = 0; c < PW; ++c) sm.upiv[J][c] = u[c];
                sm.prow_s[J] = gi;
            }
            if (act && tid == gi) {
                // pivot row: U row k0+J (columns >= J); its L part (columns < J) stays in A
                act = false;
                T *urow = p.U + (long long)(k0 + J) * ld + k0;
                T *arow = p.A + (long long)tid * ld + k0;
#pragma unroll
                for (int c = 0; c < PW; ++c) {
                    if (c < w) {
                        if (c >= J) urow[c] = a[c];
                        else arow[c] = a[c];
                    }
                }
                p.diag[k0 + J] = a[J];
                p.perm[k0 + J] = tid;
                p.pstep[tid] = k;
            } else if (act) {
                const T l = mul(a[J], rc);
                a[J] = l;
#pragma unroll
                for (int c = J + 1; c < PW; ++c) a[c] = msub(a[c], l, u[c]);
            }
        };
        static_for_l3<PW>([&](auto Jc) {
            constexpr int Jv = decltype(Jc)::value;
            if (Jv < w) column(Jc);
        });
        L3T(t3);
        L3ACC(2, t2, t3);
        // ---------------- publish: L21 of the active rows, pivot list, then the flag
        if (act) {
            T *arow = p.A + (long long)tid * ld + k0;
#pragma unroll
            for (int c = 0; c < PW; ++c)
                if (c < w) arow[c] = a[c];
            st_row_l3<T, PW>(sm.Lsave[tid], a);
        }
        lpact = act;
        if (tid < w) p.prow[k0 + tid] = sm.prow_s[tid];
        __syncthreads();
        if (tid < PW * PW) sm.upiv_prev[tid / PW][tid % PW] = sm.upiv[tid / PW][tid % PW];
        if (tid < PW) sm.prow_prev[tid] = sm.prow_s[tid];
        __threadfence();
        __syncthreads();
        if (tid == 0) st_release(&panel_done[k], 1);
        L3T(t4);
        L3ACC(3, t3, t4);
    }
}

// ------------------------------------------------------------------ worker role
FROB_DEV void sub_sync(int id) { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(LU3_ST) : "memory"); }

template <typename T, int PW>
FROB_DEV void lu3_worker(const Lu3Params<T> &p, Lu3SubSmem<T, PW> &sm, const int sub) {
    constexpr int TC = LU3_G * PW;        // tile columns
    constexpr int CPT = TC / 16;          // columns per thread (16 threads across)
    const int tid = threadIdx.x & (LU3_ST - 1);
    const int bid = 1 + sub;              // named barrier of this worker
    const int n = p.n;
    const long long ld = p.ld;
    const int *panel_done = p.flags + 2;
    int *done = p.flags + 2 + p.nb;
    const int ty = tid >> 4, tx = tid & 15;
    for (;;) {
        sub_sync(bid);
        if (tid == 0) sm.task = (long long)atomicAdd(&p.flags[1], 1);
        sub_sync(bid);
        long long t = sm.task;
        if (t >= p.ntasks) break;
        // decode (k, g, r): tasks ordered by step, then group, then row tile
        int k = 0, g = 0, r = 0;
        for (k = 0; k < p.nb; ++k) {
            const int g0 = (k + 2) / LU3_G;
            const long long cnt = (long long)max(0, p.ngroups - g0) * p.nrt;
            if (t < cnt) {
                g = g0 + (int)(t / p.nrt);
                r = (int)(t % p.nrt);
                break;
            }
            t -= cnt;
        }
        const int k0 = k * PW;
        const int cb = max(g * LU3_G, k + 2) * PW;     // first column of the tile
        const int ce = min((g + 1) * LU3_G * PW, n);  // end column
        const int r0 = r * LU3_TR;
        if (tid == 0) {
            wait_geq(&panel_done[k], 1);
            if (k >= 1) wait_geq(&done[(long long)(k - 1) * p.ngroups + g], p.nrt);
        }
        sub_sync(bid);
        if (tid < PW) sm.tprow[tid] = p.prow[k0 + tid];
        sub_sync(bid);
        const int nc = ce - cb;
        for (int idx = tid; idx < PW * PW; idx += LU3_ST) {
            const int j = idx / PW, q = idx % PW;
            sm.L11[j][q] = p.A[(long long)sm.tprow[j] * ld + k0 + q];
        }
        for (int idx = tid; idx < PW * TC; idx += LU3_ST) {
            const int j = idx / TC, c = idx % TC;
            sm.Us[j][c] = (c < nc) ? p.A[(long long)sm.tprow[j] * ld + cb + c] : zero_of(T());
        }
        for (int idx = tid; idx < LU3_TR * PW; idx += LU3_ST) {
            const int i = idx / PW, q = idx % PW;
            const int row = r0 + i;
            sm.Ls[i][q] = (row < n && p.pstep[row] > k) ? p.A[(long long)row * ld + k0 + q] : zero_of(T());
        }
        T acc[4][CPT];
        bool rowok[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int row = r0 + ty * 4 + i;
            rowok[i] = row < n && p.pstep[row] > k;
            const T *src = p.A + (long long)(rowok[i] ? row : 0) * ld + cb + tx * CPT;
#pragma unroll
            for (int j = 0; j < CPT; ++j) acc[i][j] = (rowok[i] && tx * CPT + j < nc) ? src[j] : zero_of(T());
        }
        sub_sync(bid);
        if (tid < TC) {
            T x[PW];
#pragma unroll
            for (int j = 0; j < PW; ++j) x[j] = sm.Us[j][tid];
#pragma unroll
            for (int q = 0; q < PW; ++q)
#pragma unroll
                for (int j = q + 1; j < PW; ++j) x[j] = msub(x[j], sm.L11[j][q], x[q]);
#pragma unroll
            for (int j = 0; j < PW; ++j) sm.Us[j][tid] = x[j];
            if (r == 0 && tid < nc) {
#pragma unroll
                for (int j = 0; j < PW; ++j) p.U[(long long)(k0 + j) * ld + cb + tid] = x[j];
            }
        }
        sub_sync(bid);
#pragma unroll
        for (int q = 0; q < PW; ++q) {
            T lv[4], uv[CPT];
#pragma unroll
            for (int i = 0; i < 4; ++i) lv[i] = sm.Ls[ty * 4 + i][q];
#pragma unroll
            for (int j = 0; j < CPT; ++j) uv[j] = sm.Us[q][tx * CPT + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < CPT; ++j) acc[i][j] = msub(acc[i][j], lv[i], uv[j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (!rowok[i]) continue;
            T *dst = p.A + (long long)(r0 + ty * 4 + i) * ld + cb + tx * CPT;
#pragma unroll
            for (int j = 0; j < CPT; ++j)
                if (tx * CPT + j < nc) dst[j] = acc[i][j];
        }
        __threadfence();
        sub_sync(bid);
        if (tid == 0) red_release_add(&done[(long long)k * p.ngroups + g], 1);
    }
}

template <typename T, int PW>
__global__ void __launch_bounds__(LU3_T, 1) lu3_kernel(Lu3Params<T> p) {
    extern __shared__ __align__(16) unsigned char smraw[];
    Lu3Smem<T, PW> &sm = *reinterpret_cast<Lu3Smem<T, PW> *>(smraw);
    if (threadIdx.x == 0) sm.role = atomicAdd(&p.flags[0], 1);
    __syncthreads();
    if (sm.role == 0) lu3_panel<T, PW>(p, sm.panel);
    else {
        const int sub = threadIdx.x / LU3_ST;
        lu3_worker<T, PW>(p, sm.sub[sub], sub);
    }
}

// L[i][c] = A[perm[i]][c] (c < i), 1 (c == i), 0 above; U below the diagonal := 0
template <typename T>
__global__ void lu3_assemble_kernel(const T *__restrict__ A, T *__restrict__ U, T *__restrict__ L, long long ld,
                                    int n, const int *__restrict__ perm) {
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), c = (int)(idx - (long long)i * n);
        T lv = zero_of(T());
        if (c < i) {
            lv = A[(long long)perm[i] * ld + c];
            U[(long long)i * ld + c] = zero_of(T());
        } else if (c == i) {
            lv = one_of(T());
        }
        L[(long long)i * ld + c] = lv;
    }
}

__global__ void lu3_init_kernel(int *pstep, int n, int *flags, int nflags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) pstep[i] = INT_MAX;
    if (i < nflags) flags[i] = 0;
}

// ------------------------------------------------------------------ host side
size_t lu3_int_elems(int n) {
    const int PW = 8;
    const int nb = (n + PW - 1) / PW;
    const int ngroups = (nb + LU3_G - 1) / LU3_G;
    return (size_t)n /* pstep */ + (size_t)nb * 16 /* prow */ + 2 + nb + (size_t)nb * ngroups + 64;
}

template <typename T>
cudaError_t lu3_factor(int n, T *A, long long ld, T *U, T *L, int *perm, int *iw, T *diag, LuStats *stats,
                       cudaStream_t s) {
    constexpr int PW = Lu3W<T>::PW;
    if (n > LU3_MAX_N || n < 1) return cudaErrorInvalidValue;
    Lu3Params<T> p{};
    p.A = A;
    p.U = U;
    p.ld = ld;
    p.n = n;
    p.nb = (n + PW - 1) / PW;
    p.ngroups = (p.nb + LU3_G - 1) / LU3_G;
    p.nrt = (n + LU3_TR - 1) / LU3_TR;
    p.perm = perm;
    p.pstep = iw;
    p.prow = iw + n;
    p.flags = p.prow + (size_t)p.nb * PW;
    p.diag = diag;
    long long nt = 0;
    for (int k = 0; k < p.nb; ++k) nt += (long long)std::max(0, p.ngroups - (k + 2) / LU3_G) * p.nrt;
    p.ntasks = nt;
    const int nflags = 2 + p.nb + p.nb * p.ngroups;
    const size_t smem = sizeof(Lu3Smem<T, PW>);
    static int grid_of[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e;
    if (dev >= 64) return cudaErrorInvalidDevice;
    if (grid_of[dev] == 0) {
        if ((e = cudaFuncSetAttribute(lu3_kernel<T, PW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
            cudaSuccess)
            return e;
        int per_sm = 0, sms = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu3_kernel<T, PW>, LU3_T, smem)) != cudaSuccess)
            return e;
        if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
        if (per_sm < 1 || sms < 2) return cudaErrorInvalidConfiguration;
        grid_of[dev] = per_sm * sms;
    }
    const int total = std::max(n, nflags);
    count_launch();
    lu3_init_kernel<<<(total + 255) / 256, 256, 0, s>>>(p.pstep, n, p.flags, nflags);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    {
        void *args[] = {&p};
        count_launch();
        if ((e = cudaLaunchCooperativeKernel((void *)lu3_kernel<T, PW>, dim3(grid_of[dev]), dim3(LU3_T), args, smem, s)) !=
            cudaSuccess)
            return e;
    }
    {
        const long long tot = (long long)n * n;
        const int blocks = (int)std::min<long long>((tot + 255) / 256, 148LL * 8);
        count_launch();
        lu3_assemble_kernel<T><<<blocks, 256, 0, s>>>(A, U, L, ld, n, perm);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (stats) e = lu_stats_launch<T>(diag, n, stats, s);
    return e;
}
template cudaError_t lu3_factor<double>(int, double *, long long, double *, double *, int *, int *, double *,
                                        LuStats *, cudaStream_t);
template cudaError_t lu3_factor<double2>(int, double2 *, long long, double2 *, double2 *, int *, int *, double2 *,
                                         LuStats *, cudaStream_t);

}  // namespace frob
