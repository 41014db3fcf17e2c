// batched.cu -- batched small-n Frobenius inversion and complex-LU comparator:
// one CTA per matrix, everything resident on chip (BASELINE config 3; config 1).
//
// Per matrix (Alg 1):
//   load Z (interleaved, coalesced) -> planar A, B in shared memory
//   X^{-1} by a register-resident Gauss-Jordan sweep with partial pivoting
//       (each thread owns a 4x4 block; no row swaps: the pivot order is recorded and
//        undone when the inverse is written back -- "exchange" form of GJ)
//   branch check (reading R1'): kappa_inf(A) = ||A||_inf ||A^{-1}||_inf from the computed
//       inverse; lazy: B is swept only when A is singular or kappa_inf(A) > kappa_switch(n)
//   C = X^{-1} Y,  M = X + Y C,  Re = M^{-1} (sweep),  Im = -C Re
//       the three GEMMs run on the FP64 tensor cores (DMMA m8n8k4) from shared memory
//   store X interleaved (branch S1: Re - i(-Im) ... see the epilogue)
// The real inversion used here is Gauss-Jordan, which computes the same inverse as
// Alg 3 (2n^3 flops) with n sequential steps instead of 3n ("batched path").
#include <climits>
#include <cmath>
#include <utility>
#include "common.cuh"
#include "../../include/frobinv.h"

namespace frob {

// DMMA without `volatile`: the compiler may interleave independent tiles (the f64 mma's latency is long)
FROB_DEV void dmma_s(double &c0, double &c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}
FROB_DEV double fast_recip(double x) { return frcp(x); }
FROB_DEV double2 fast_recip(double2 x) { return recip(x); }

// Register-block geometry: N x N matrix, each thread owns a BR x BC block.
template <int N, int BR = 4, int BC = 4>
struct Geo {
    static constexpr int RT = N / BR;          // thread rows (<= 32: one warp reduces a column)
    static constexpr int CT = N / BC;          // thread columns
    static constexpr int THREADS = RT * CT;
    static constexpr int S = N + 4;            // padded smem row stride
    static_assert(RT <= 32, "column candidates must fit one warp");
};
template <int N>
struct BCfg {
    static constexpr int S = N + 4;
    static constexpr int THREADS = Geo<N>::THREADS;
};

template <typename F, int... J>
FROB_DEV void bstatic_for_impl(F &&f, std::integer_sequence<int, J...>) {
    (f(std::integral_constant<int, J>{}), ...);
}
template <int K, typename F>
FROB_DEV void bstatic_for(F &&f) {
    bstatic_for_impl(f, std::make_integer_sequence<int, K>{});
}

// static-index select from a small register array (avoids local-memory indexing)
template <typename T, int K>
FROB_DEV T sel_k(const T (&v)[K], int idx) {
    T r = v[0];
#pragma unroll
    for (int i = 1; i < K; ++i)
        if (idx == i) r = v[i];
    return r;
}

// shared state of the sweep (double-buffered by step parity)
template <typename T, int N>
struct SweepShared1 {
    T slot[2][N / 4][N];   // each block-row's candidate row (double-buffered by step parity)
    unsigned long long candk[2][32];
    int candi[2][32];
    int pivrow[N];
    int pos[N];
    double pmag_k[N];
};

template <typename T, int N>
struct SweepShared {
    T colk[2][N];
    T rowp[2][N];
    unsigned long long candk[2][32];
    int candi[2][32];
    int pivrow[N];
    int pos[N];
    double pmag_k[N];
};

// after a sweep: pivot magnitude range (warp-parallel), identity for padding, pos[] = inverse
// of pivrow[]
template <typename T, int N, int NT, typename SH>
FROB_DEV void sweep_finish(SH &sh, int n, double &pmax, double &pmin) {
    const int tid = threadIdx.x, lane = tid & 31;
    double mx = 0.0, mn = INFINITY;
    for (int k = lane; k < n; k += 32) {
        mx = fmax(mx, sh.pmag_k[k]);
        mn = fmin(mn, sh.pmag_k[k]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    pmax = mx;
    pmin = mn;
    for (int k = tid; k < N; k += NT)
        if (k >= n) sh.pivrow[k] = k;
    __syncthreads();
    for (int k = tid; k < N; k += NT) sh.pos[sh.pivrow[k]] = k;
    __syncthreads();
}

// Gauss-Jordan sweep (exchange form, partial pivoting) on the register blocks a[BR][BC]
// over the leading n x n part of an N x N matrix (padding = identity).  On return the
// inverse, scattered: A^{-1}[pos[i]][pivrow[j]] = a(i, j).
template <typename T, int N, int BR, int BC>
FROB_DEV void gj_sweep(T (&a)[BR][BC], int n, SweepShared<T, N> &sh, double &pmax, double &pmin) {
    using G = Geo<N, BR, BC>;
    const int tid = threadIdx.x, lane = tid & 31;
    const int ti = tid / G::CT, tj = tid % G::CT;
    const int r0 = ti * BR, c0 = tj * BC;
    // loop-carried state is kept small (the 1024-thread n = 128 kernel has 64 registers):
    // used rows live in shared memory (pos[] doubles as the flag array), pivot magnitudes
    // are reduced after the loop
    for (int k = tid; k < N; k += G::THREADS) sh.pos[k] = 0;
    __syncthreads();
    // one step of the sweep; the column's position inside its register block (KC) is a
    // compile-time constant (the steps are unrolled by BC), so no register selects on it
    auto step = [&](const int k, auto KCc) {
        constexpr int KC = decltype(KCc)::value;
        const int par = k & 1;
        const bool owner = (tj == k / BC);
        if (owner) {
            unsigned long long bk = 0;
            int bi = INT_MAX;
#pragma unroll
            for (int q = 0; q < BR; ++q) {
                const int r = r0 + q;
                const T v = a[q][KC];
                sh.colk[par][r] = v;
                if (r < n && !sh.pos[r]) {
                    const unsigned long long kk = pkey_bits(v);
                    if (kk > bk) { bk = kk; bi = r; }
                }
            }
            sh.candk[par][ti] = bk;
            sh.candi[par][ti] = bi;
        }
        __syncthreads();
        const ArgMaxK m = warp_argmax_key(lane < G::RT ? sh.candk[par][lane] : 0ull,
                                          lane < G::RT ? sh.candi[par][lane] : INT_MAX);
        const int p = m.i;
        const T piv = sh.colk[par][p];
        if (tid == 0) { sh.pivrow[k] = p; sh.pmag_k[k] = pmag(piv); sh.pos[p] = 1; }
        if (ti == p / BR) {
            // 1/piv only where it is used: the pivot row's block-row scales the row for everyone
            // (a correctly rounded division is a multi-instruction sequence with a slow-path branch)
            const T ip = is_zero(piv) ? zero_of(T()) : recip(piv);
            const int q = p % BR;
#pragma unroll
            for (int c = 0; c < BC; ++c) {
                T v = a[0][c];
#pragma unroll
                for (int qq = 1; qq < BR; ++qq)
                    if (q == qq) v = a[qq][c];
                sh.rowp[par][c0 + c] = (owner && c == KC) ? ip : mul(v, ip);
            }
        }
        __syncthreads();
        T rp[BC], ck[BR];
#pragma unroll
        for (int c = 0; c < BC; ++c) rp[c] = sh.rowp[par][c0 + c];
#pragma unroll
        for (int q = 0; q < BR; ++q) ck[q] = sh.colk[par][r0 + q];
        // uniform exchange-form update: the owner of column k zeroes it first (a - ck * rp then
        // gives -ck / piv there), the pivot row is written last
        if (owner) {
#pragma unroll
            for (int q = 0; q < BR; ++q) a[q][KC] = zero_of(T());
        }
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) a[q][c] = msub(a[q][c], ck[q], rp[c]);
        if (ti == p / BR) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
                if (r0 + q == p) {
#pragma unroll
                    for (int c = 0; c < BC; ++c) a[q][c] = rp[c];
                }
        }
    };
    for (int kb = 0; kb * BC < n; ++kb) {
        bstatic_for<BC>([&](auto KCc) {
            constexpr int KC = decltype(KCc)::value;
            const int k = kb * BC + KC;
            if (k < n) step(k, KCc);
        });
    }
    __syncthreads();
    sweep_finish<T, N, G::THREADS>(sh, n, pmax, pmin);
}

// One barrier per step.  Thread (ti, tj) owns rows ti*BR.., columns tj*BC..; the CT threads
// of a block-row are consecutive lanes of one warp, so the column-k values of a block-row come
// by shuffle from the lane owning column block k/BC.  Each block-row publishes its best row
// for column k (with the candidate) before the barrier; after it, the pivot row is read from
// the winning block-row's slot, so no second barrier is needed.
template <typename T, int N, int BR, int BC>
FROB_DEV void gj_sweep_1bar(T (&a)[BR][BC], int n, SweepShared1<T, N> &sh, double &pmax, double &pmin) {
    using G = Geo<N, BR, BC>;
    static_assert(BR == 4, "slot layout assumes 4-row blocks");
    static_assert((G::CT & (G::CT - 1)) == 0 && G::CT <= 32, "block-rows must be lane groups");
    const int tid = threadIdx.x, lane = tid & 31;
    const int ti = tid / G::CT, tj = tid % G::CT;
    const int r0 = ti * BR, c0 = tj * BC;
    const int gbase = lane & ~(G::CT - 1);  // first lane of my block-row group
    unsigned used = 0;                      // my rows already used as pivots
    // steps unrolled by BC: the column's position in its register block (KC) is static
    auto step = [&](const int k, auto KCc) {
        constexpr int KC = decltype(KCc)::value;
        const int par = k & 1;
        const int kb = k / BC;
        // column-k values of my block-row (before this step's update)
        T ck[BR];
#pragma unroll
        for (int q = 0; q < BR; ++q) ck[q] = shfl(a[q][KC], gbase + kb);
        unsigned long long bk = 0;
        int qb = 0;
#pragma unroll
        for (int q = 0; q < BR; ++q) {
            if (r0 + q < n && !((used >> q) & 1u)) {
                const unsigned long long kk = pkey_bits(ck[q]);
                if (kk > bk) { bk = kk; qb = q; }
            }
        }
        if (tj == 0) {
            sh.candk[par][ti] = bk;
            sh.candi[par][ti] = bk ? r0 + qb : INT_MAX;
        }
#pragma unroll
        for (int c = 0; c < BC; ++c) {
            T v = a[0][c];
#pragma unroll
            for (int q = 1; q < BR; ++q)
                if (qb == q) v = a[q][c];
            sh.slot[par][ti][c0 + c] = v;
        }
        __syncthreads();
        const ArgMaxK m = warp_argmax_key(lane < G::RT ? sh.candk[par][lane] : 0ull,
                                          lane < G::RT ? sh.candi[par][lane] : INT_MAX);
        const int p = m.i;
        const int tip = p / BR;
        const T piv = sh.slot[par][tip][k];
        // every thread scales its own copy of the pivot row: the branch-free reciprocal for real
        // pivots (MUFU + two Newton steps, ~1 ulp) instead of the correctly rounded division
        const T ip = is_zero(piv) ? zero_of(T()) : fast_recip(piv);
        if (tid == 0) { sh.pivrow[k] = p; sh.pmag_k[k] = pmag(piv); }
        if (tip == ti) used |= 1u << (p - r0);
        // exchange-form update, uniform over the block: the owner of column k first zeroes it
        // and puts 1/piv into the pivot-row vector, so a - ck * rp gives -ck/piv there; the
        // pivot row is overwritten with rp afterwards
        T rp[BC];
#pragma unroll
        for (int c = 0; c < BC; ++c) rp[c] = mul(sh.slot[par][tip][c0 + c], ip);
        if (tj == kb) {
            rp[KC] = ip;
#pragma unroll
            for (int q = 0; q < BR; ++q) a[q][KC] = zero_of(T());
        }
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) a[q][c] = msub(a[q][c], ck[q], rp[c]);
        if (ti == tip) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
                if (r0 + q == p) {
#pragma unroll
                    for (int c = 0; c < BC; ++c) a[q][c] = rp[c];
                }
        }
    };
    for (int kb = 0; kb * BC < n; ++kb) {
        bstatic_for<BC>([&](auto KCc) {
            constexpr int KC = decltype(KCc)::value;
            const int k = kb * BC + KC;
            if (k < n) step(k, KCc);
        });
    }
    __syncthreads();
    sweep_finish<T, N, G::THREADS>(sh, n, pmax, pmin);
}

// write the sweep result as the inverse into a row-major matrix M (stride ldm)
template <typename T, int N, int BR, int BC, typename SH>
FROB_DEV void sweep_store(const T (&a)[BR][BC], const SH &sh, T *M, int ldm) {
    using G = Geo<N, BR, BC>;
    const int tid = threadIdx.x;
    const int r0 = (tid / G::CT) * BR, c0 = (tid % G::CT) * BC;
#pragma unroll
    for (int q = 0; q < BR; ++q) {
        const int orow = sh.pos[r0 + q];
#pragma unroll
        for (int c = 0; c < BC; ++c) M[orow * ldm + sh.pivrow[c0 + c]] = a[q][c];
    }
}

// load register blocks through an accessor f(i, j) (only called for i, j < n);
// rows/cols >= n get identity padding
template <typename T, int N, int BR, int BC, typename F>
FROB_DEV void load_blocks_f(T (&a)[BR][BC], int n, F f) {
    using G = Geo<N, BR, BC>;
    const int tid = threadIdx.x;
    const int r0 = (tid / G::CT) * BR, c0 = (tid % G::CT) * BC;
#pragma unroll
    for (int q = 0; q < BR; ++q)
#pragma unroll
        for (int c = 0; c < BC; ++c) {
            const int i = r0 + q, j = c0 + c;
            a[q][c] = (i < n && j < n) ? f(i, j) : ((i == j) ? one_of(T()) : zero_of(T()));
        }
}
template <typename T, int N>
FROB_DEV void load_blocks(T (&a)[4][4], const T *M, int n) {
    load_blocks_f<T, N, 4, 4>(a, n, [&](int i, int j) { return M[i * BCfg<N>::S + j]; });
}

// first 1-based pivot column with |u_kk| < 100 n u max (reading R2), 0 if none
template <typename T, int N, typename SH>
FROB_DEV int sweep_info(const SH &sh, int n, double pmax) {
    const double thr = 100.0 * n * 1.1102230246251565e-16 * pmax;
    const int lane = threadIdx.x & 31;
    int first = INT_MAX;
    for (int k = lane; k < n; k += 32)
        if (!(sh.pmag_k[k] >= thr) || sh.pmag_k[k] == 0.0) { first = k; break; }
    first = (int)redux_min((unsigned)first);
    return first == INT_MAX ? 0 : first + 1;
}

// ----------------------------------------------------------------- in-CTA DMMA GEMM
// acc = X * Y over the N x N smem operands (stride S). Warp tiling per N.
template <int N> struct WT;
template <> struct WT<32> { static constexpr int WGM = 2, WGN = 1, MT = 2, NT = 4; };
template <> struct WT<64> { static constexpr int WGM = 2, WGN = 4, MT = 4, NT = 2; };
template <> struct WT<128> { static constexpr int WGM = 2, WGN = 8, MT = 4, NT = 2; };  // per 64-row half, 16 warps

// acc = op_A * op_B over an N x N x N product with operands given by accessors
// fa(row, k) and fb(k, col) (shared or global memory; DMMA fragments loaded directly).
template <int N, typename FA, typename FB>
FROB_DEV void cta_mma_f(FA fa, FB fb, double (&acc)[WT<N>::MT][WT<N>::NT][2], int row_off = 0) {
    using W = WT<N>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = row_off + (warp / W::WGN) * (W::MT * 8), wn0 = (warp % W::WGN) * (W::NT * 8);
#pragma unroll
    for (int i = 0; i < W::MT; ++i)
#pragma unroll
        for (int j = 0; j < W::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 2
    for (int kk = 0; kk < N; kk += 4) {
        double a[W::MT], b[W::NT];
#pragma unroll
        for (int i = 0; i < W::MT; ++i) a[i] = fa(wm0 + i * 8 + g, kk + t);
#pragma unroll
        for (int j = 0; j < W::NT; ++j) b[j] = fb(kk + t, wn0 + j * 8 + g);
#pragma unroll
        for (int i = 0; i < W::MT; ++i)
#pragma unroll
            for (int j = 0; j < W::NT; ++j) dmma_s(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
}

template <int N>
FROB_DEV void cta_mma(const double *Xs, const double *Ys, int kmax, double (&acc)[WT<N>::MT][WT<N>::NT][2]) {
    using C = BCfg<N>;
    using W = WT<N>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp / W::WGN) * (W::MT * 8), wn0 = (warp % W::WGN) * (W::NT * 8);
#pragma unroll
    for (int i = 0; i < W::MT; ++i)
#pragma unroll
        for (int j = 0; j < W::NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kk = 0; kk < kmax; kk += 4) {
        double a[W::MT], b[W::NT];
#pragma unroll
        for (int i = 0; i < W::MT; ++i) a[i] = Xs[(wm0 + i * 8 + g) * C::S + kk + t];
#pragma unroll
        for (int j = 0; j < W::NT; ++j) b[j] = Ys[(kk + t) * C::S + wn0 + j * 8 + g];
#pragma unroll
        for (int i = 0; i < W::MT; ++i)
#pragma unroll
            for (int j = 0; j < W::NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
}

template <int N, typename F>
FROB_DEV void cta_mma_foreach(const double (&acc)[WT<N>::MT][WT<N>::NT][2], F f, int row_off = 0) {
    using W = WT<N>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = row_off + (warp / W::WGN) * (W::MT * 8), wn0 = (warp % W::WGN) * (W::NT * 8);
#pragma unroll
    for (int i = 0; i < W::MT; ++i)
#pragma unroll
        for (int j = 0; j < W::NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) f(wm0 + i * 8 + g, wn0 + j * 8 + 2 * t + e, acc[i][j][e]);
}

// ----------------------------------------------------------------- AUTO rule R1' helpers
// block-wide maximum (all threads call; scratch >= 32 doubles; returns the max to every thread)
FROB_DEV double block_max(double v, double *scratch, int nthreads) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
    __syncthreads();
    double m = 0.0;
    for (int i = 0; i < (nthreads + 31) / 32; ++i) m = fmax(m, scratch[i]);
    __syncthreads();
    return m;
}

// ||M||_inf of the leading n x n part through an accessor (row sums in fixed order)
template <typename F>
FROB_DEV double mat_norm_inf(int n, F f, double *scratch, int nthreads) {
    double m = 0.0;
    for (int r = threadIdx.x; r < n; r += nthreads) {
        double sum = 0.0;
        for (int c = 0; c < n; ++c) sum += fabs(f(r, c));
        m = fmax(m, sum);
    }
    return block_max(m, scratch, nthreads);
}

// ||X^{-1}||_inf of the inverse a Gauss-Jordan sweep left in the register blocks: the blocks hold
// a row and column permutation of it (padding rows >= n: identity, padding columns: zero), which
// leaves the maximum absolute row sum unchanged.  The CT threads of a block-row are consecutive
// lanes of one warp, so each row sum is a shuffle reduction; scratch: >= 32 doubles.
template <int N, int BR, int BC>
FROB_DEV double reg_norm_inf(const double (&a)[BR][BC], int n, double *scratch) {
    using G = Geo<N, BR, BC>;
    static_assert((G::CT & (G::CT - 1)) == 0 && G::CT <= 32, "block-rows must be lane groups");
    const int tid = threadIdx.x, r0 = (tid / G::CT) * BR;
    double m = 0.0;
#pragma unroll
    for (int q = 0; q < BR; ++q) {
        double sum = 0.0;
#pragma unroll
        for (int c = 0; c < BC; ++c) sum += fabs(a[q][c]);
#pragma unroll
        for (int o = 1; o < G::CT; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (r0 + q < n) m = fmax(m, sum);
    }
    return block_max(m, scratch, G::THREADS);
}

// ----------------------------------------------------------------- Frobenius kernel
// n <= 32: one-barrier sweep (measured 6% faster); n <= 64: two-barrier sweep (the one-barrier
// variant's candidate-row publishing costs more than the barrier it saves, 7.0 vs 10.0 ms)
template <int N> struct FrobSweep { using SH = SweepShared<double, N>; };
template <> struct FrobSweep<32> { using SH = SweepShared1<double, 32>; };
template <int N>
FROB_DEV void frob_sweep(double (&a)[4][4], int n, SweepShared<double, N> &sh, double &pmax, double &pmin) {
    gj_sweep<double, N, 4, 4>(a, n, sh, pmax, pmin);
}
template <int N>
FROB_DEV void frob_sweep(double (&a)[4][4], int n, SweepShared1<double, N> &sh, double &pmax, double &pmin) {
    gj_sweep_1bar<double, N, 4, 4>(a, n, sh, pmax, pmin);
}
template <int N>
struct FrobSmem {
    double buf[3][N * BCfg<N>::S];
    typename FrobSweep<N>::SH sw;
};

template <int N>
__global__ void __launch_bounds__(BCfg<N>::THREADS)
frob_batched_kernel(const double2 *__restrict__ Z, long long sZ, double2 *__restrict__ X, long long sX,
                    int n, int branch, int *__restrict__ info, unsigned char *__restrict__ bused) {
    using C = BCfg<N>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    FrobSmem<N> &sm = *reinterpret_cast<FrobSmem<N> *>(smem_raw);
    const int tid = threadIdx.x;
    const long long b = blockIdx.x;
    const double2 *Zb = Z + b * sZ;
    double2 *Xb = X + b * sX;
    double *As = sm.buf[0], *Bs = sm.buf[1], *Ws = sm.buf[2];

    // a0: coalesced interleaved load -> planar A, B (zero padded)
    for (int idx = tid; idx < N * N; idx += C::THREADS) {
        const int i = idx / N, j = idx - i * N;
        double2 z = make_double2(0.0, 0.0);
        if (i < n && j < n) z = Zb[i * n + j];
        As[i * C::S + j] = z.x;
        Bs[i * C::S + j] = z.y;
    }
    __syncthreads();

    double a[4][4];
    double pmax, pmin;
    int use = (branch == FROB_BRANCH_B) ? 2 : 1;
    load_blocks<double, N>(a, use == 1 ? As : Bs, n);
    frob_sweep<N>(a, n, sm.sw, pmax, pmin);
    int inf_x = sweep_info<double, N>(sm.sw, n, pmax);
    sweep_store<double, N, 4, 4>(a, sm.sw, Ws, C::S);
    if (branch == FROB_BRANCH_AUTO) {
        // reading R1': kappa_inf(A) from the computed inverse; above kappa_switch(n) (or A singular)
        // sweep B too and keep the part with the smaller kappa_inf
        const double na = mat_norm_inf(n, [&](int i, int j) { return As[i * C::S + j]; }, sm.sw.pmag_k, C::THREADS);
        const double ka = inf_x ? INFINITY : na * reg_norm_inf<N, 4, 4>(a, n, sm.sw.pmag_k);
        if (inf_x != 0 || !(ka <= kappa_switch(n))) {
            __syncthreads();
            load_blocks<double, N>(a, Bs, n);
            double qmax, qmin;
            frob_sweep<N>(a, n, sm.sw, qmax, qmin);
            const int inf_b = sweep_info<double, N>(sm.sw, n, qmax);
            const double nb = mat_norm_inf(n, [&](int i, int j) { return Bs[i * C::S + j]; }, sm.sw.pmag_k, C::THREADS);
            const double kb = inf_b ? INFINITY : nb * reg_norm_inf<N, 4, 4>(a, n, sm.sw.pmag_k);
            if (inf_b == 0 && (inf_x != 0 || kb < ka)) {
                use = 2;
                inf_x = 0;
                __syncthreads();
                sweep_store<double, N, 4, 4>(a, sm.sw, Ws, C::S);
            } else if (inf_b != 0 && inf_x != 0) {
                inf_x = -1;  // both singular
            }
        }
    }
    __syncthreads();
    double *Xs = (use == 1) ? As : Bs;   // X of Alg 1
    double *Ys = (use == 1) ? Bs : As;   // Y of Alg 1 (S2: Y = -A via sgn)
    const double sgn = (use == 1) ? 1.0 : -1.0;

    // a3: C = X^{-1} (sgn Y)  -> Ws (after everyone has read X^{-1})
    double acc[WT<N>::MT][WT<N>::NT][2];
    cta_mma<N>(Ws, Ys, N, acc);
    __syncthreads();
    cta_mma_foreach<N>(acc, [&](int i, int j, double v) { Ws[i * C::S + j] = sgn * v; });
    __syncthreads();
    // a4: M = X + (sgn Y) C  -> Xs
    cta_mma<N>(Ys, Ws, N, acc);
    __syncthreads();
    cta_mma_foreach<N>(acc, [&](int i, int j, double v) {
        Xs[i * C::S + j] = (i < n && j < n) ? fma(sgn, v, Xs[i * C::S + j]) : 0.0;
    });
    __syncthreads();
    // a5: Re = M^{-1} -> Ys
    load_blocks<double, N>(a, Xs, n);
    frob_sweep<N>(a, n, sm.sw, pmax, pmin);
    const int inf_m = sweep_info<double, N>(sm.sw, n, pmax);
    sweep_store<double, N, 4, 4>(a, sm.sw, Ys, C::S);
    __syncthreads();
    // a6/a7: Im = -C Re, interleaved store
    cta_mma<N>(Ws, Ys, N, acc);
    cta_mma_foreach<N>(acc, [&](int i, int j, double v) {
        if (i < n && j < n) {
            const double re = Ys[i * C::S + j];
            Xb[i * n + j] = (use == 1) ? make_double2(re, -v) : make_double2(-v, -re);
        }
    });
    if (tid == 0) {
        info[b] = (inf_x < 0) ? 1 : (inf_x ? inf_x : inf_m);
        if (bused) bused[b] = (inf_x < 0) ? 0 : (unsigned char)use;
    }
}

// ----------------------------------------------------------------- Frobenius, n <= 32: one warp per matrix
// Lane i holds row i of the matrix being inverted, so the pivot search of a column is a warp REDUX
// (no block barrier) and the pivot row is the pivot lane's own registers (it scales the row and
// publishes it through shared memory; no select trees).  The three GEMMs are 32 x 32 x 32 DMMA
// products.  Per warp only W (X^{-1}, then C, then M, then Re) lives in shared memory; the parts A, B
// are read from L1 / L2 where a step needs them and C also goes to the second half of the output
// matrix for a6 -- 10 KB of shared memory and <= 128 registers per warp, 16 warps per SM.
#ifndef FROB_W32_WARPS
#define FROB_W32_WARPS 4
#endif
constexpr int W32_WARPS = FROB_W32_WARPS;  // matrices per CTA (A/B build knob)
constexpr int W32_S = 36;     // shared row stride (doubles)
struct W32Smem {
    double W[32 * W32_S];
    double rp[2][32];         // the scaled pivot row (by step parity)
    int pivrow[32], pos[32];
    double pmag[32];
};

// exchange-form Gauss-Jordan sweep on the rows in registers (lane = row), partial pivoting, first
// maximum; on return row i holds inverse[pos[i]][pivrow[j]] = a[j].  Returns the LAPACK-style info
// (reading R2) and the max abs row sum of the inverse (for R1').
FROB_DEV int w32_sweep(double (&a)[32], int n, W32Smem &sm, double &nrm_inv) {
    const int lane = threadIdx.x & 31;
    bool used = false;
    bstatic_for<32>([&](auto kk) {
        constexpr int k = decltype(kk)::value;
        const bool el = !used && ((lane < n) == (k < n));
        const unsigned long long key = el ? pkey_bits(a[k]) : 0ull;
        const unsigned hi = (unsigned)(key >> 32), lo32 = (unsigned)key;
        const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo32 : 0u);
        const int p = (int)__reduce_min_sync(0xffffffffu, (key != 0ull && hi == mh && lo32 == ml) ? (unsigned)lane : 0xffffffffu);
        double *rp = sm.rp[k & 1];
        if (lane == p) {
            const double piv = a[k];
            const double ip = (piv == 0.0) ? 0.0 : frcp(piv);
#pragma unroll
            for (int j = 0; j < 32; ++j) a[j] = (j == k) ? ip : a[j] * ip;
#pragma unroll
            for (int h = 0; h < 16; ++h) *reinterpret_cast<double2 *>(&rp[2 * h]) = make_double2(a[2 * h], a[2 * h + 1]);
            used = true;
            sm.pivrow[k] = p;
            sm.pmag[k] = fabs(piv);
        }
        __syncwarp();
        if (lane != p) {
            const double ck = a[k];
            a[k] = 0.0;
#pragma unroll
            for (int h = 0; h < 16; ++h) {
                const double2 r = *reinterpret_cast<const double2 *>(&rp[2 * h]);
                a[2 * h] = fma(-ck, r.x, a[2 * h]);
                a[2 * h + 1] = fma(-ck, r.y, a[2 * h + 1]);
            }
        }
    });
    __syncwarp();
    sm.pos[sm.pivrow[lane]] = lane;
    double rs = 0.0;
#pragma unroll
    for (int j = 0; j < 32; ++j) rs += fabs(a[j]);
    double m = (lane < n) ? rs : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    nrm_inv = m;
    // reading R2: first pivot column with |u_kk| < 100 n u max|u_ii| (or exactly 0)
    double pm = (lane < n) ? sm.pmag[lane] : 0.0;
    double pmax = pm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    const double thr = 100.0 * n * 1.1102230246251565e-16 * pmax;
    const bool bad = (lane < n) && (!(pm >= thr) || pm == 0.0);
    const unsigned bm = __ballot_sync(0xffffffffu, bad);
    __syncwarp();
    return bm ? __ffs(bm) : 0;
}

// the sweep result (scrambled rows) -> M as the plain inverse
FROB_DEV void w32_store(const double (&a)[32], const W32Smem &sm, double *M) {
    const int lane = threadIdx.x & 31;
    const int orow = sm.pos[lane];
#pragma unroll
    for (int j = 0; j < 32; ++j) M[orow * W32_S + sm.pivrow[j]] = a[j];
}

// acc (16 tiles of 8 x 8: tile (i, j) rows 8 i + g, columns 8 j + 2 t + e) = A B over K = 32,
// fragments through accessors
template <typename FA, typename FB>
FROB_DEV void w32_mma(FA fa, FB fb, double (&acc)[4][4][2]) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 2
    for (int kk = 0; kk < 32; kk += 4) {
        double av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = fa(8 * i + g, kk + t);
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = fb(kk + t, 8 * j + g);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_s(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
}

template <typename F>
FROB_DEV void w32_foreach(const double (&acc)[4][4][2], F f) {
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) f(8 * i + g, 8 * j + 2 * t + e, acc[i][j][e]);
}

__global__ void __launch_bounds__(32 * W32_WARPS, 16 / W32_WARPS)
frob_batched32w_kernel(const double2 *__restrict__ Z, long long sZ, double2 *__restrict__ X, long long sX, int n,
                       int batch, int branch, int *__restrict__ info, unsigned char *__restrict__ bused) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const long long b = (long long)blockIdx.x * W32_WARPS + wid;
    if (b >= batch) return;  // whole warps only (no block barrier in this kernel)
    W32Smem &sm = reinterpret_cast<W32Smem *>(smem_raw)[wid];
    const double *Zd = reinterpret_cast<const double *>(Z + b * sZ);
    double2 *Xb = X + b * sX;
    double *Cg = reinterpret_cast<double *>(Xb) + (long long)n * n;  // planar C scratch (second half)
    auto part = [&](int p, int i, int j) { return (i < n && j < n) ? Zd[2 * (i * n + j) + p] : 0.0; };

    int use = (branch == FROB_BRANCH_B) ? 2 : 1;
    double a[32];
    // row `lane` of part xp (identity padding) -> registers
    auto load_rows = [&](int xp) {
#pragma unroll
        for (int j = 0; j < 32; ++j) a[j] = (lane < n && j < n) ? Zd[2 * (lane * n + j) + xp] : (lane == j ? 1.0 : 0.0);
    };
    auto row_norm = [&]() {  // ||X||_inf of the part in registers (rows < n)
        double rs = 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) rs += fabs(a[j]);
        double m = (lane < n) ? rs : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        return m;
    };
    load_rows(use - 1);
    double nx = row_norm(), ni;
    int inf_x = w32_sweep(a, n, sm, ni);
    w32_store(a, sm, sm.W);
    if (branch == FROB_BRANCH_AUTO) {
        // reading R1' (see frob_batched_kernel)
        const double ka = inf_x ? INFINITY : nx * ni;
        if (inf_x != 0 || !(ka <= kappa_switch(n))) {
            // B into the registers (its rows); A's inverse stays in W in case B is not better
            load_rows(1);
            const double nb = row_norm();
            double nib;
            const int inf_b = w32_sweep(a, n, sm, nib);
            const double kb = inf_b ? INFINITY : nb * nib;
            if (inf_b == 0 && (inf_x != 0 || kb < ka)) {
                use = 2;
                inf_x = 0;
                w32_store(a, sm, sm.W);
            } else if (inf_b != 0 && inf_x != 0) {
                inf_x = -1;  // both singular
            }
        }
    }
    __syncwarp();
    const double sgn = (use == 1) ? 1.0 : -1.0;  // Y of Alg 1 (S2: Y = -A)
    const int xp = use - 1, yp = 2 - use;
    auto Yv = [&](int i, int j) { return part(yp, i, j); };  // raw Y; the sign goes on C
    double acc[4][4][2];
    // a3: C = X^{-1} (sgn Y) -> W (X^{-1} is then done) and -> Cg
    w32_mma([&](int r, int k) { return sm.W[r * W32_S + k]; }, Yv, acc);
    __syncwarp();
    w32_foreach(acc, [&](int i, int j, double v) {
        sm.W[i * W32_S + j] = sgn * v;
        if (i < n && j < n) Cg[i * n + j] = sgn * v;
    });
    __syncwarp();
    // a4: M = X + (sgn Y) C -> W
    w32_mma(Yv, [&](int k, int c) { return sm.W[k * W32_S + c]; }, acc);
    __syncwarp();
    w32_foreach(acc, [&](int i, int j, double v) { sm.W[i * W32_S + j] = (i < n && j < n) ? fma(sgn, v, part(xp, i, j)) : 0.0; });
    __syncwarp();
    // a5: Re = M^{-1} -> W
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = (lane < n && j < n) ? sm.W[lane * W32_S + j] : (lane == j ? 1.0 : 0.0);
    double nm;
    const int inf_m = w32_sweep(a, n, sm, nm);
    w32_store(a, sm, sm.W);
    __syncwarp();
    // a6/a7: Im = -C Re, interleaved store
    w32_mma([&](int r, int k) { return (r < n && k < n) ? Cg[r * n + k] : 0.0; },
            [&](int k, int c) { return sm.W[k * W32_S + c]; }, acc);
    __syncwarp();
    w32_foreach(acc, [&](int i, int j, double v) {
        if (i < n && j < n) {
            const double re = sm.W[i * W32_S + j];
            Xb[i * n + j] = (use == 1) ? make_double2(re, -v) : make_double2(-v, -re);
        }
    });
    if (lane == 0) {
        info[b] = (inf_x < 0) ? 1 : (inf_x ? inf_x : inf_m);
        if (bused) bused[b] = (inf_x < 0) ? 0 : (unsigned char)use;
    }
}

// Complex comparator, n <= 32, in the same row-per-lane warp design (a like-for-like n = 32 comparison):
// complex Gauss-Jordan (exchange form, partial pivoting on |re|+|im|, first maximum), lane i = row i.
struct Z32Smem {
    double2 rp[2][32];
    int pivrow[32], pos[32];
    double pmag[32];
};
#ifndef FROB_Z32_MINB
#define FROB_Z32_MINB 3  // 3 CTAs per SM (168 registers, some spilling): 3.54 vs 3.89 ms at 1 (A/B: tools/abz32.py)
#endif
__global__ void __launch_bounds__(32 * W32_WARPS, FROB_Z32_MINB)
zinv_batched32w_kernel(const double2 *__restrict__ Z, long long sZ, double2 *__restrict__ X, long long sX, int n,
                       int batch, int *__restrict__ info) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const long long b = (long long)blockIdx.x * W32_WARPS + wid;
    if (b >= batch) return;
    Z32Smem &sm = reinterpret_cast<Z32Smem *>(smem_raw)[wid];
    const double2 *Zb = Z + b * sZ;
    double2 *Xb = X + b * sX;
    double2 a[32];
#pragma unroll
    for (int j = 0; j < 32; ++j)
        a[j] = (lane < n && j < n) ? Zb[lane * n + j] : make_double2(lane == j ? 1.0 : 0.0, 0.0);
    bool used = false;
    bstatic_for<32>([&](auto kk) {
        constexpr int k = decltype(kk)::value;
        const bool el = !used && ((lane < n) == (k < n));
        const unsigned long long key = el ? pkey_bits(a[k]) : 0ull;
        const unsigned hi = (unsigned)(key >> 32), lo32 = (unsigned)key;
        const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo32 : 0u);
        const int p = (int)__reduce_min_sync(0xffffffffu, (key != 0ull && hi == mh && lo32 == ml) ? (unsigned)lane : 0xffffffffu);
        double2 *rp = sm.rp[k & 1];
        if (lane == p) {
            const double2 piv = a[k];
            const double2 ip = is_zero(piv) ? make_double2(0.0, 0.0) : fast_recip(piv);
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                a[j] = (j == k) ? ip : mul(a[j], ip);
                rp[j] = a[j];
            }
            used = true;
            sm.pivrow[k] = p;
            sm.pmag[k] = pmag(piv);
        }
        __syncwarp();
        if (lane != p) {
            const double2 ck = a[k];
            a[k] = make_double2(0.0, 0.0);
#pragma unroll
            for (int j = 0; j < 32; ++j) a[j] = msub(a[j], ck, rp[j]);
        }
    });
    __syncwarp();
    sm.pos[sm.pivrow[lane]] = lane;
    __syncwarp();
    // reading R2 (as sweep_info): first pivot column with |u_kk| < 100 n u max|u_ii| (or exactly 0)
    const double pm = (lane < n) ? sm.pmag[lane] : 0.0;
    double pmax = pm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pmax = fmax(pmax, __shfl_xor_sync(0xffffffffu, pmax, o));
    const double thr = 100.0 * n * 1.1102230246251565e-16 * pmax;
    const unsigned bm = __ballot_sync(0xffffffffu, (lane < n) && (!(pm >= thr) || pm == 0.0));
    const int orow = sm.pos[lane];
    if (orow < n) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int c = sm.pivrow[j];
            if (c < n) Xb[orow * n + c] = a[j];
        }
    }
    if (lane == 0) info[b] = bm ? __ffs(bm) : 0;
}

// ----------------------------------------------------------------- in-CTA GEMM, N = 128, staged operand
// acc0 / acc1 (rows 0..63 / 64..127, the WT<128> warp tiling) = A B over K = 128.  The operand read
// from L2 (A if STAGE_A, else B) goes through 16-wide k-slabs in shared memory (two buffers; the next
// slab's four elements per thread are loaded into registers while the current slab is consumed);
// the other one comes through `fo` (shared memory).  Replaces fragment loads straight from L2.
constexpr int SLAB_K = 16, SLAB_AS = 20, SLAB_BS = 132;  // k per slab, A-slab / B-slab row strides
constexpr int SLAB_DOUBLES = 2 * 128 * SLAB_AS;          // >= 2 * SLAB_K * SLAB_BS
struct ZeroInit {
    FROB_DEV double operator()(int, int) const { return 0.0; }
};
template <bool STAGE_A, typename FG, typename FO, typename FI = ZeroInit>
FROB_DEV void cta_mma2_staged(FG fg, FO fo, double *slab, double (&acc0)[WT<128>::MT][WT<128>::NT][2],
                              double (&acc1)[WT<128>::MT][WT<128>::NT][2], FI fi = FI()) {
    using W = WT<128>;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp / W::WGN) * (W::MT * 8), wn0 = (warp % W::WGN) * (W::NT * 8);
    constexpr int BUF = STAGE_A ? 128 * SLAB_AS : SLAB_K * SLAB_BS;
    // accumulator (row, col) of element (i, j, e): (wm0 + 8 i + g [+ 64], wn0 + 8 j + 2 t + e)
#pragma unroll
    for (int i = 0; i < W::MT; ++i)
#pragma unroll
        for (int j = 0; j < W::NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                acc0[i][j][e] = fi(wm0 + i * 8 + g, wn0 + j * 8 + 2 * t + e);
                acc1[i][j][e] = fi(64 + wm0 + i * 8 + g, wn0 + j * 8 + 2 * t + e);
            }
    double v[4];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + 512 * q;
            v[q] = STAGE_A ? fg(e >> 4, k0 + (e & 15)) : fg(k0 + (e >> 7), e & 127);
        }
    };
    auto put = [&](double *buf) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = tid + 512 * q;
            if (STAGE_A) buf[(e >> 4) * SLAB_AS + (e & 15)] = v[q];
            else buf[(e >> 7) * SLAB_BS + (e & 127)] = v[q];
        }
    };
    fetch(0);
    put(slab);
    __syncthreads();
    for (int s = 0; s < 128 / SLAB_K; ++s) {
        const double *cur = slab + (s & 1) * BUF;
        if (s + 1 < 128 / SLAB_K) fetch((s + 1) * SLAB_K);
#pragma unroll
        for (int kk = 0; kk < SLAB_K; kk += 4) {
            const int kg = s * SLAB_K + kk;
            double a0[W::MT], a1[W::MT], b[W::NT];
#pragma unroll
            for (int i = 0; i < W::MT; ++i) {
                const int r = wm0 + i * 8 + g;
                a0[i] = STAGE_A ? cur[r * SLAB_AS + kk + t] : fo(r, kg + t);
                a1[i] = STAGE_A ? cur[(64 + r) * SLAB_AS + kk + t] : fo(64 + r, kg + t);
            }
#pragma unroll
            for (int j = 0; j < W::NT; ++j)
                b[j] = STAGE_A ? fo(kg + t, wn0 + j * 8 + g) : cur[(kk + t) * SLAB_BS + wn0 + j * 8 + g];
#pragma unroll
            for (int i = 0; i < W::MT; ++i)
#pragma unroll
                for (int j = 0; j < W::NT; ++j) {
                    dmma_s(acc0[i][j][0], acc0[i][j][1], a0[i], b[j]);
                    dmma_s(acc1[i][j][0], acc1[i][j][1], a1[i], b[j]);
                }
        }
        if (s + 1 < 128 / SLAB_K) put(slab + ((s + 1) & 1) * BUF);
        __syncthreads();
    }
}

// ----------------------------------------------------------------- Frobenius, 64 < n <= 128
// 512 threads.  The two inversions by the blocked, warp-specialised Gauss-Jordan sweep below
// (gj128_sweep); the three GEMMs by DMMA from shared / L1-resident operands (cta_mma_f).  One
// 135 KB shared buffer (X^{-1}, then M, then Re); C = X^{-1} Y lives in the second half of the
// OUTPUT matrix (planar n x n doubles) until the final epilogue overwrites it with the result.
// phase clock stamps of sampled CTAs (probe builds with -DFROB_B128_TL: tools/batched128_phases.py)
#ifdef FROB_B128_TL
__device__ long long g_b128_tl[16][8];
#define B128_TL(i) do { __syncthreads(); if (threadIdx.x == 0 && (blockIdx.x & 1023) == 0) \
    g_b128_tl[(blockIdx.x >> 10) & 15][i] = clock64(); } while (0)
extern "C" int frob_b128_tl_read(long long *h) {
    return (int)cudaMemcpyFromSymbol(h, g_b128_tl, sizeof(g_b128_tl));
}
// per-panel timeline of block 0's last sweep (plain stores, nothing waits on them)
__device__ long long g_g8tl[16][6];
#define G8_TL(b, slot) do { if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) g_g8tl[(b) & 15][slot] = clock64(); } while (0)
extern "C" int frob_g8_tl_read(long long *h) { return (int)cudaMemcpyFromSymbol(h, g_g8tl, sizeof(g_g8tl)); }
#else
#define B128_TL(i) do { } while (0)
#define G8_TL(b, slot) do { } while (0)
#endif

// ----------------------------------------------------------------- blocked Gauss-Jordan, N = 128
// The exchange-form sweep (same pivots as gj_sweep: partial pivoting, first maximum; result
// scattered as inverse[pos[i]][pivrow[j]] = element (i, j)) in 8-column panels.  The matrix lives
// in the DMMA accumulators of the 16 warps (each a 32 x 32 block of 8 x 8 tiles).  One warp (the
// panel warp) factors panel b in LU form in its registers (its own tiles parked in shared memory
// meanwhile): pivot search by REDUX, pivot row through shared memory, no block barrier; with M =
// A_RK = L11 U11 (rows R = the panel's pivot rows in order) and A_IK = L21 U11, sweeping the panel
// acts on every other column block J as
//     A_IJ -= L21 W,   A_RJ = V,   W = L11^-1 A_RJ,   V = U11^-1 W   (forward / back substitution)
//     A_IK = -L21 L11^-1,   A_RK = U11^-1 L11^-1.
// The other columns take the substitution form (rank-8 DMMA with the multipliers) -- NOT the product
// of the swept panel with the old pivot rows: that form rounds ~20x worse on ill-conditioned parts
// (tools/gj_block_accuracy.py), this one as well as the unblocked sweep.  The owners of the
// next panel's columns update them first and hand them over (look-ahead).
constexpr int G8_W = 8;                  // panel width
constexpr int G8_T = 512;                // 16 warps
constexpr int G8_PW = 15;                // the panel warp (tile rows 96.., tile columns 96..)
constexpr int G8_PS = 10;                // panel buffer row stride (doubles; 16-byte rows)
constexpr int G8_TS = 132;               // T / W / V buffer row stride
constexpr int G8_BAR_U = 1, G8_BAR_PANEL = 2, G8_BAR_FACT = 3;  // named barriers (0 = __syncthreads)
struct G8Shared {
    double pb[2][128 * G8_PS];   // panel b: handed to the panel warp, then its LU form (multipliers / U rows)
    double tb[2][G8_W * G8_TS];  // T = the pivot rows (old), then W
    double tw[G8_W * G8_TS];     // W (written after, read before a U barrier: one buffer)
    double tv[G8_W * G8_TS];     // V
    double park[32 * 32];        // the panel warp's own tiles while it factors a panel; norm row sums
    double lu[G8_W * G8_W];      // the panel's pivot rows (L11 strictly below, U11 on / above the diagonal)
    double rpiv[G8_W];           // 1 / u_cc
    double uinv[2][G8_W * G8_W]; // U11^-1 (by panel parity: the last owners of panel b read it while
    double linv[2][G8_W * G8_W]; // L11^-1    panel b+1's are formed)
    int prow[2][G8_W];
    signed char rowslot[2][128];  // panel slot of a pivot row, -1 otherwise
};
struct Frob128Smem {
    double S[128 * 132];
    SweepShared<double, 128> sw;
    union {
        G8Shared gs;                  // the sweeps
        double slab[SLAB_DOUBLES];    // the GEMMs' staged operand
    };
};

FROB_DEV void nbar_sync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
FROB_DEV void nbar_arrive(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }

// accumulator element (i, j, e) of warp w: row 32 (w >> 2) + 8 i + g, column 32 (w & 3) + 8 j + 2 t + e
template <typename F>
FROB_DEV void gj128_load(double (&a)[4][4][2], int n, F f) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = 32 * (warp >> 2) + (lane >> 2), c0 = 32 * (warp & 3) + 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = r0 + 8 * i, c = c0 + 8 * j + e;
                a[i][j][e] = (r < n && c < n) ? f(r, c) : (r == c ? 1.0 : 0.0);
            }
}

FROB_DEV void gj128_store(const double (&a)[4][4][2], const SweepShared<double, 128> &sh, double *M, int ldm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = 32 * (warp >> 2) + (lane >> 2), c0 = 32 * (warp & 3) + 2 * (lane & 3);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int orow = sh.pos[r0 + 8 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) M[orow * ldm + sh.pivrow[c0 + 8 * j + e]] = a[i][j][e];
    }
}

// max absolute row sum of the sweep result (rows < n); scratch >= 32 doubles
FROB_DEV double gj128_norm_inf(const double (&a)[4][4][2], int n, double *part, double *scratch) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int r0 = 32 * (warp >> 2) + (lane >> 2);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        double sum = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) sum += fabs(a[i][j][0]) + fabs(a[i][j][1]);
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        if ((lane & 3) == 0) part[(warp & 3) * 128 + r0 + 8 * i] = sum;
    }
    __syncthreads();
    double m = 0.0;
    const int r = threadIdx.x;
    if (r < n) m = ((part[r] + part[128 + r]) + part[256 + r]) + part[384 + r];
    return block_max(m, scratch, G8_T);
}

// The panel warp's LU factorisation of panel b: lane l holds rows l + 32 q (q < 4), panel column c
// in p[q][c >> 1][c & 1]; umask = my rows already used as pivots (earlier panels' pivot rows are
// ordinary rows here, as in the exchange form).  Per column the owner lane of the pivot row
// publishes it through shared memory; the chain is branch-free.
FROB_DEV void g8_panel(double (&p)[4][4][2], int b, int n, unsigned &umask, SweepShared<double, 128> &sh,
                       G8Shared &gs) {
    const int lane = threadIdx.x & 31, par = b & 1;
    double *pb = gs.pb[par];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const double2 v = *reinterpret_cast<const double2 *>(&pb[(lane + 32 * q) * G8_PS + 2 * h]);
            p[q][h][0] = v.x;
            p[q][h][1] = v.y;
        }
    if (b >= 2 && lane < G8_W) gs.rowslot[par][gs.prow[par][lane]] = -1;
    unsigned pmask = 0;                 // my rows pivoted in this panel (they hold U rows from then on)
    bstatic_for<G8_W>([&](auto cc) {
        constexpr int c = decltype(cc)::value;
        const int k = b * G8_W + c;
        // candidates, branch-free: key 0 = not eligible; first max (rows l + 32 q grow with q)
        unsigned long long kq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int r = lane + 32 * q;
            const bool el = !((umask >> q) & 1u) && ((r < n) == (k < n));
            kq[q] = el ? pkey_bits(p[q][c >> 1][c & 1]) : 0ull;
        }
        const bool s01 = kq[1] > kq[0], s23 = kq[3] > kq[2];
        const unsigned long long k01 = s01 ? kq[1] : kq[0], k23 = s23 ? kq[3] : kq[2];
        const bool s = k23 > k01;
        const unsigned long long bk = s ? k23 : k01;
        const int qb = s ? (s23 ? 3 : 2) : (s01 ? 1 : 0);
        const unsigned hi = (unsigned)(bk >> 32), lo32 = (unsigned)bk;
        const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
        const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo32 : 0u);
        const int pr = (int)__reduce_min_sync(0xffffffffu, (bk != 0ull && hi == mh && lo32 == ml)
                                                                 ? (unsigned)(lane + 32 * qb) : 0xffffffffu);
        const int qp = pr >> 5;
        const bool me = (lane == (pr & 31));
        double vq = p[0][c >> 1][c & 1];
        vq = (qp == 1) ? p[1][c >> 1][c & 1] : vq;
        vq = (qp == 2) ? p[2][c >> 1][c & 1] : vq;
        vq = (qp == 3) ? p[3][c >> 1][c & 1] : vq;
        const double piv = __shfl_sync(0xffffffffu, vq, pr & 31);
        // the pivot row (multipliers in columns < c, U in columns >= c) -> shared, by its owner
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (me && qp == q) {
#pragma unroll
                for (int h = 0; h < G8_W / 2; ++h)
                    *reinterpret_cast<double2 *>(&gs.lu[c * G8_W + 2 * h]) = make_double2(p[q][h][0], p[q][h][1]);
            }
        const unsigned bit = me ? (1u << qp) : 0u;
        pmask |= bit;
        umask |= bit;
        const double ip = (piv == 0.0) ? 0.0 : frcp(piv);
        if (lane == 0) {
            gs.rpiv[c] = ip;
            sh.pivrow[k] = pr;
            sh.pmag_k[k] = fabs(piv);
            gs.prow[par][c] = pr;
            gs.rowslot[par][pr] = (signed char)c;
        }
        __syncwarp();
        double u[G8_W];
#pragma unroll
        for (int c2 = c + 1; c2 < G8_W; ++c2) u[c2] = gs.lu[c * G8_W + c2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool up = !((pmask >> q) & 1u);
            const double m = p[q][c >> 1][c & 1] * ip;
            const double mm = up ? m : 0.0;
            p[q][c >> 1][c & 1] = up ? m : p[q][c >> 1][c & 1];
#pragma unroll
            for (int c2 = c + 1; c2 < G8_W; ++c2) p[q][c2 >> 1][c2 & 1] = fma(-mm, u[c2], p[q][c2 >> 1][c2 & 1]);
        }
    });
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int h = 0; h < 4; ++h)
            *reinterpret_cast<double2 *>(&pb[(lane + 32 * q) * G8_PS + 2 * h]) = make_double2(p[q][h][0], p[q][h][1]);
    __syncwarp();
}

// U11^-1 (Uinv U = I, column by column: Uinv[i][c] = -(sum_{k<c} Uinv[i][k] U[k][c]) / u_cc) by
// threads 0..7 (row i = thread) and L11^-1 (L Linv = I, row by row: Linv[c][j] = delta_cj -
// sum_{i<c} L[c][i] Linv[i][j]) by threads 8..15 (column j = thread - 8), from the LU-form pivot rows
FROB_DEV void g8_tri_inverses(G8Shared &gs, int ti, int par) {
    const bool urole = ti < G8_W;
    const int r = ti & (G8_W - 1);
    double tr[G8_W];
#pragma unroll
    for (int c = 0; c < G8_W; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < c; ++i) acc = fma(tr[i], urole ? gs.lu[i * G8_W + c] : gs.lu[c * G8_W + i], acc);
        const double ip = gs.rpiv[c];
        tr[c] = urole ? ((r == c) ? ip : (r < c ? -acc * ip : 0.0)) : ((r == c ? 1.0 : 0.0) - acc);
    }
#pragma unroll
    for (int j = 0; j < G8_W; ++j) {
        if (urole) gs.uinv[par][r * G8_W + j] = tr[j];
        else gs.linv[par][j * G8_W + r] = tr[j];
    }
}

FROB_DEV void gj128_sweep(double (&a)[4][4][2], int n, SweepShared<double, 128> &sh, G8Shared &gs, double &pmax,
                          double &pmin) {
    constexpr int NP = 128 / G8_W;
    const int tid = threadIdx.x, lane = tid & 31;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);  // warp-uniform for the compiler
    const int g = lane >> 2, t = lane & 3;
    const int wc = warp & 3, r0 = 32 * (warp >> 2) + g;
    const bool pw = (warp == G8_PW);
    unsigned umask = 0;
    for (int i = tid; i < 2 * 128; i += G8_T) (&gs.rowslot[0][0])[i] = -1;
    __syncthreads();
    // threads meeting at the panel-b hand-over: its four owner warps (+ the panel warp)
    auto panel_cnt = [](int b) { return ((b >> 2) == (G8_PW & 3)) ? 128 : 160; };
    auto hand_over = [&](int b, int jb) {  // my tiles of column block jb (panel b) -> panel buffer
        double *pb = gs.pb[b & 1];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j == jb) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    *reinterpret_cast<double2 *>(&pb[(r0 + 8 * i) * G8_PS + 2 * t]) = make_double2(a[i][j][0], a[i][j][1]);
            }
        if (!pw) nbar_arrive(G8_BAR_PANEL, panel_cnt(b));
    };
    auto run_panel = [&](int b) {  // panel warp: park my tiles, factor panel b, signal, restore
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) gs.park[(i * 8 + j * 2 + e) * 32 + lane] = a[i][j][e];
        nbar_sync(G8_BAR_PANEL, panel_cnt(b));
        G8_TL(b, 0);
        g8_panel(a, b, n, umask, sh, gs);
        nbar_arrive(G8_BAR_FACT, G8_T);
        G8_TL(b, 1);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) a[i][j][e] = gs.park[(i * 8 + j * 2 + e) * 32 + lane];
    };
    if (wc == 0) hand_over(0, 0);
    if (pw) run_panel(0);
    for (int b = 0; b < NP; ++b) {
        const int par = b & 1, jb = b & 3;
        const bool bown = (wc == (b >> 2));
        const int b1 = b + 1, j1 = b1 & 3;
        const bool nown = (b1 < NP) && (wc == (b1 >> 2));
        if (!pw) nbar_sync(G8_BAR_FACT, G8_T);
        if (warp == 0) G8_TL(b, 2);
        const double *pb = gs.pb[par];
        double *tb = gs.tb[par];
        double *tv = gs.tv;
        // T: my part of the panel's pivot rows, before the update
        int slot[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            slot[i] = gs.rowslot[par][r0 + 8 * i];
            if (slot[i] >= 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    *reinterpret_cast<double2 *>(&tb[slot[i] * G8_TS + 32 * wc + 8 * j + 2 * t]) =
                        make_double2(a[i][j][0], a[i][j][1]);
            }
        }
        // meanwhile 16 threads of warp 4 form U11^-1 and L11^-1
        if (tid >= 128 && tid < 128 + 2 * G8_W) g8_tri_inverses(gs, tid - 128, par);
        if (warp == 4) G8_TL(b, 5);
        nbar_sync(G8_BAR_U, G8_T);
        if (warp == 0) G8_TL(b, 3);
        // W = L11^-1 T and V = U11^-1 W (2 + 2 DMMA per 8-column tile) by warps 0..3, one 32-column band each
        if (warp < 4) {
            double *tw = gs.tw;
            const double l0 = gs.linv[par][g * G8_W + t], l1 = gs.linv[par][g * G8_W + 4 + t];
            const double u0 = gs.uinv[par][g * G8_W + t], u1 = gs.uinv[par][g * G8_W + 4 + t];
            double d[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                d[j][0] = d[j][1] = 0.0;
                dmma_s(d[j][0], d[j][1], l0, tb[t * G8_TS + 32 * wc + 8 * j + g]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_s(d[j][0], d[j][1], l1, tb[(4 + t) * G8_TS + 32 * wc + 8 * j + g]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                *reinterpret_cast<double2 *>(&tw[g * G8_TS + 32 * wc + 8 * j + 2 * t]) = make_double2(d[j][0], d[j][1]);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                d[j][0] = d[j][1] = 0.0;
                dmma_s(d[j][0], d[j][1], u0, tw[t * G8_TS + 32 * wc + 8 * j + g]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) dmma_s(d[j][0], d[j][1], u1, tw[(4 + t) * G8_TS + 32 * wc + 8 * j + g]);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                *reinterpret_cast<double2 *>(&tv[g * G8_TS + 32 * wc + 8 * j + 2 * t]) = make_double2(d[j][0], d[j][1]);
        }
        nbar_sync(G8_BAR_U, G8_T);
        if (warp == 0) G8_TL(b, 4);
        // A fragments: -(multipliers) for the rows outside the panel's pivots, 0 for those
        double pa[4][2];
        auto load_pa = [&]() {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const bool pv = gs.rowslot[par][r0 + 8 * i] >= 0;
                pa[i][0] = pv ? 0.0 : -pb[(r0 + 8 * i) * G8_PS + t];
                pa[i][1] = pv ? 0.0 : -pb[(r0 + 8 * i) * G8_PS + 4 + t];
            }
        };
        auto upd = [&](auto jj) {
            constexpr int j = decltype(jj)::value;
            const double t0 = gs.tw[t * G8_TS + 32 * wc + 8 * j + g];
            const double t1 = gs.tw[(4 + t) * G8_TS + 32 * wc + 8 * j + g];
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma_s(a[i][j][0], a[i][j][1], pa[i][0], t0);
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma_s(a[i][j][0], a[i][j][1], pa[i][1], t1);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (slot[i] >= 0) {
                    const double2 v = *reinterpret_cast<const double2 *>(&tv[slot[i] * G8_TS + 32 * wc + 8 * j + 2 * t]);
                    a[i][j][0] = v.x;
                    a[i][j][1] = v.y;
                }
            }
        };
        load_pa();
        if (nown) {  // the next panel's columns first
            bstatic_for<4>([&](auto jj) {
                if (decltype(jj)::value == j1) upd(jj);
            });
            hand_over(b1, j1);
        }
        // The panel warp factors panel b + 1 BEFORE the rest of its update b (off the chain: the
        // others wait at FACT for that factor only).  Safe: W / V (tw, tv) of panel b are rewritten
        // only after the first U barrier of b + 1, which the panel warp reaches after this update;
        // pb / rowslot / linv / uinv of panel b (parity b & 1) only in panel b + 2.  The factor uses
        // the accumulators as scratch (parked meanwhile), so pa and slot are read again afterwards.
        if (pw && b1 < NP) {
            run_panel(b1);
            load_pa();
#pragma unroll
            for (int i = 0; i < 4; ++i) slot[i] = gs.rowslot[par][r0 + 8 * i];
        }
        bstatic_for<4>([&](auto jj) {
            constexpr int j = decltype(jj)::value;
            if (!(bown && j == jb) && !(nown && j == j1)) upd(jj);
        });
        if (bown) {
            // my rows of the swept panel, straight into the accumulators: X L11^-1 with X = -(multipliers)
            // for a non-pivot row and X = row c of U11^-1 for pivot row p_c (two DMMA per tile)
            const double l0 = gs.linv[par][t * G8_W + g], l1 = gs.linv[par][(4 + t) * G8_W + g];
            const int ra = 32 * (warp >> 2);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j == jb) {
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int r = ra + 8 * i + g;  // the A-fragment row of this lane
                        const int sl = gs.rowslot[par][r];
                        const double x0 = (sl >= 0) ? gs.uinv[par][sl * G8_W + t] : -pb[r * G8_PS + t];
                        const double x1 = (sl >= 0) ? gs.uinv[par][sl * G8_W + 4 + t] : -pb[r * G8_PS + 4 + t];
                        a[i][j][0] = a[i][j][1] = 0.0;
                        dmma_s(a[i][j][0], a[i][j][1], x0, l0);
                        dmma_s(a[i][j][0], a[i][j][1], x1, l1);
                    }
                }
        }
    }
    __syncthreads();
    sweep_finish<double, 128, G8_T>(sh, n, pmax, pmin);
}

// Planar operand views of the interleaved input: part 0 = Re Z = A, part 1 = Im Z = B.
FROB_DEV double zpart(const double *Zd, int n, int part, int i, int j) { return Zd[2 * (i * n + j) + part]; }

// One copy of each step in the kernel (the part in use, its sign and the output layout are runtime
// values): the unrolled sweep and GEMM bodies are large.
__global__ void __launch_bounds__(G8_T, 1)
frob_batched128_kernel(const double2 *__restrict__ Z, long long sZ, double2 *__restrict__ X, long long sX, int n,
                       int branch, int *__restrict__ info, unsigned char *__restrict__ bused) {
    constexpr int N = 128, SS = 132;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Frob128Smem &sm = *reinterpret_cast<Frob128Smem *>(smem_raw);
    double *S = sm.S;
    const int tid = threadIdx.x;
    const long long b = blockIdx.x;
    const double *Zd = reinterpret_cast<const double *>(Z + b * sZ);
    double2 *Xb = X + b * sX;
    // scratch: planar C (n x n) in the SECOND half of the output matrix, so the final
    // epilogue for rows < 64 (bytes [0, 1024 n)) never clobbers C rows >= 64 (n >= 64)
    double *Cg = reinterpret_cast<double *>(Xb) + (long long)n * n;

    int use = (branch == FROB_BRANCH_B) ? 2 : 1;
    int inf_x = 0, inf_m = 0;
    double ka = 0.0;
    B128_TL(0);
    // pass 0: X^{-1} of the part in use; pass 1 (AUTO, reading R1'): the other part; pass 2: M^{-1}
    for (int pass = 0;;) {
        double a[4][4][2];
        double pmax, pmin;
        const int xpart = (pass == 0) ? use - 1 : 2 - use;  // the part swept in passes 0 / 1
        if (pass < 2) gj128_load(a, n, [&](int i, int j) { return zpart(Zd, n, xpart, i, j); });
        else gj128_load(a, n, [&](int i, int j) { return S[i * SS + j]; });
        // ||part||_inf for the AUTO rule from the registers just loaded (park / pmag_k are free until
        // the sweep): a few barriers instead of a serial, uncoalesced row-sum pass over global memory
        const double nrm_part = (branch == FROB_BRANCH_AUTO && pass < 2) ? gj128_norm_inf(a, n, sm.gs.park, sm.sw.pmag_k) : 0.0;
        gj128_sweep(a, n, sm.sw, sm.gs, pmax, pmin);
        const int inf = sweep_info<double, N>(sm.sw, n, pmax);
        if (pass == 2) {
            inf_m = inf;
            gj128_store(a, sm.sw, S, SS);
            break;
        }
        if (pass == 0) {
            inf_x = inf;
            gj128_store(a, sm.sw, S, SS);
            B128_TL(1);
            if (branch == FROB_BRANCH_AUTO) {
                ka = inf_x ? INFINITY : nrm_part * gj128_norm_inf(a, n, sm.gs.park, sm.sw.pmag_k);
                if (inf_x != 0 || !(ka <= kappa_switch(n))) {
                    __syncthreads();
                    pass = 1;
                    continue;
                }
            }
        } else {
            const int inf_b = inf;
            const double kb = inf_b ? INFINITY : nrm_part * gj128_norm_inf(a, n, sm.gs.park, sm.sw.pmag_k);
            if (inf_b == 0 && (inf_x != 0 || kb < ka)) {
                use = 2;
                inf_x = 0;
                __syncthreads();
                gj128_store(a, sm.sw, S, SS);
            } else if (inf_b != 0 && inf_x != 0) {
                inf_x = -1;
            }
        }
        __syncthreads();
        // X = part use-1, Y = sgn * part 2-use (S2: Y = -A)
        const int xp = use - 1, yp = 2 - use;
        // sgn * v as a sign-bit flip (integer pipe, not the FP64 pipe the DMMAs issue to); same bits
        const unsigned long long sbit = (use == 1) ? 0ull : 0x8000000000000000ull;
        auto Yv = [&](int i, int j) {
            return (i < n && j < n) ? __longlong_as_double(__double_as_longlong(zpart(Zd, n, yp, i, j)) ^ sbit) : 0.0;
        };
        double acc0[WT<N>::MT][WT<N>::NT][2], acc1[WT<N>::MT][WT<N>::NT][2];
        B128_TL(2);
        // a3: C = X^{-1} Y (both 64-row halves in registers, Y staged), then C -> S (X^{-1} is done) and -> Cg
        cta_mma2_staged<false>(Yv, [&](int r, int k) { return S[r * SS + k]; }, sm.slab, acc0, acc1);
        __syncthreads();
        auto put_c = [&](int i, int j, double v) {
            S[i * SS + j] = v;  // zero in the padding (Y is)
            if (i < n && j < n) Cg[i * n + j] = v;
        };
        cta_mma_foreach<N>(acc0, put_c, 0);
        cta_mma_foreach<N>(acc1, put_c, 64);
        __syncthreads();
        B128_TL(3);
        // a4: M = X + Y C with C from shared memory (Y staged) -> S
        // (the accumulators start from X: its reads overlap the first slab's instead of the epilogue)
        cta_mma2_staged<true>(Yv, [&](int k, int c) { return S[k * SS + c]; }, sm.slab, acc0, acc1,
                              [&](int i, int j) { return (i < n && j < n) ? zpart(Zd, n, xp, i, j) : 0.0; });
        __syncthreads();
        auto put_m = [&](int i, int j, double v) { S[i * SS + j] = v; };  // 0 in the padding (X, Y are)
        cta_mma_foreach<N>(acc0, put_m, 0);
        cta_mma_foreach<N>(acc1, put_m, 64);
        __syncthreads();
        B128_TL(4);
        pass = 2;
    }
    __syncthreads();
    B128_TL(5);
    // a6/a7: Im = -C Re (C staged from the output buffer), interleaved store once every warp has read C
    {
        double acc0[WT<N>::MT][WT<N>::NT][2], acc1[WT<N>::MT][WT<N>::NT][2];
        const bool s1 = (use == 1);
        auto out = [&](int i, int j, double v) {
            if (i < n && j < n) {
                const double re = S[i * SS + j];
                Xb[i * n + j] = s1 ? make_double2(re, -v) : make_double2(-v, -re);
            }
        };
        cta_mma2_staged<true>([&](int r, int k) { return (r < n && k < n) ? Cg[r * n + k] : 0.0; },
                              [&](int k, int c) { return S[k * SS + c]; }, sm.slab, acc0, acc1);
        cta_mma_foreach<N>(acc0, out, 0);
        cta_mma_foreach<N>(acc1, out, 64);
    }
    B128_TL(6);
    if (tid == 0) {
        info[b] = (inf_x < 0) ? 1 : (inf_x ? inf_x : inf_m);
        if (bused) bused[b] = (inf_x < 0) ? 0 : (unsigned char)use;
    }
}

// ----------------------------------------------------------------- complex-LU comparator
// Complex Gauss-Jordan sweep with partial pivoting on |re|+|im| (same pivots as complex
// LU with partial pivoting); inverse written straight to the output.
template <int N>
struct ZSmem {
    double2 buf[N * BCfg<N>::S];
    SweepShared1<double2, N> sw;
};

template <int N>
__global__ void __launch_bounds__(BCfg<N>::THREADS)
zinv_batched_kernel(const double2 *__restrict__ Z, long long sZ, double2 *__restrict__ X, long long sX,
                    int n, int *__restrict__ info) {
    using C = BCfg<N>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ZSmem<N> &sm = *reinterpret_cast<ZSmem<N> *>(smem_raw);
    const int tid = threadIdx.x;
    const long long b = blockIdx.x;
    const double2 *Zb = Z + b * sZ;
    double2 *Xb = X + b * sX;
    for (int idx = tid; idx < N * N; idx += C::THREADS) {
        const int i = idx / N, j = idx - i * N;
        sm.buf[i * C::S + j] = (i < n && j < n) ? Zb[i * n + j] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    double2 a[4][4];
    double pmax, pmin;
    load_blocks<double2, N>(a, sm.buf, n);
    gj_sweep_1bar<double2, N, 4, 4>(a, n, sm.sw, pmax, pmin);
    const int inf = sweep_info<double2, N>(sm.sw, n, pmax);
    sweep_store<double2, N, 4, 4>(a, sm.sw, sm.buf, C::S);
    __syncthreads();
    for (int idx = tid; idx < n * n; idx += C::THREADS) {
        const int i = idx / n, j = idx - i * n;
        Xb[i * n + j] = sm.buf[i * C::S + j];
    }
    if (tid == 0) info[b] = inf;
}


// ----------------------------------------------------------------- complex GJ, 64 < n <= 128
// A complex 128 x 128 matrix (256 KB) fits neither one SM's registers nor its shared memory, so
// the comparator runs each matrix on a CLUSTER of two 512-thread CTAs: CTA c holds rows
// [64c, 64c + 64) in registers (4 x 4 complex blocks per thread, as the one-CTA kernels).  Per
// Gauss-Jordan step: candidates of column k, CTA argmax; each CTA pushes its candidate (key,
// row) into both CTAs' slots with st.async + mbarrier complete_tx and both take the same pivot;
// the pivot row's owner scales it and pushes it into the other CTA the same way (the owner goes
// on at once, the other waits on its row barrier); uniform exchange-form update.  One-way
// pushes only: no cluster barrier inside the sweep.
struct ZC128Smem {
    double2 colk[2][128];
    double2 rowp[2][128];
    unsigned long long candk[2][16];
    int candi[2][16];
    uint4 xc[2][2];  // [parity][sender]: {key lo, key hi, row, 0}
    unsigned long long cbar[2], rbar;
    int pivrow[128];
    int pos[128];
    double pmag_k[128];
};
FROB_DEV void zst_async16(unsigned raddr, const uint4 v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     raddr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
                 : "memory");
}
FROB_DEV void zmbar_expect(unsigned addr, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(tx) : "memory");
}

__global__ void __launch_bounds__(512, 1)
zinv_batched128c_kernel(const double2 *__restrict__ Z, long long sZ, double2 *__restrict__ X, long long sX,
                        int n, int *__restrict__ info) {
    constexpr int N = 128, BR = 4, BC = 4, CT = N / BC;  // 32 column-threads x 16 row-threads
    __shared__ __align__(16) ZC128Smem sm;
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const long long b = blockIdx.x >> 1;
    const double2 *Zb = Z + b * sZ;
    double2 *Xb = X + b * sX;
    const int ti = tid / CT, tj = tid % CT;
    const int rb = (int)rank * 64;        // first global row of this CTA
    const int r0 = rb + ti * BR, c0 = tj * BC;
    const unsigned other = rank ^ 1u;
    double2 a[BR][BC];
#pragma unroll
    for (int q = 0; q < BR; ++q)
#pragma unroll
        for (int c = 0; c < BC; ++c) {
            const int i = r0 + q, j = c0 + c;
            a[q][c] = (i < n && j < n) ? Zb[(long long)i * n + j] : make_double2(i == j ? 1.0 : 0.0, 0.0);
        }
    if (tid == 0) {
        mbar_init(smem_u32(&sm.cbar[0]), 1u);
        mbar_init(smem_u32(&sm.cbar[1]), 1u);
        mbar_init(smem_u32(&sm.rbar), 1u);
        mbar_init_fence();
    }
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers exist before any push
    if (tid == 0) {
        zmbar_expect(smem_u32(&sm.cbar[0]), 32u);
        if (n > 1) zmbar_expect(smem_u32(&sm.cbar[1]), 32u);
        zmbar_expect(smem_u32(&sm.rbar), (unsigned)(N * 16));
    }
    int rphase = 0;        // row-barrier phases completed (steps at which this CTA did not own the pivot)
    unsigned used = 0;     // this thread's rows r0 .. r0+3 already pivots (no shared flags: no barrier needed)
    auto step = [&](const int k, auto KCc) {
        constexpr int KC = decltype(KCc)::value;
        const int par = k & 1;
        const bool owner = (tj == k / BC);
        // (1) candidates of column k among this CTA's unused rows; the CTA argmax is pushed into
        // both CTAs' slots
        if (owner) {
            unsigned long long bk = 0;
            int bi = INT_MAX;
#pragma unroll
            for (int q = 0; q < BR; ++q) {
                const int r = r0 + q;
                const double2 v = a[q][KC];
                sm.colk[par][r] = v;
                if (r < n && !((used >> q) & 1u)) {
                    const unsigned long long kk = pkey_bits(v);
                    if (kk > bk) { bk = kk; bi = r; }
                }
            }
            sm.candk[par][ti] = bk;
            sm.candi[par][ti] = bi;
        }
        __syncthreads();
        if (tid < 32) {
            const ArgMaxK m = warp_argmax_key(lane < 16 ? sm.candk[par][lane] : 0ull, lane < 16 ? sm.candi[par][lane] : INT_MAX);
            if (lane < 2) {
                const uint4 v = make_uint4((unsigned)m.k, (unsigned)(m.k >> 32), (unsigned)m.i, 0u);
                const unsigned tgt = (unsigned)lane;  // lane 0 -> CTA 0, lane 1 -> CTA 1
                zst_async16(mapa_u32(smem_u32(&sm.xc[par][rank]), tgt), v, mapa_u32(smem_u32(&sm.cbar[par]), tgt));
            }
        }
        mbar_wait_parity(smem_u32(&sm.cbar[par]), (unsigned)((k >> 1) & 1));
        // (2) the cluster's pivot (max key, then the smallest row)
        const uint4 x0 = sm.xc[par][0], x1 = sm.xc[par][1];
        const unsigned long long k0 = ((unsigned long long)x0.y << 32) | x0.x, k1 = ((unsigned long long)x1.y << 32) | x1.x;
        const int i0 = (int)x0.z, i1 = (int)x1.z;
        const bool w1 = (k1 > k0 || (k1 == k0 && i1 < i0));
        const int p = w1 ? i1 : i0;
        const unsigned long long pk = w1 ? k1 : k0;
        const unsigned prank = (unsigned)(p >> 6);
        __syncwarp();
        if (tid == 0) {
            if (k + 2 < n) zmbar_expect(smem_u32(&sm.cbar[par]), 32u);
            sm.pivrow[k] = p;
            sm.pmag_k[k] = __longlong_as_double((long long)(pk - 1ull));  // key = bits(|re|+|im|) + 1
        }
        if (p >= r0 && p < r0 + BR) used |= 1u << (p - r0);
        if (prank == rank) {
            // (3a) the owner scales the pivot row into its own rowp and pushes it to the other CTA
            if (ti == (p - rb) / BR) {
                const int q = (p - rb) % BR;
                const double2 piv = sm.colk[par][p];
                const double2 ip = is_zero(piv) ? zero_of(double2()) : recip(piv);
                const unsigned dst = mapa_u32(smem_u32(&sm.rowp[par][c0]), other);
                const unsigned rb_other = mapa_u32(smem_u32(&sm.rbar), other);
#pragma unroll
                for (int c = 0; c < BC; ++c) {
                    double2 v = a[0][c];
#pragma unroll
                    for (int qq = 1; qq < BR; ++qq)
                        if (q == qq) v = a[qq][c];
                    const double2 y = (owner && c == KC) ? ip : mul(v, ip);
                    sm.rowp[par][c0 + c] = y;
                    zst_async16(dst + c * 16u, make_uint4(__double2loint(y.x), __double2hiint(y.x), __double2loint(y.y),
                                                         __double2hiint(y.y)), rb_other);
                }
            }
            __syncthreads();
        } else {
            // (3b) the other CTA waits for the pushed pivot row
            mbar_wait_parity(smem_u32(&sm.rbar), (unsigned)(rphase & 1));
            ++rphase;
            __syncwarp();
            if (tid == 0) zmbar_expect(smem_u32(&sm.rbar), (unsigned)(N * 16));
        }
        // (4) uniform exchange-form update (the owner of column k zeroes it first; the pivot row
        // is written last)
        double2 rp[BC], ck[BR];
#pragma unroll
        for (int c = 0; c < BC; ++c) rp[c] = sm.rowp[par][c0 + c];
#pragma unroll
        for (int q = 0; q < BR; ++q) ck[q] = sm.colk[par][r0 + q];
        if (owner) {
#pragma unroll
            for (int q = 0; q < BR; ++q) a[q][KC] = zero_of(double2());
        }
#pragma unroll
        for (int q = 0; q < BR; ++q)
#pragma unroll
            for (int c = 0; c < BC; ++c) a[q][c] = msub(a[q][c], ck[q], rp[c]);
        if (prank == rank && ti == (p - rb) / BR) {
#pragma unroll
            for (int q = 0; q < BR; ++q)
                if (r0 + q == p) {
#pragma unroll
                    for (int c = 0; c < BC; ++c) a[q][c] = rp[c];
                }
        }
    };
    for (int kb = 0; kb * BC < n; ++kb) {
        bstatic_for<BC>([&](auto KCc) {
            constexpr int KC = decltype(KCc)::value;
            const int k = kb * BC + KC;
            if (k < n) step(k, KCc);
        });
    }
    __syncthreads();
    double pmax, pmin;
    sweep_finish<double2, N, 512>(sm, n, pmax, pmin);
    const int inf = sweep_info<double2, N>(sm, n, pmax);
    // exchange form -> inverse: X[pos[i]][pivrow[j]] = a(i, j)
#pragma unroll
    for (int q = 0; q < BR; ++q) {
        const int i = r0 + q;
        if (i >= n) continue;
        const int orow = sm.pos[i];
#pragma unroll
        for (int c = 0; c < BC; ++c) {
            const int j = c0 + c;
            if (j < n) Xb[(long long)orow * n + sm.pivrow[j]] = a[q][c];
        }
    }
    if (tid == 0 && rank == 0) info[b] = inf;
    cluster_sync_all();  // every push has landed (all were waited for) before either CTA leaves
}

template <typename K>
static cudaError_t set_smem(K kern, size_t bytes) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

}  // namespace frob

using namespace frob;

extern "C" {

size_t frob_inv_batched_workspace_bytes(int n, int batch) { (void)n; (void)batch; return 0; }
size_t zinv_lu_batched_workspace_bytes(int n, int batch) { (void)n; (void)batch; return 0; }

frob_status frob_inv_batched(int n, int batch, const double *Z, long long strideZ, double *X,
                             long long strideX, int branch, int *d_info, unsigned char *d_branch_used,
                             void *ws, size_t ws_bytes, void *stream) {
    (void)ws; (void)ws_bytes;
    if (n < 1 || n > 128 || batch < 0 || !d_info || strideZ < (long long)n * n || strideX < (long long)n * n ||
        branch < 0 || branch > 2)
        return FROB_ERR_INVALID_ARG;
    if (batch == 0) return FROB_OK;
    if (!Z || !X) return FROB_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const double2 *Zc = reinterpret_cast<const double2 *>(Z);
    double2 *Xc = reinterpret_cast<double2 *>(X);
    cudaError_t e;
    if (n <= 32) {
        const size_t smem = sizeof(W32Smem) * W32_WARPS;
        if ((e = set_smem(frob_batched32w_kernel, smem)) != cudaSuccess) return FROB_ERR_CUDA;
        count_launch();
        ProfScope ps("frob_batched32w", s, 10.0 * n * (double)n * n * batch);
        frob_batched32w_kernel<<<(batch + W32_WARPS - 1) / W32_WARPS, 32 * W32_WARPS, smem, s>>>(
            Zc, strideZ, Xc, strideX, n, batch, branch, d_info, d_branch_used);
    } else if (n <= 64) {
        const size_t smem = sizeof(FrobSmem<64>);
        if ((e = set_smem(frob_batched_kernel<64>, smem)) != cudaSuccess) return FROB_ERR_CUDA;
        count_launch();
        ProfScope ps("frob_batched<64>", s, 10.0 * n * (double)n * n * batch);
        frob_batched_kernel<64><<<batch, BCfg<64>::THREADS, smem, s>>>(Zc, strideZ, Xc, strideX, n, branch,
                                                                       d_info, d_branch_used);
    } else {
        const size_t smem = sizeof(Frob128Smem);
        if ((e = set_smem(frob_batched128_kernel, smem)) != cudaSuccess) return FROB_ERR_CUDA;
        count_launch();
        ProfScope ps("frob_batched128", s, 10.0 * n * (double)n * n * batch);
        frob_batched128_kernel<<<batch, G8_T, smem, s>>>(Zc, strideZ, Xc, strideX, n, branch, d_info,
                                                         d_branch_used);
    }
    return cudaGetLastError() == cudaSuccess ? FROB_OK : FROB_ERR_CUDA;
}

frob_status zinv_lu_batched(int n, int batch, const double *Z, long long strideZ, double *X,
                            long long strideX, int *d_info, void *ws, size_t ws_bytes, void *stream) {
    (void)ws; (void)ws_bytes;
    if (n < 1 || n > 128 || batch < 0 || !d_info || strideZ < (long long)n * n || strideX < (long long)n * n)
        return FROB_ERR_INVALID_ARG;
    if (batch == 0) return FROB_OK;
    if (!Z || !X) return FROB_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const double2 *Zc = reinterpret_cast<const double2 *>(Z);
    double2 *Xc = reinterpret_cast<double2 *>(X);
    cudaError_t e;
    if (n > 64) {
        cudaLaunchConfig_t cfg{};
        cudaLaunchAttribute attr[1];
        cfg.gridDim = dim3(2u * (unsigned)batch);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = s;
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        count_launch();
        ProfScope ps("zinv_batched128c", s, 8.0 * n * (double)n * n * batch);
        if (cudaLaunchKernelEx(&cfg, zinv_batched128c_kernel, Zc, strideZ, Xc, strideX, n, d_info) != cudaSuccess)
            return FROB_ERR_CUDA;
        return cudaGetLastError() == cudaSuccess ? FROB_OK : FROB_ERR_CUDA;
    }
    if (n <= 32) {
        const size_t smem = sizeof(Z32Smem) * W32_WARPS;
        if ((e = set_smem(zinv_batched32w_kernel, smem)) != cudaSuccess) return FROB_ERR_CUDA;
        count_launch();
        ProfScope ps("zinv_batched32w", s, 8.0 * n * (double)n * n * batch);
        zinv_batched32w_kernel<<<(batch + W32_WARPS - 1) / W32_WARPS, 32 * W32_WARPS, smem, s>>>(
            Zc, strideZ, Xc, strideX, n, batch, d_info);
    } else {
        const size_t smem = sizeof(ZSmem<64>);
        if ((e = set_smem(zinv_batched_kernel<64>, smem)) != cudaSuccess) return FROB_ERR_CUDA;
        count_launch();
        ProfScope ps("zinv_batched<64>", s, 8.0 * n * (double)n * n * batch);
        zinv_batched_kernel<64><<<batch, BCfg<64>::THREADS, smem, s>>>(Zc, strideZ, Xc, strideX, n, d_info);
    }
    return cudaGetLastError() == cudaSuccess ? FROB_OK : FROB_ERR_CUDA;
}

}  // extern "C"
