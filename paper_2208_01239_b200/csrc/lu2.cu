// lu2.cu -- latency-oriented LU with partial pivoting for the inversion path
// (Alg 3 line 1), orders n <= LU2_MAX_N, real and complex.
//
// One step per PW-column panel, two kernels per step, PDL-chained:
//   lu_panel2_kernel   m x PW panel in REGISTERS of one 512-thread CTA (R rows per thread);
//                      per column: speculative candidate of the next column computed while
//                      the current rank-1 update is still in flight, one __syncthreads,
//                      block argmax by 16-lane REDUX; rows never move inside the panel and
//                      are written to their final positions at the end (in place).
//   lu_update2_kernel  the rest of the step, fused: row interchanges of the panel (as a
//                      gather), U12 = L11^{-1} A12 and A22 -= L21 U12, over the whole
//                      trailing matrix, PING-PONG between two buffers (reads B[k%2], writes
//                      B[(k+1)%2]) so the gather needs no ordering between tiles.
// Row interchanges are never applied to the columns left of a panel.  Each step records a
// snapshot of the position of every original row; lu_assemble2_kernel finally writes U
// (upper, zeros below) and L (unit lower, zeros above) in final row order, reading each L
// column block through its snapshot -- the split form inv_from_ul consumes directly.
#include <climits>
#include <cstdlib>
#include <cstdio>
#include <utility>
#include <algorithm>
#include <mutex>
#include "lu.cuh"
#include "tma.cuh"

namespace frob {

// Kernel timeline tracer (build with -DFROB_TL; tools/lu2_timeline.py): per (kernel kind, step)
// the earliest CTA start (after its dependency wait) and the latest CTA end, %globaltimer ns.
#ifdef FROB_TL
__device__ unsigned long long g_tl_start[5][1024], g_tl_end[5][1024];
__device__ int g_tl_call;  // LU calls since the last reset (slot = call * 128 + step)
FROB_DEV unsigned long long tl_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ long long g_nx_tr[2][8];
#define NXT(i) do { if (gridDim.x == 1 && blockIdx.y <= 1 && threadIdx.x == 0 && k0 == 320) g_nx_tr[blockIdx.y][i] = clock64(); } while (0)
#define TL_SLOT(step) ((((g_tl_call - 1) & 7) * 128 + (step)) & 1023)
#define TL_BEGIN(kind, step) do { if (threadIdx.x == 0) atomicMin(&g_tl_start[kind][TL_SLOT(step)], tl_now()); } while (0)
#define TL_END(kind, step) do { if (threadIdx.x == 0) atomicMax(&g_tl_end[kind][TL_SLOT(step)], tl_now()); } while (0)
#else
#define TL_BEGIN(kind, step) do { } while (0)
#define TL_END(kind, step) do { } while (0)
#define NXT(i) do { } while (0)
#endif

constexpr int P2_T = 512;
constexpr int P2_WARPS = P2_T / 32;
constexpr int P2_STG = 18;  // staging row stride in doubles (16 + 2: 16-byte aligned, conflict free)

// panel width of one step: two 128-byte row halves (32 real / 16 complex columns)

// mv2 layout (ints): [0] = number of moves, [1, 1 + MV2_MAX) dst, [1 + MV2_MAX, 1 + 2 MV2_MAX) src
constexpr int MV2_MAX = 64;
constexpr int MV2_INTS = 1 + 2 * MV2_MAX;

template <typename F, int... J>
FROB_DEV void static_for_impl(F &&f, std::integer_sequence<int, J...>) {
    (f(std::integral_constant<int, J>{}), ...);
}
template <int N, typename F>
FROB_DEV void static_for(F &&f) {
    static_for_impl(f, std::make_integer_sequence<int, N>{});
}

#ifdef FROB_P2_TRACE
__device__ long long g_p2_trace[64];
#define P2T(i) do { if (threadIdx.x == 0) g_p2_trace[i] = clock64(); } while (0)
#define P2TJ(j, i) do { if ((j) == 5) P2T(i); } while (0)
#else
#define P2T(i) do { } while (0)
#define P2TJ(j, i) do { } while (0)
#endif

FROB_DEV double rcp_spec(double x) { return (x == 0.0) ? 0.0 : frcp(x); }
FROB_DEV double2 rcp_spec(double2 x) { return is_zero(x) ? make_double2(0.0, 0.0) : recip(x); }

template <typename T, int PW>
FROB_DEV void st_row_smem(T *dst, const T (&r)[PW]) {
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int c = 0; c < PW; c += 2) *reinterpret_cast<double2 *>(dst + c) = make_double2(r[c], r[c + 1]);
    } else {
#pragma unroll
        for (int c = 0; c < PW; ++c) dst[c] = r[c];
    }
}
template <typename T, int PW>
FROB_DEV void ld_row_smem(T (&u)[PW], const T *src) {
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

// ---------------------------------------------------------------------------------------
// Fused look-ahead (lu2_factor): a panel kernel of step k > 0 receives its columns NOT yet
// updated by step k-1 and applies that update itself, instead of a separate kernel on the
// critical path between two panels: for its rows r (positions after step k-1),
//   a[r][c] = Bp[src(r)][c] - sum_q Lp[r][q] U12p[q][c],   c in this panel's columns,
// src = step k-1's row moves (gather), Lp = step k-1's multipliers (Bp, its panel columns),
// U12p = L11p^{-1} Xp from step k-1's pivot rows (every CTA solves it; the writer also stores it
// as the U rows of step k-1 for these columns into B).  Half 0 lands in registers, half 1 in the
// staging buffer, exactly where the TMA path would have put them.
template <typename T, int PWT>
struct PreSmem {
    int mdst[MV2_MAX], msrc[MV2_MAX];
    int nm;
    __align__(16) T L11[PWT][PWT + 16 / (int)sizeof(T)];
    __align__(16) T U[PWT][PWT + 16 / (int)sizeof(T)];
};

template <typename T, int PH, bool TWO>
FROB_DEV void pre_update(const T *__restrict__ Bp, const int *__restrict__ mvp, int kp0, T *__restrict__ B,
                         long long ld, int n, int k0, int w, int g, bool writer, int lrow, T (&a)[PH],
                         unsigned char *stgb, unsigned char *d0s, PreSmem<T, (TWO ? 2 * PH : PH)> &sm) {
    constexpr int PWT = TWO ? 2 * PH : PH;
    constexpr int E = 16 / (int)sizeof(T);
    const int tid = threadIdx.x;
    const int m = n - k0;
    if (tid < MV2_MAX) {
        const int nm = mvp[0];
        if (tid == 0) sm.nm = nm;
        sm.mdst[tid] = tid < nm ? mvp[1 + tid] : -1;
        sm.msrc[tid] = tid < nm ? mvp[1 + MV2_MAX + tid] : -1;
    }
    for (int idx = tid; idx < PWT * (PWT / E); idx += P2_T) {
        const int i = idx / (PWT / E), e = (idx % (PWT / E)) * E;
        cp_async16(&sm.L11[i][e], Bp + (long long)(kp0 + i) * ld + kp0 + e);
    }
    __syncthreads();
    const int nm = sm.nm;
    for (int idx = tid; idx < PWT * (PWT / E); idx += P2_T) {
        const int i = idx / (PWT / E), e = (idx % (PWT / E)) * E;
        int src = kp0 + i;
        for (int q = 0; q < nm; ++q)
            if (sm.mdst[q] == kp0 + i) src = sm.msrc[q];
        if (e < w) cp_async16(&sm.U[i][e], Bp + (long long)src * ld + k0 + e);  // (w even or ld > n)
    }
    const int r = k0 + g;
    int src = r;
    for (int q = 0; q < nm; ++q)
        if (sm.mdst[q] == r) src = sm.msrc[q];
    // this row's D values (gathered) are requested before the solve, straight into shared memory
    // (half 0 into d0s, half 1 into its staging row): no registers held across the solve
    {
        const T *d = Bp + (long long)src * ld + k0;
#pragma unroll
        for (int h = 0; h < (TWO ? 2 : 1); ++h) {
            unsigned char *base = h ? stgb : d0s;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                unsigned char *dst = base + swz128(lrow, c);
                if (g < m && h * PH + c * E < w) cp_async16(dst, d + h * PH + c * E);
                else *reinterpret_cast<double2 *>(dst) = make_double2(0.0, 0.0);
            }
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // U12p = L11p^{-1} Xp (unit lower forward substitution), one thread per column
    if (tid < PWT) {
        T x[PWT];
#pragma unroll
        for (int i = 0; i < PWT; ++i) x[i] = sm.U[i][tid];
#pragma unroll
        for (int q = 0; q < PWT; ++q)
#pragma unroll
            for (int i = q + 1; i < PWT; ++i) x[i] = msub(x[i], sm.L11[i][q], x[q]);
#pragma unroll
        for (int i = 0; i < PWT; ++i) sm.U[i][tid] = x[i];
        if (writer && tid < w) {
#pragma unroll
            for (int i = 0; i < PWT; ++i) B[(long long)(kp0 + i) * ld + k0 + tid] = x[i];
        }
    }
    __syncthreads();
    // this row's multipliers of the previous step (one vector load batch), then each half:
    // x = D - L U12p over the half's columns, from and back to shared memory / registers
    T lrow_v[PWT];
    if (g < m) {
        const T *lr = Bp + (long long)r * ld + kp0;
        if constexpr (sizeof(T) == 8) {
#pragma unroll
            for (int q = 0; q < PWT; q += 2) {
                const double2 v = *reinterpret_cast<const double2 *>(lr + q);
                lrow_v[q] = v.x;
                lrow_v[q + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int q = 0; q < PWT; ++q) lrow_v[q] = lr[q];
        }
    }
    auto half = [&](unsigned char *base, int h, T (&x)[PH]) {
        double t[16];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const double2 v = *reinterpret_cast<const double2 *>(base + swz128(lrow, c));
            t[2 * c] = v.x;
            t[2 * c + 1] = v.y;
        }
#pragma unroll
        for (int c = 0; c < PH; ++c) {
            if constexpr (sizeof(T) == 8) x[c] = t[c];
            else x[c] = make_double2(t[2 * c], t[2 * c + 1]);
        }
        if (g < m) {
#pragma unroll
            for (int q = 0; q < PWT; ++q) {
#pragma unroll
                for (int c = 0; c < PH; ++c) x[c] = msub(x[c], lrow_v[q], sm.U[q][h * PH + c]);
            }
        }
#pragma unroll
        for (int c = 0; c < PH; ++c)
            if (h * PH + c >= w) x[c] = zero_of(T());
    };
    if constexpr (TWO) {
        T x1[PH];
        half(stgb, 1, x1);
        const double *xd = reinterpret_cast<const double *>(x1);
#pragma unroll
        for (int c = 0; c < 8; ++c)
            *reinterpret_cast<double2 *>(stgb + swz128(lrow, c)) = make_double2(xd[2 * c], xd[2 * c + 1]);
    }
    half(d0s, 0, a);
}

// Panel of step k0: rows [k0, n) x columns [k0, k0 + w) of B (ld), w <= 2 * PH, factored in
// place as two PH-column halves (PH = 16 real / 8 complex: 128-byte row halves).  Thread t owns
// relative rows t + q * P2_T (q < R).  Half 0 is TMA-loaded and moved to registers; half 1 is
// TMA-loaded into the staging buffer while half 0 is factored, then receives half 0's rank-PH
// update there (U12 = L11^{-1} X by PH threads), and the two halves swap places: half 1 goes to
// registers, half 0's factored rows wait in the staging buffer.  Rows never move inside the
// panel; both halves are written to their final positions at the end.  mv2 receives the row
// moves of the step, diag[k0 + j] the pivot values.
template <typename T, int PH, int R, bool TWO>
__global__ void __launch_bounds__(P2_T, 1)
lu_panel2_kernel(const __grid_constant__ CUtensorMap tmap, T *__restrict__ B, long long ld, int n, int k0, int w,
                 int *__restrict__ mv2, T *__restrict__ diag, const T *__restrict__ Bp, const int *__restrict__ mvp,
                 int kp0) {
    extern __shared__ __align__(1024) unsigned char stgb[];  // R * P2_T rows x 128 B, 128B-swizzled (TMA)
    __shared__ __align__(8) unsigned long long tbar;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&tbar), 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();
    pdl_trigger();  // after the wait: the BULK update launched behind this panel relies on it
    TL_BEGIN(0, k0 / Panel2W<T>::PW);
    P2T(0);
    constexpr int PW = 2 * PH;                     // panel width in elements
    __shared__ unsigned long long ck[2][P2_WARPS];
    __shared__ int ci[2][P2_WARPS];
    __shared__ __align__(16) T wrow[2][P2_WARPS][PH];
    __shared__ int pivrow[PW];
    __shared__ int vac[PW];
    __shared__ unsigned evm_s;
    __shared__ T L11s[PH][PH + 1];
    __shared__ T U12s[PH][PH + 1];
    __shared__ int sdst[R * P2_T];

    constexpr int RW = PH * (int)(sizeof(T) / 8);  // doubles per row half (16)
    static_assert(RW == 16, "panel row halves are 128 bytes");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = n - k0;
    const int E = (int)(sizeof(T) / 8);
    const int nbox = (m + 255) / 256;
    const bool two = TWO && w > PH;  // TWO = false compiles the second half out (complex: spills)
    auto tma_half = [&](int h, unsigned parity_unused) {
        (void)parity_unused;
        mbar_arrive_expect_tx(smem_u32(&tbar), (unsigned)(nbox * 256 * 128));
        for (int b = 0; b < nbox; ++b)
            tma_load_2d(smem_u32(stgb + b * 256 * 128), &tmap, (k0 + h * PH) * E, k0 + 256 * b, smem_u32(&tbar));
    };
    auto row_from_stg = [&](int r, T (&dst)[PH]) {
        double t[16];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const double2 v = *reinterpret_cast<const double2 *>(stgb + swz128(r, c));
            t[2 * c] = v.x;
            t[2 * c + 1] = v.y;
        }
#pragma unroll
        for (int c = 0; c < PH; ++c) {
            if constexpr (sizeof(T) == 8) dst[c] = t[c];
            else dst[c] = make_double2(t[2 * c], t[2 * c + 1]);
        }
    };
    auto row_to_stg = [&](int r, const T (&src)[PH]) {
        const double *rd = reinterpret_cast<const double *>(src);
#pragma unroll
        for (int c = 0; c < 8; ++c)
            *reinterpret_cast<double2 *>(stgb + swz128(r, c)) = make_double2(rd[2 * c], rd[2 * c + 1]);
    };

    T a[R][PH];
    int grow[R], pst[R];
    unsigned live = 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        grow[q] = q * P2_T + tid;
        pst[q] = -1;
        if (grow[q] < m) live |= 1u << q;
    }
    const bool fused = R == 1 && Bp != nullptr;
    __shared__ PreSmem<T, (TWO ? 2 * PH : PH)> psm;
    if (fused) {
        // ---- fused look-ahead: this panel applies the previous step's update to its columns
        if constexpr (R == 1)
            pre_update<T, PH, TWO>(Bp, mvp, kp0, B, ld, n, k0, w, tid, true, tid, a[0], stgb, stgb + P2_T * 128, psm);
        __syncthreads();
    } else {
        // ---- half 0: TMA load -> registers; half 1 then streams into the staging buffer
        if (tid == 0) tma_half(0, 0u);
        __syncthreads();
        mbar_wait_cta(smem_u32(&tbar), 0u);
#pragma unroll
        for (int q = 0; q < R; ++q) row_from_stg(grow[q], a[q]);
        __syncthreads();  // every thread has read its half-0 rows: the staging buffer is free
        if (two && tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_half(1, 1u);
        }
    }
    P2T(1);

    auto candidate = [&](auto Jc, unsigned long long &bk, int &bi, int &bq) {
        constexpr int J = decltype(Jc)::value;
        bk = 0ull;
        bi = INT_MAX;
        bq = 0;
#pragma unroll
        for (int q = 0; q < R; ++q)
            if ((live >> q) & 1u) {
                const unsigned long long kq = pkey_bits(a[q][J]);
                if (kq > bk) { bk = kq; bi = grow[q]; bq = q; }
            }
    };
    auto publish_first = [&]() {
        unsigned long long bk; int bi, bq;
        candidate(std::integral_constant<int, 0>{}, bk, bi, bq);
        const ArgMaxK wa = warp_argmax_key(bk, bi);
        if (lane == 0) { ck[0][warp] = wa.k; ci[0][warp] = wa.i; }
        if (bi == wa.i && wa.k != 0ull) {
#pragma unroll
            for (int q = 0; q < R; ++q)
                if (q == bq) st_row_smem<T, PH>(wrow[0][warp], a[q]);
        }
    };

    // ---- column loop over one half (fully unrolled: static register indices), JO = offset of
    // the half.  Software-pipelined: the rank-1 update of pivot J-1 on columns >= J+1 is
    // deferred into iteration J, right after the barrier; only column J+1 (needed for the
    // candidate keys) and the published candidate row are updated eagerly.
    T u[PH];          // pivot row of the current (then previous) column
    T lp[R];          // multipliers of the pending (deferred) update
    unsigned pact = 0;  // rows with a pending update
    auto run_half = [&](const int JO, const int wh) {
#pragma unroll
        for (int c = 0; c < PH; ++c) u[c] = zero_of(T());
#pragma unroll
        for (int q = 0; q < R; ++q) lp[q] = zero_of(T());
        pact = 0;
        auto column = [&](auto Jc) {
            constexpr int J = decltype(Jc)::value;
            constexpr int s = J & 1;
            P2TJ(J, 40);
            __syncthreads();
            P2TJ(J, 41);
            // (a) deferred update of pivot J-1 (columns >= J+1)
#pragma unroll
            for (int q = 0; q < R; ++q)
                if ((pact >> q) & 1u) {
#pragma unroll
                    for (int c = J + 1; c < PH; ++c) a[q][c] = msub(a[q][c], lp[q], u[c]);
                }
            // (b) block argmax over the warp candidates, pivot row + its reciprocal
            const ArgMaxK ba = warp_argmax_key(lane < P2_WARPS ? ck[s][lane] : 0ull,
                                               lane < P2_WARPS ? ci[s][lane] : INT_MAX);
            const int gi = ba.i;
            const unsigned ww = ((unsigned)gi & (unsigned)(P2_T - 1)) >> 5;
            ld_row_smem<T, PH>(u, wrow[s][ww]);
            const T rc = rcp_spec(u[J]);
            P2TJ(J, 42);
            if (tid == 0) {
                pivrow[JO + J] = gi;
                diag[k0 + JO + J] = u[J];
            }
            // (c) multipliers, eager update of column J+1
            T l[R];
            pact = 0;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const bool lv = (live >> q) & 1u;
                const bool isp = lv && grow[q] == gi;
                if (isp) { live &= ~(1u << q); pst[q] = JO + J; }
                const bool act = lv && !isp;
                l[q] = act ? mul(a[q][J], rc) : zero_of(T());
                if (act) {
                    pact |= 1u << q;
                    a[q][J] = l[q];
                    if constexpr (J + 1 < PH) a[q][J + 1] = msub(a[q][J + 1], l[q], u[J + 1]);
                }
                lp[q] = l[q];
            }
            P2TJ(J, 43);
            if constexpr (J + 1 < PH) {
                if (J + 1 < wh) {
                    // (e) candidate of column J+1, warp argmax
                    unsigned long long bk; int bi, bq;
                    candidate(std::integral_constant<int, J + 1>{}, bk, bi, bq);
                    const ArgMaxK wa = warp_argmax_key(bk, bi);
                    if (lane == 0) { ck[s ^ 1][warp] = wa.k; ci[s ^ 1][warp] = wa.i; }
                    P2TJ(J, 44);
                    // (f) the warp winner publishes its row updated through pivot J
                    if (bi == wa.i && wa.k != 0ull) {
                        T lw = l[0];
#pragma unroll
                        for (int q = 1; q < R; ++q)
                            if (q == bq) lw = l[q];
                        T *dst = wrow[s ^ 1][warp];
                        auto rowval = [&](const int c) {
                            T v = a[0][c];
#pragma unroll
                            for (int q = 1; q < R; ++q)
                                if (q == bq) v = a[q][c];
                            return (c >= J + 2) ? msub(v, lw, u[c]) : v;
                        };
                        if constexpr (sizeof(T) == 8) {
#pragma unroll
                            for (int c = 0; c < PH; c += 2)
                                *reinterpret_cast<double2 *>(dst + c) = make_double2(rowval(c), rowval(c + 1));
                        } else {
#pragma unroll
                            for (int c = 0; c < PH; ++c) dst[c] = rowval(c);
                        }
                    }
                    P2TJ(J, 45);
                }
            }
            P2T(2 + J);
        };
        static_for<PH>([&](auto Jc) {
            constexpr int Jv = decltype(Jc)::value;
            if (Jv < wh) column(Jc);
        });
    };

    publish_first();
    run_half(0, min(w, PH));
    __syncthreads();

    if constexpr (TWO) if (two) {
        // ---- half 1: U12 = L11^{-1} X from half 0's pivot rows, rank-PH update, swap
        P2T(30);
        if (!fused) mbar_wait_cta(smem_u32(&tbar), 1u);
        P2T(31);
#pragma unroll
        for (int q = 0; q < R; ++q)
            if (pst[q] >= 0) {
                T x[PH];
                row_from_stg(grow[q], x);
#pragma unroll
                for (int c = 0; c < PH; ++c) {
                    L11s[pst[q]][c] = a[q][c];
                    U12s[pst[q]][c] = x[c];
                }
            }
        __syncthreads();
        if (tid < PH) {
            T x[PH];
#pragma unroll
            for (int j = 0; j < PH; ++j) x[j] = U12s[j][tid];
#pragma unroll
            for (int q = 0; q < PH; ++q)
#pragma unroll
                for (int j = q + 1; j < PH; ++j) x[j] = msub(x[j], L11s[j][q], x[q]);
#pragma unroll
            for (int j = 0; j < PH; ++j) U12s[j][tid] = x[j];
        }
        __syncthreads();
        P2T(33);
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int g = grow[q];
            if (g >= m) continue;
            T x[PH];
            row_from_stg(g, x);
            if (pst[q] >= 0) {
#pragma unroll
                for (int c = 0; c < PH; ++c) x[c] = U12s[pst[q]][c];
            } else {
#pragma unroll
                for (int j = 0; j < PH; ++j) {
                    const T lj = a[q][j];
#pragma unroll
                    for (int c = 0; c < PH; ++c) x[c] = msub(x[c], lj, U12s[j][c]);
                }
            }
            row_to_stg(g, a[q]);  // half 0's factored row waits in the staging buffer
#pragma unroll
            for (int c = 0; c < PH; ++c) a[q][c] = x[c];
        }
        __syncthreads();
        P2T(34);
        publish_first();
        run_half(PH, w - PH);
        __syncthreads();
    }
    P2T(20);

    // ---- final positions: pivot j -> j; evicted top rows (< w, not pivots) fill the rows
    // vacated by pivots that came from below (>= w), in pivot order.
    if (warp == 0) {
        const int pj = lane < w ? pivrow[lane] : -1;
        bool rp = false;
        if (lane < w)
            for (int q = 0; q < w; ++q) rp |= (pivrow[q] == lane);
        const unsigned pivmask = __ballot_sync(0xffffffffu, rp);
        const unsigned wmask = (w >= 32) ? 0xffffffffu : ((1u << w) - 1u);
        const unsigned evmask = wmask & ~pivmask;
        const bool isv = lane < w && pj >= w;
        const unsigned vb = __ballot_sync(0xffffffffu, isv);
        if (isv) vac[__popc(vb & ((1u << lane) - 1u))] = pj;
        if (lane == 0) evm_s = evmask;
        __syncwarp();
        // moves (absolute rows): top position j <- pivot row; vacated <- evicted
        const bool moved = lane < w && pj != lane;
        const unsigned mb = __ballot_sync(0xffffffffu, moved);
        const int nm = __popc(mb);
        if (moved) {
            const int q = __popc(mb & ((1u << lane) - 1u));
            mv2[1 + q] = k0 + lane;
            mv2[1 + MV2_MAX + q] = k0 + pj;
        }
        const bool ev = (evmask >> lane) & 1u;
        if (ev) {
            const int q = nm + __popc(evmask & ((1u << lane) - 1u));
            mv2[1 + q] = k0 + vac[__popc(evmask & ((1u << lane) - 1u))];
            mv2[1 + MV2_MAX + q] = k0 + lane;
        }
        if (lane == 0) mv2[0] = nm + __popc(evmask);
    }
    __syncthreads();
    const unsigned evm = evm_s;
    int mydst[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int g = grow[q];
        int dst = g;
        if (pst[q] >= 0) dst = pst[q];
        else if (g < w) dst = vac[__popc(evm & ((1u << g) - 1u))];
        mydst[q] = dst;
        if (g < m) sdst[q * P2_T + tid] = dst;
    }
    __syncthreads();
    // coalesced write-back, 8 threads per 128-byte row half
    const long long ldd = ld * E;
    double *P = reinterpret_cast<double *>(B) + (long long)k0 * ldd + (long long)k0 * E;
    auto write_half = [&](int h, bool by_origin) {
        const int wd = (min(w, (h + 1) * PH) - h * PH) * E;
#pragma unroll 4
        for (int idx = tid; idx < m * 8; idx += P2_T) {
            const int r = idx >> 3, c = idx & 7;
            if (2 * c >= wd) continue;
            const int d = by_origin ? sdst[r] : r;
            const double2 v = *reinterpret_cast<const double2 *>(stgb + swz128(r, c));
            double *out = P + (long long)d * ldd + h * PH * E + 2 * c;
            if (2 * c + 1 < wd) *reinterpret_cast<double2 *>(out) = v;
            else out[0] = v.x;
        }
    };
    if constexpr (TWO) if (two) {
        write_half(0, true);  // half 0 rows sit at their original positions in the staging buffer
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < R; ++q)
        if (grow[q] < m) row_to_stg(mydst[q], a[q]);
    __syncthreads();
    write_half(two ? 1 : 0, false);
    TL_END(0, k0 / Panel2W<T>::PW);
    P2T(21);
}

// ---------------------------------------------------------------------------------------
// Cluster variant of the panel for m > P2_T rows: CS = ceil(m / P2_T) CTAs (a thread-block
// cluster), CTA r owns relative rows [r P2_T, (r+1) P2_T), one row per thread, and TMA-loads
// only those.  Per column, after the CTA argmax, warp 0 pushes the CTA candidate (key, row
// index, its row of the current half: 144 B) into slot r of EVERY CTA of the cluster with
// st.async + mbarrier complete_tx; the deferred rank-1 update of the previous pivot overlaps
// the exchange; every CTA then takes the same cluster argmax (same key order as the single-CTA
// kernel: identical pivots) and reads the pivot row from its own shared memory.  At the half
// transition the owners of half 0's pivot rows push their L11 and X rows the same way.  Rows
// never move inside the panel; each CTA writes its rows to their final positions at the end;
// rank 0 emits the move list and the pivot values.  (A column costs one DSMEM round trip,
// ~520 cycles, more than the single-CTA kernel; in exchange each SM holds 1/CS of the panel.)
constexpr int P2C_MAX = 16;  // non-portable cluster size (one GPC): m <= 8192
constexpr int P2C_PUSH_WARPS = 3;
struct __align__(16) XSlot2 {
    unsigned long long key;
    int idx, pad;
    double row[16];  // the candidate's 128-byte row half
};
FROB_DEV void st_async_16b(unsigned raddr, const uint4 v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     raddr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
                 : "memory");
}

template <typename T, int PH, bool TWO>
__global__ void __launch_bounds__(P2_T, 1)
lu_panel2c_kernel(const __grid_constant__ CUtensorMap tmap, T *__restrict__ B, long long ld, int n, int k0, int w,
                  int *__restrict__ mv2, T *__restrict__ diag, const T *__restrict__ Bp, const int *__restrict__ mvp,
                  int kp0) {
    extern __shared__ __align__(1024) unsigned char stgb[];  // P2_T local rows x 128 B, 128B-swizzled (TMA)
    __shared__ __align__(8) unsigned long long tbar, hbar, xbar[2];
    __shared__ __align__(16) XSlot2 xs[2][P2C_MAX];
    __shared__ __align__(16) T L11s[PH][PH];  // half transition: pushed rows (128 B each)
    __shared__ __align__(16) T U12s[PH][PH];
    __shared__ __align__(16) T obox[2][PH][PH];  // this CTA's pivot rows of half 0: L11 | X
    __shared__ unsigned long long ck[2][P2_WARPS];
    __shared__ int ci[2][P2_WARPS];
    __shared__ __align__(16) T wrow[2][P2_WARPS][PH];
    constexpr int PW = 2 * PH;
    __shared__ int pivrow[PW];
    __shared__ int vac[PW];
    __shared__ unsigned evm_s;
    __shared__ int sdst[P2_T];
    static_assert(PH * sizeof(T) == 128, "row halves are 128 bytes");

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned rank, CSu;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(CSu));
    const int CS = (int)CSu;
    const int rbeg = (int)rank * P2_T;
    const int m = n - k0;
    const int E = (int)(sizeof(T) / 8);
    const bool two = TWO && w > PH;
    constexpr unsigned XB = (unsigned)sizeof(XSlot2);
    if (tid == 0) {
        mbar_init(smem_u32(&tbar), 1u);
        mbar_init(smem_u32(&hbar), 1u);
        mbar_init(smem_u32(&xbar[0]), 1u);
        mbar_init(smem_u32(&xbar[1]), 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync_all();  // every CTA's barriers exist before any remote complete_tx
    if (tid == 0) {
        mbar_arrive_expect_tx(smem_u32(&xbar[0]), (unsigned)CS * XB);
        if (w > 1) mbar_arrive_expect_tx(smem_u32(&xbar[1]), (unsigned)CS * XB);
        if (two) mbar_arrive_expect_tx(smem_u32(&hbar), (unsigned)(2 * PH * 128));
    }
    pdl_wait();
    pdl_trigger();  // after the wait (see lu2_factor)
    TL_BEGIN(1, k0 / Panel2W<T>::PW);
#define P2CT(i) do { if (rank == 0) P2T(i); } while (0)
#define P2CTJ(j, i) do { if ((j) == 5) P2CT(i); } while (0)
    P2CT(0);
    const int mr = min(P2_T, m - rbeg);  // rows of this CTA (>= 1)
    const int nbox = (mr + 255) / 256;
    auto tma_half = [&](int h) {
        mbar_arrive_expect_tx(smem_u32(&tbar), (unsigned)(nbox * 256 * 128));
        for (int b = 0; b < nbox; ++b)
            tma_load_2d(smem_u32(stgb + b * 256 * 128), &tmap, (k0 + h * PH) * E, k0 + rbeg + 256 * b,
                        smem_u32(&tbar));
    };
    auto row_from_stg = [&](int r, T (&dst)[PH]) {
        double t[16];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const double2 v = *reinterpret_cast<const double2 *>(stgb + swz128(r, c));
            t[2 * c] = v.x;
            t[2 * c + 1] = v.y;
        }
#pragma unroll
        for (int c = 0; c < PH; ++c) {
            if constexpr (sizeof(T) == 8) dst[c] = t[c];
            else dst[c] = make_double2(t[2 * c], t[2 * c + 1]);
        }
    };
    auto row_to_stg = [&](int r, const T (&src)[PH]) {
        const double *rd = reinterpret_cast<const double *>(src);
#pragma unroll
        for (int c = 0; c < 8; ++c)
            *reinterpret_cast<double2 *>(stgb + swz128(r, c)) = make_double2(rd[2 * c], rd[2 * c + 1]);
    };

    const int g = rbeg + tid;  // relative row of this thread
    T a[PH];
    int pst = -1;
    bool live = g < m;
    const bool fused = Bp != nullptr;
    __shared__ PreSmem<T, (TWO ? 2 * PH : PH)> psm;
    if (fused) {
        // fused look-ahead (see pre_update); rank 0 stores the previous step's U rows
        pre_update<T, PH, TWO>(Bp, mvp, kp0, B, ld, n, k0, w, g, rank == 0, tid, a, stgb, stgb + P2_T * 128, psm);
        __syncthreads();
    } else {
        if (tid == 0) tma_half(0);
        __syncthreads();
        mbar_wait_cta(smem_u32(&tbar), 0u);
        row_from_stg(tid, a);
        __syncthreads();  // the staging buffer is free
        if (two && tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tma_half(1);
        }
    }

    auto publish_first = [&]() {
        const unsigned long long bk = live ? pkey_bits(a[0]) : 0ull;
        const ArgMaxK wa = warp_argmax_key(bk, live ? g : INT_MAX);
        if (lane == 0) { ck[0][warp] = wa.k; ci[0][warp] = wa.i; }
        if (live && g == wa.i && wa.k != 0ull) st_row_smem<T, PH>(wrow[0][warp], a);
    };

    T u[PH];
    T lp = zero_of(T());
    bool pact = false;
    auto run_half = [&](const int JO, const int wh) {
#pragma unroll
        for (int c = 0; c < PH; ++c) u[c] = zero_of(T());
        lp = zero_of(T());
        pact = false;
        auto column = [&](auto Jc) {
            constexpr int J = decltype(Jc)::value;
            constexpr int s = J & 1;
            const int t = JO + J;  // exchange number (JO even: buffer s = t & 1)
            __syncthreads();
            P2CTJ(J, 40);
            // (a) CTA argmax, push of the CTA candidate to every CTA of the cluster (warps 0-2
            // each take the argmax and a third of the CS x 9 16-byte chunks)
            if (warp < P2C_PUSH_WARPS) {
                const ArgMaxK ca = warp_argmax_key(lane < P2_WARPS ? ck[s][lane] : 0ull,
                                                   lane < P2_WARPS ? ci[s][lane] : INT_MAX);
                const int cw = (ca.i == INT_MAX) ? 0 : ((ca.i - rbeg) >> 5);
                const unsigned slot = smem_u32(&xs[s][rank]);
                const unsigned bar = smem_u32(&xbar[s]);
                for (int task = lane + 32 * warp; task < CS * 9; task += 32 * P2C_PUSH_WARPS) {
                    const int r = task / 9, c = task - r * 9;
                    uint4 v;
                    if (c == 0) v = make_uint4((unsigned)ca.k, (unsigned)(ca.k >> 32), (unsigned)ca.i, 0u);
                    else v = *reinterpret_cast<const uint4 *>(reinterpret_cast<const unsigned char *>(wrow[s][cw]) +
                                                              (c - 1) * 16);
                    st_async_16b(mapa_u32(slot + c * 16, (unsigned)r), v, mapa_u32(bar, (unsigned)r));
                }
            }
            P2CTJ(J, 41);
            // (b) deferred update of pivot J-1 (columns >= J+1), overlapping the exchange
            if (pact) {
#pragma unroll
                for (int c = J + 1; c < PH; ++c) a[c] = msub(a[c], lp, u[c]);
            }
            // (c) cluster argmax, pivot row + reciprocal
            P2CTJ(J, 42);
            mbar_wait_parity(smem_u32(&xbar[s]), (unsigned)((t >> 1) & 1));
            P2CTJ(J, 43);
            const ArgMaxK ga = warp_argmax_key(lane < CS ? xs[s][lane].key : 0ull, lane < CS ? xs[s][lane].idx : INT_MAX);
            const int gi = ga.i;
            const int owner = min(gi / P2_T, CS - 1);
            ld_row_smem<T, PH>(u, reinterpret_cast<const T *>(xs[s][owner].row));
            if (tid == 0 && t + 2 < w) mbar_arrive_expect_tx(smem_u32(&xbar[s]), (unsigned)CS * XB);
            const T rc = rcp_spec(u[J]);
            if (tid == 0) {
                pivrow[JO + J] = gi;
                if (rank == 0) diag[k0 + JO + J] = u[J];
            }
            P2CTJ(J, 44);
            // (d) multiplier, eager update of column J+1
            const bool isp = live && g == gi;
            const bool act = live && !isp;
            if (isp) { live = false; pst = JO + J; }
            const T l = act ? mul(a[J], rc) : zero_of(T());
            pact = act;
            if (act) {
                a[J] = l;
                if constexpr (J + 1 < PH) a[J + 1] = msub(a[J + 1], l, u[J + 1]);
            }
            lp = l;
            P2CTJ(J, 45);
            if constexpr (J + 1 < PH) {
                if (J + 1 < wh) {
                    // (e) candidate of column J+1, warp argmax; (f) the warp winner publishes
                    const unsigned long long bk = live ? pkey_bits(a[J + 1]) : 0ull;
                    const ArgMaxK wa = warp_argmax_key(bk, live ? g : INT_MAX);
                    if (lane == 0) { ck[s ^ 1][warp] = wa.k; ci[s ^ 1][warp] = wa.i; }
                    if (live && g == wa.i && wa.k != 0ull) {
                        T *dst = wrow[s ^ 1][warp];
                        auto rowval = [&](const int c) { return (c >= J + 2) ? msub(a[c], l, u[c]) : a[c]; };
                        if constexpr (sizeof(T) == 8) {
#pragma unroll
                            for (int c = 0; c < PH; c += 2)
                                *reinterpret_cast<double2 *>(dst + c) = make_double2(rowval(c), rowval(c + 1));
                        } else {
#pragma unroll
                            for (int c = 0; c < PH; ++c) dst[c] = rowval(c);
                        }
                    }
                }
            }
            P2CT(2 + J + (JO ? 16 : 0) * 0);
        };
        static_for<PH>([&](auto Jc) {
            constexpr int Jv = decltype(Jc)::value;
            if (Jv < wh) column(Jc);
        });
    };

    P2CT(1);
    publish_first();
    run_half(0, min(w, PH));
    __syncthreads();
    P2CT(19);

    if constexpr (TWO) if (two) {
        // ---- half 1: gather half 0's pivot rows (L11 | X) from their owners, U12 = L11^{-1} X,
        // rank-PH update of this CTA's rows, swap
        if (!fused) mbar_wait_cta(smem_u32(&tbar), 1u);
        if (pst >= 0) {
            T x[PH];
            row_from_stg(tid, x);
            st_row_smem<T, PH>(obox[0][pst], a);
            st_row_smem<T, PH>(obox[1][pst], x);
        }
        __syncthreads();
        P2CT(22);
        {
            const unsigned hb = smem_u32(&hbar);
            for (int task = tid; task < PH * CS * 16; task += P2_T) {
                const int j = task / (CS * 16), rem = task - j * (CS * 16), r = rem >> 4, c = rem & 15;
                if (pivrow[j] / P2_T != (int)rank) continue;
                const int part = c >> 3, off = (c & 7) * 16;
                const uint4 v = *reinterpret_cast<const uint4 *>(reinterpret_cast<const unsigned char *>(obox[part][j]) + off);
                const unsigned dst = smem_u32(part ? &U12s[j][0] : &L11s[j][0]) + off;
                st_async_16b(mapa_u32(dst, (unsigned)r), v, mapa_u32(hb, (unsigned)r));
            }
        }
        P2CT(23);
        mbar_wait_parity(smem_u32(&hbar), 0u);
        P2CT(24);
        if (tid < PH) {
            T x[PH];
#pragma unroll
            for (int j = 0; j < PH; ++j) x[j] = U12s[j][tid];
#pragma unroll
            for (int q = 0; q < PH; ++q)
#pragma unroll
                for (int j = q + 1; j < PH; ++j) x[j] = msub(x[j], L11s[j][q], x[q]);
#pragma unroll
            for (int j = 0; j < PH; ++j) U12s[j][tid] = x[j];
        }
        __syncthreads();
        P2CT(25);
        if (g < m) {
            T x[PH];
            row_from_stg(tid, x);
            if (pst >= 0) {
#pragma unroll
                for (int c = 0; c < PH; ++c) x[c] = U12s[pst][c];
            } else {
#pragma unroll
                for (int j = 0; j < PH; ++j) {
                    const T lj = a[j];
#pragma unroll
                    for (int c = 0; c < PH; ++c) x[c] = msub(x[c], lj, U12s[j][c]);
                }
            }
            row_to_stg(tid, a);  // half 0's factored row waits in the staging buffer
#pragma unroll
            for (int c = 0; c < PH; ++c) a[c] = x[c];
        }
        __syncthreads();
        P2CT(18);
        publish_first();
        run_half(PH, w - PH);
        __syncthreads();
    }
    P2CT(20);

    // ---- final positions (pivrow is the same in every CTA): pivot j -> j; evicted top rows
    // (< w, not pivots) fill the rows vacated by pivots from below (>= w), in pivot order
    if (warp == 0) {
        const int pj = lane < w ? pivrow[lane] : -1;
        bool rp = false;
        if (lane < w)
            for (int q = 0; q < w; ++q) rp |= (pivrow[q] == lane);
        const unsigned pivmask = __ballot_sync(0xffffffffu, rp);
        const unsigned wmask = (w >= 32) ? 0xffffffffu : ((1u << w) - 1u);
        const unsigned evmask = wmask & ~pivmask;
        const bool isv = lane < w && pj >= w;
        const unsigned vb = __ballot_sync(0xffffffffu, isv);
        if (isv) vac[__popc(vb & ((1u << lane) - 1u))] = pj;
        if (lane == 0) evm_s = evmask;
        __syncwarp();
        if (rank == 0) {
            const bool moved = lane < w && pj != lane;
            const unsigned mb = __ballot_sync(0xffffffffu, moved);
            const int nm = __popc(mb);
            if (moved) {
                const int q = __popc(mb & ((1u << lane) - 1u));
                mv2[1 + q] = k0 + lane;
                mv2[1 + MV2_MAX + q] = k0 + pj;
            }
            const bool ev = (evmask >> lane) & 1u;
            if (ev) {
                const int q = nm + __popc(evmask & ((1u << lane) - 1u));
                mv2[1 + q] = k0 + vac[__popc(evmask & ((1u << lane) - 1u))];
                mv2[1 + MV2_MAX + q] = k0 + lane;
            }
            if (lane == 0) mv2[0] = nm + __popc(evmask);
        }
    }
    __syncthreads();
    {
        const unsigned evm = evm_s;
        int dst = g;
        if (pst >= 0) dst = pst;
        else if (g < w) dst = vac[__popc(evm & ((1u << g) - 1u))];
        sdst[tid] = (g < m) ? dst : -1;
    }
    __syncthreads();
    // coalesced write-back of this CTA's rows, 8 threads per 128-byte row half
    const long long ldd = ld * E;
    double *P = reinterpret_cast<double *>(B) + (long long)k0 * ldd + (long long)k0 * E;
    auto write_half = [&](int h) {
        const int wd = (min(w, (h + 1) * PH) - h * PH) * E;
#pragma unroll 4
        for (int idx = tid; idx < mr * 8; idx += P2_T) {
            const int r = idx >> 3, c = idx & 7;
            if (2 * c >= wd) continue;
            const double2 v = *reinterpret_cast<const double2 *>(stgb + swz128(r, c));
            double *out = P + (long long)sdst[r] * ldd + h * PH * E + 2 * c;
            if (2 * c + 1 < wd) *reinterpret_cast<double2 *>(out) = v;
            else out[0] = v.x;
        }
    };
    if constexpr (TWO) if (two) {
        write_half(0);  // half 0's rows sit at their local positions in the staging buffer
        __syncthreads();
    }
    if (g < m) row_to_stg(tid, a);
    __syncthreads();
    write_half(two ? 1 : 0);
    TL_END(1, k0 / Panel2W<T>::PW);
    P2CT(21);
#undef P2CT
#undef P2CTJ
}

// ---------------------------------------------------------------------------------------
// Update of step k0: for rows i in [k0, n) and columns c in [k0+w, n):
//   top rows (i < k0+w):   Bn[i][c] = U12 = L11^{-1} Bk[src_top][c]
//   other rows:            Bn[i][c] = Bk[src(i)][c] - L21[i][:] U12[:][c]
// where src maps the step's row moves (gather).  L11, L21 are the panel's output in Bk.
// Active tiles only exist while k0 + w < n, i.e. with w == PW.  Latency plan: L11, L21 and
// the identity-mapped D rows are requested before the move list is read; the pivot rows
// (X) and the few remapped D rows follow once it is known.
// Block (0, 0) also applies the moves to perm / iperm and stores the iperm snapshot.
constexpr int U2_TR = 64, U2_TC = 64, U2_T = 256;

template <typename T> struct SPad { static constexpr int P = 2; };   // 16-byte aligned smem rows
template <> struct SPad<double2> { static constexpr int P = 1; };

template <typename T>
FROB_DEV void cp_row16(T *dst, const T *src, int nelem) {  // nelem * sizeof(T) multiple of 16
    constexpr int E = 16 / sizeof(T);
    for (int e = 0; e < nelem; e += E) cp_async16(dst + e, src + e);
}

template <typename T, int PW>
__global__ void __launch_bounds__(U2_T, 2)
lu_update2_kernel(const T *__restrict__ Bk, T *__restrict__ Bn, long long ld, int n, int k0, int w,
                  const int *__restrict__ mv2, int *__restrict__ perm, int *__restrict__ iperm,
                  int *__restrict__ snap) {
    pdl_trigger();
    pdl_wait();
    constexpr int SP = SPad<T>::P;
    constexpr int E = 16 / (int)sizeof(T);  // elements per 16-byte chunk
    __shared__ int mdst[MV2_MAX], msrc[MV2_MAX];
    __shared__ int nmv_s;
    __shared__ __align__(16) T L11[PW][PW + SP];
    __shared__ __align__(16) T Us[PW][U2_TC];          // X, then U12 in place
    __shared__ __align__(16) T Ls[U2_TR][PW + SP];     // L21 rows of this tile
    const int tid = threadIdx.x;
    const int c0 = k0 + w + blockIdx.x * U2_TC;
    const int r0 = k0 + w + blockIdx.y * U2_TR;
    const bool tile = c0 < n;
    const bool rows = tile && r0 < n;
    const int nc = min(U2_TC, n - c0);
    const int ty = tid >> 4, tx = tid & 15;
    // ---- 1. requests independent of the move list
    if (tile) {
        for (int idx = tid; idx < PW * (PW / E); idx += U2_T) {
            const int i = idx / (PW / E), e = (idx % (PW / E)) * E;
            cp_async16(&L11[i][e], Bk + (long long)(k0 + i) * ld + k0 + e);
        }
        if (rows) {
            for (int idx = tid; idx < U2_TR * (PW / E); idx += U2_T) {
                const int r = idx / (PW / E), e = (idx % (PW / E)) * E;
                if (r0 + r < n) cp_async16(&Ls[r][e], Bk + (long long)(r0 + r) * ld + k0 + e);
            }
        }
    }
    cp_async_commit();
    T acc[4][4];
    if (rows) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = r0 + ty * 4 + i;
            const T *src = Bk + (long long)(r < n ? r : 0) * ld + c0 + tx * 4;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = (r < n && tx * 4 + j < nc) ? src[j] : zero_of(T());
        }
    }
    // ---- 2. the move list
    if (tid < MV2_MAX) {
        const int nm = mv2[0];
        if (tid == 0) nmv_s = nm;
        mdst[tid] = tid < nm ? mv2[1 + tid] : -1;
        msrc[tid] = tid < nm ? mv2[1 + MV2_MAX + tid] : -1;
    }
    __syncthreads();
    const int nm = nmv_s;
    if (blockIdx.x == 0 && blockIdx.y == 0) {
        // perm / iperm: new perm[dst] = old perm[src]; snapshot of iperm after the step
        int pv = 0;
        if (tid < nm) pv = perm[msrc[tid]];
        __syncthreads();
        if (tid < nm) {
            perm[mdst[tid]] = pv;
            iperm[pv] = mdst[tid];
        }
        __syncthreads();
        if (snap)
            for (int i = tid; i < n; i += U2_T) snap[i] = iperm[i];
    }
    if (!tile) return;
    // ---- 3. pivot rows X (top sources) and remapped D rows
    for (int idx = tid; idx < PW * (U2_TC / E); idx += U2_T) {
        const int i = idx / (U2_TC / E), e = (idx % (U2_TC / E)) * E;
        int src = k0 + i;
        for (int q = 0; q < nm; ++q)
            if (mdst[q] == k0 + i) src = msrc[q];
        if (e < nc) cp_async16(&Us[i][e], Bk + (long long)src * ld + c0 + e);
    }
    cp_async_commit();
    if (rows) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = r0 + ty * 4 + i;
            int src = r;
            for (int q = 0; q < nm; ++q)
                if (mdst[q] == r) src = msrc[q];
            if (src != r && r < n) {
                const T *sp = Bk + (long long)src * ld + c0 + tx * 4;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (tx * 4 + j < nc) acc[i][j] = sp[j];
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    // ---- 4. U12 = L11^{-1} X (unit lower forward substitution), one thread per column
    if (tid < U2_TC) {
        T x[PW];
#pragma unroll
        for (int i = 0; i < PW; ++i) x[i] = Us[i][tid];
#pragma unroll
        for (int q = 0; q < PW; ++q)
#pragma unroll
            for (int i = q + 1; i < PW; ++i) x[i] = msub(x[i], L11[i][q], x[q]);
#pragma unroll
        for (int i = 0; i < PW; ++i) Us[i][tid] = x[i];
        if (blockIdx.y == 0 && tid < nc) {
#pragma unroll
            for (int i = 0; i < PW; ++i) Bn[(long long)(k0 + i) * ld + c0 + tid] = x[i];
        }
    }
    __syncthreads();
    if (!rows) return;
    // ---- 5. A22 -= L21 U12
#pragma unroll
    for (int q = 0; q < PW; ++q) {
        T lv[4], uv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) lv[i] = Ls[ty * 4 + i][q];
#pragma unroll
        for (int j = 0; j < 4; ++j) uv[j] = Us[q][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = msub(acc[i][j], lv[i], uv[j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = r0 + ty * 4 + i;
        if (r >= n) continue;
        T *dst = Bn + (long long)r * ld + c0 + tx * 4;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (tx * 4 + j < nc) dst[j] = acc[i][j];
    }
}

// Tensor-pipe variant of the update (the default): the same gather and TRSM, then the rank-PW
// product on DMMA m8n8k4 fragments in the GEMM engine's register layout (8 warps as 2 x 4, warp
// tile 32 x 16), C fragments loaded straight from the (gathered) source rows; U12 is computed
// once per column block (first row block of tiles) and shared through Bn + a release flag.
constexpr int U2M_WGM = 2, U2M_WGN = 4;
template <typename T> struct U2Pad { static constexpr int P = 4; };   // row offset = 8 words mod 32
template <> struct U2Pad<double2> { static constexpr int P = 2; };

// CTAs per SM: real 3 (80 registers since the U12 solve went to four threads per column;
// n = 4096 BULK step 95 -> 77 us at m = 4096), complex 2
template <typename T> struct U2MinB { static constexpr int B = 3; };
template <> struct U2MinB<double2> { static constexpr int B = 2; };

template <typename T, int PW>
FROB_DEV void update2m_body(const T *__restrict__ Bk, T *__restrict__ Bn, long long ld, int n, int k0, int w,
                            const int *__restrict__ mv2, int *__restrict__ perm, int *__restrict__ iperm,
                            int *__restrict__ snap, int *__restrict__ u12f, int tag, int cbeg, int cend, int doperm,
                            bool stream) {
    constexpr int SP = U2Pad<T>::P;
    constexpr int E = 16 / (int)sizeof(T);
    constexpr int WM = U2_TR / U2M_WGM, WN = U2_TC / U2M_WGN, MT = WM / 8, NT = WN / 8;
    constexpr int V = AccW<T>::V;
    static_assert(U2M_WGM * U2M_WGN * 32 == U2_T, "8 warps");
    __shared__ int mdst[MV2_MAX], msrc[MV2_MAX];
    __shared__ int nmv_s;
    __shared__ __align__(16) T L11[PW][PW + SP];
    __shared__ __align__(16) T Us[PW][U2_TC + SP];     // X, then -U12 in place
    __shared__ __align__(16) T Ls[U2_TR][PW + SP];     // L21 rows of this tile
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp / U2M_WGN) * WM, wn0 = (warp % U2M_WGN) * WN;
    const int c0 = cbeg + blockIdx.x * U2_TC;
    const int r0 = k0 + w + blockIdx.y * U2_TR;
    // doperm == 2: the grid's extra last row of CTAs does the perm / iperm / snapshot work alone (off
    // the tiles' critical path: it cost the (0, 0) tile ~6k cycles of NEXT's ~10k)
    const bool pcta = doperm == 2 && blockIdx.y == gridDim.y - 1;
    const bool tile = c0 < cend && !pcta;
    const bool rows = tile && r0 < n;
    const int nc = min(U2_TC, cend - c0);
    NXT(0);
    // ---- 1. requests independent of the move list
    if (tile) {
        for (int idx = tid; idx < PW * (PW / E); idx += U2_T) {
            const int i = idx / (PW / E), e = (idx % (PW / E)) * E;
            cp_async16(&L11[i][e], Bk + (long long)(k0 + i) * ld + k0 + e);
        }
        if (rows) {
            for (int idx = tid; idx < U2_TR * (PW / E); idx += U2_T) {
                const int r = idx / (PW / E), e = (idx % (PW / E)) * E;
                if (r0 + r < n) cp_async16(&Ls[r][e], Bk + (long long)(r0 + r) * ld + k0 + e);
            }
        }
    }
    cp_async_commit();
    double acc[MT][NT][V];
    auto load_c = [&](int i, const T *src) {  // C fragments of row group i from a source row
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const int cc = wn0 + j * 8 + 2 * t;
            // (BULK: streaming loads -- evict-first in L2, so the trailing matrix passing through
            // does not push the concurrently running panel's code and columns out of L2)
            if constexpr (sizeof(T) == 8) {
                if (cc + 1 < nc) {  // one 16-byte load (cc even, rows 16-byte aligned)
                    const double2 *p2 = reinterpret_cast<const double2 *>(src + cc);
                    const double2 v = stream ? __ldcs(p2) : *p2;
                    acc[i][j][0] = v.x;
                    acc[i][j][1] = v.y;
                    continue;
                }
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const T v = (cc + e < nc) ? (stream ? __ldcs(src + cc + e) : src[cc + e]) : zero_of(T());
                if constexpr (sizeof(T) == 8) acc[i][j][e] = acc_re(v);
                else { acc[i][j][e] = acc_re(v); acc[i][j][2 + e] = acc_im(v); }
            }
        }
    };
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < V; ++e) acc[i][j][e] = 0.0;
    if (rows) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int r = r0 + wm0 + i * 8 + g;
            if (r < n) load_c(i, Bk + (long long)r * ld + c0);
        }
    }
    // ---- 2. the move list
    // source rows of this tile's rows [r0, r0 + U2_TR) and of the top rows [k0, k0 + PW): identity,
    // then the step's moves applied once (instead of a search of the move list per row)
    __shared__ int rmap[U2_TR + PW];
    __shared__ int u12ready_s;
    // (a grid with a single column tile -- the NEXT kernel -- lets every tile solve for itself:
    // no hand-off on its critical path)
    const bool solo = gridDim.x == 1;
    const bool prod = solo || blockIdx.y == 0;
    if (tid < U2_TR + PW) rmap[tid] = (tid < U2_TR) ? r0 + tid : k0 + (tid - U2_TR);
    if (tid < MV2_MAX) {
        const int nm = mv2[0];
        if (tid == 0) nmv_s = nm;
        mdst[tid] = tid < nm ? mv2[1 + tid] : -1;
        msrc[tid] = tid < nm ? mv2[1 + MV2_MAX + tid] : -1;
    }
    if (tid == 0 && !prod) {  // U12 of this column block already published? (one look, no spin)
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(u12f + blockIdx.x) : "memory");
        u12ready_s = v >= tag;
    }
    __syncthreads();
    const int nm = nmv_s;
    // consumer tiles whose U12 is already out request it now, beside the move list's row map
    const bool early = tile && !prod && u12ready_s;
    if (early) {
        for (int idx = tid; idx < PW * (U2_TC / E); idx += U2_T) {
            const int i = idx / (U2_TC / E), e = (idx % (U2_TC / E)) * E;
            if (e < nc) cp_async16(&Us[i][e], Bn + (long long)(k0 + i) * ld + c0 + e);
        }
        cp_async_commit();
    }
    if (tid < nm) {
        const int d = mdst[tid];
        if (d >= r0 && d < r0 + U2_TR) rmap[d - r0] = msrc[tid];
        else if (d >= k0 && d < k0 + PW) rmap[U2_TR + d - k0] = msrc[tid];
    }
    __syncthreads();
    NXT(1);
    if (doperm && (doperm == 2 ? (pcta && blockIdx.x == 0) : (blockIdx.x == 0 && blockIdx.y == 0))) {
        int pv = 0;
        if (tid < nm) pv = perm[msrc[tid]];
        __syncthreads();
        if (tid < nm) {
            perm[mdst[tid]] = pv;
            iperm[pv] = mdst[tid];
        }
        __syncthreads();
        if (snap)
            for (int i = tid; i < n; i += U2_T) snap[i] = iperm[i];
    }
    if (!tile) return;
    // ---- 3. the first row block of tiles PRODUCES U12 of its columns (gather of the pivot rows X,
    // TRSM), stores it in Bn's top rows and raises the column block's flag; the other tiles load
    // it from there (L2) once the flag is up, instead of each repeating the TRSM
    if (prod) {
        for (int idx = tid; idx < PW * (U2_TC / E); idx += U2_T) {
            const int i = idx / (U2_TC / E), e = (idx % (U2_TC / E)) * E;
            const int src = rmap[U2_TR + i];
            if (e < nc) cp_async16(&Us[i][e], Bk + (long long)src * ld + c0 + e);
        }
    }
    cp_async_commit();
    if (rows) {
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int r = r0 + wm0 + i * 8 + g;
            const int src = rmap[wm0 + i * 8 + g];
            if (src != r && r < n) load_c(i, Bk + (long long)src * ld + c0);
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    NXT(2);
    if (prod) {
        // ---- 4. U12 = L11^{-1} X (unit lower forward substitution): four threads per column (rows
        // part, part + 4, ...), x_q passed along the quad by shuffle -- a 4x shorter chain per thread
        {
            static_assert(U2_T == 4 * U2_TC, "four threads per column");
            constexpr int RP = PW / 4;
            const int c = tid >> 2, part = tid & 3;
            T x[RP];
#pragma unroll
            for (int ii = 0; ii < RP; ++ii) x[ii] = Us[part + 4 * ii][c];
#pragma unroll
            for (int q = 0; q < PW; ++q) {
                T xq;
                if constexpr (sizeof(T) == 8) {
                    xq = __shfl_sync(0xffffffffu, x[q >> 2], (lane & ~3) | (q & 3));
                } else {
                    xq.x = __shfl_sync(0xffffffffu, x[q >> 2].x, (lane & ~3) | (q & 3));
                    xq.y = __shfl_sync(0xffffffffu, x[q >> 2].y, (lane & ~3) | (q & 3));
                }
#pragma unroll
                for (int ii = (q >> 2); ii < RP; ++ii) {
                    const int i = part + 4 * ii;
                    if (i > q) x[ii] = msub(x[ii], L11[i][q], xq);
                }
            }
#pragma unroll
            for (int ii = 0; ii < RP; ++ii) Us[part + 4 * ii][c] = x[ii];
            if (c < nc && blockIdx.y == 0) {
#pragma unroll
                for (int ii = 0; ii < RP; ++ii) Bn[(long long)(k0 + part + 4 * ii) * ld + c0 + c] = x[ii];
            }
        }
        __syncthreads();
        if (tid == 0 && !solo) {
            __threadfence();
            asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(u12f + blockIdx.x), "r"(tag) : "memory");
        }
    } else if (!early) {
        if (tid == 0) {
            long long it = 0;
            int v;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(u12f + blockIdx.x) : "memory");
                if (v >= tag) break;
                __nanosleep(32);
                if (++it > (1LL << 26)) __trap();  // a producer that never runs: fail, do not hang
            }
        }
        __syncthreads();
        for (int idx = tid; idx < PW * (U2_TC / E); idx += U2_T) {
            const int i = idx / (U2_TC / E), e = (idx % (U2_TC / E)) * E;
            if (e < nc) cp_async16(&Us[i][e], Bn + (long long)(k0 + i) * ld + c0 + e);
        }
        cp_async_commit();
        cp_async_wait<0>();
        __syncthreads();
    }
    NXT(3);
    if (!rows) return;
    // ---- 5. C += (-L21) U12 on the tensor pipe
#pragma unroll
    for (int kk = 0; kk < PW; kk += 4) {
        T a[MT], b[NT];
#pragma unroll
        for (int i = 0; i < MT; ++i) a[i] = scal(Ls[wm0 + i * 8 + g][kk + t], -1.0);
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = Us[kk + t][wn0 + j * 8 + g];
        mma_tile<MT, NT>(acc, a, b);
    }
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int r = r0 + wm0 + i * 8 + g;
        if (r >= n) continue;
        T *dst = Bn + (long long)r * ld + c0;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            const int cc = wn0 + j * 8 + 2 * t;
            if constexpr (sizeof(T) == 8) {
                if (cc + 1 < nc) {
                    const double2 v2 = make_double2(acc[i][j][0], acc[i][j][1]);
                    if (stream) __stcs(reinterpret_cast<double2 *>(dst + cc), v2);
                    else *reinterpret_cast<double2 *>(dst + cc) = v2;
                }
                else if (cc < nc) dst[cc] = acc[i][j][0];
            } else {
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    if (cc + e < nc) dst[cc + e] = acc_val(acc[i][j], e);
            }
        }
    }
    NXT(5);
}


// Launch modes (look-ahead pipeline of lu2_factor, see there):
//   NEXT  (lookahead = 0): the columns of the next panel; waits for its predecessor as usual and
//         applies the step's moves to perm / iperm (+ snapshot).
//   BULK  (lookahead = 1): all columns right of the next panel; launched behind the NEXT panel,
//         which it does not need, so it does NOT wait at entry (its inputs are complete: the
//         panel it follows only released it after its own wait); the last CTA to finish waits for
//         that panel before exiting, so the grid's completion still implies the panel's.
template <typename T, int PW>
__global__ void __launch_bounds__(U2_T, U2MinB<T>::B)
lu_update2m_kernel(const T *__restrict__ Bk, T *__restrict__ Bn, long long ld, int n, int k0, int w,
                   const int *__restrict__ mv2, int *__restrict__ perm, int *__restrict__ iperm,
                   int *__restrict__ snap, int *__restrict__ u12f, int tag, int cbeg, int cend, int doperm,
                   int lookahead, int *__restrict__ done_ctr) {
    pdl_trigger();
    if (!lookahead) pdl_wait();
    TL_BEGIN(lookahead ? 3 : 2, k0 / PW);
    update2m_body<T, PW>(Bk, Bn, ld, n, k0, w, mv2, perm, iperm, snap, u12f, tag, cbeg, cend, doperm,
                         lookahead && n > 2048);
    TL_END(lookahead ? 3 : 2, k0 / PW);
    if (lookahead) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const int total = (int)(gridDim.x * gridDim.y);
            if (atomicAdd(done_ctr, 1) == total - 1) pdl_wait();
        }
    }
}

// Final U / L in final row order (see the file header).  snap[b * n + orig] = position of
// original row `orig` after step b.
// Rows [r0, r1) only (EarlyInv assembles the first h rows ahead of the rest).
template <typename T>
__global__ void lu_assemble2_kernel(const T *__restrict__ B0, const T *__restrict__ B1, long long ld, int n, int W,
                                    const int *__restrict__ perm, const int *__restrict__ snap, T *__restrict__ U,
                                    T *__restrict__ L, long long ldo, int r0, int r1) {
    pdl_trigger();
    pdl_wait();
    const long long total = (long long)(r1 - r0) * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = r0 + (int)(idx / n), c = (int)(idx % n);
        const int k = i / W, b = c / W;
        const T *Bk = (k & 1) ? B1 : B0;
        T uval = zero_of(T()), lval = zero_of(T());
        if (c >= i) {
            const T *Bs = (b == k) ? Bk : ((k & 1) ? B0 : B1);
            uval = Bs[(long long)i * ld + c];
            if (c == i) lval = one_of(T());
        } else if (b == k) {
            lval = Bk[(long long)i * ld + c];
        } else {
            const int p = snap[(long long)b * n + perm[i]];
            lval = ((b & 1) ? B1 : B0)[(long long)p * ld + c];
        }
        if (U == L) {
            U[(long long)i * ldo + c] = (c >= i) ? uval : lval;  // packed: strict L below, U on and above
        } else {
            U[(long long)i * ldo + c] = uval;
            L[(long long)i * ldo + c] = lval;
        }
    }
}

__global__ void iota2_kernel(int *p, int *q, int n, int *flags, int nflags) {
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { p[i] = i; q[i] = i; }
    if (flags && i < nflags) flags[i] = 0;
#ifdef FROB_TL
    if (flags && i == 0) atomicAdd(&g_tl_call, 1);
#endif
}

// ---------------------------------------------------------------------------------------
// tail of the int workspace: U12-ready flags (NEXT and BULK grids) + per-step finish counters
static size_t lu2_sync_ints(int n) {
    const size_t ncb = (size_t)(n + U2_TC - 1) / U2_TC + 1;
    return 2 * ncb + (size_t)(n + 7) / 8 + 1;
}

// can a cluster of cs panel CTAs (one SM each) be placed at all on this device?
template <typename T>
static bool panel2c_cluster_fits(int cs) {
    constexpr int PH = Panel2W<T>::PH;
    constexpr bool TWO = Panel2W<T>::PW > PH;
    const size_t smem = (size_t)2 * P2_T * 128 + 1024;
    if (cudaFuncSetAttribute(lu_panel2c_kernel<T, PH, TWO>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(lu_panel2c_kernel<T, PH, TWO>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) !=
            cudaSuccess)
        return false;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3((unsigned)cs);
    cfg.blockDim = dim3(P2_T);
    cfg.dynamicSmemBytes = smem;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, lu_panel2c_kernel<T, PH, TWO>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return nc > 0;
}

int lu2_panel_max_m() {
    static int v = [] {
        const char *e = tuning_env("FROB_P2C_MAX");
        int cs = e ? atoi(e) : P2C_MAX;
        cs = (cs >= 1 && cs < P2C_MAX) ? cs : P2C_MAX;
        // clusters above the portable 8 need 16 free SMs in one GPC: keep 8 if they do not fit
        if (cs > 8 && !(panel2c_cluster_fits<double>(cs) && panel2c_cluster_fits<double2>(cs))) cs = 8;
        return cs * P2_T;
    }();
    return v;
}

int lu2_max_n() {
    static int v = [] {
        const char *e = tuning_env("FROB_LU2_MAX");
        const int x = e ? atoi(e) : LU2_MAX_N;
        return x < LU2_MAX_N ? x : LU2_MAX_N;
    }();
    return v;
}

size_t lu2_int_elems(int n) {
    const int W = 8;  // smallest panel width (complex): most steps
    const size_t steps = (size_t)(n + W - 1) / W;
    return (size_t)n /* iperm */ + steps * MV2_INTS + steps * (size_t)n /* snapshots */ + lu2_sync_ints(n);
}

template <typename T, int PH, int R>
static cudaError_t launch_panel2(const CUtensorMap &tm, T *B, long long ld, int n, int k0, int w, int *mv2, T *diag,
                                 cudaStream_t s, const T *Bp = nullptr, const int *mvp = nullptr, int kp0 = 0) {
    const size_t smem = (size_t)(R + 1) * P2_T * 128 + 1024;  // staging + the fused look-ahead's D0 rows
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(lu_panel2_kernel<T, PH, R, (Panel2W<T>::PW > PH)>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    // panel flops: column j scales m-j-1 rows and updates their w-j-1 remaining entries
    double wk = 0.0;
    for (int j = 0; j < w; ++j) wk += (double)(n - k0 - j - 1) * (1.0 + 2.0 * (w - j - 1));
    ProfScope ps(sizeof(T) == 8 ? "lu_panel2<double>" : "lu_panel2<double2>", s, wk * (sizeof(T) == 8 ? 1.0 : 4.0));
    return launch_pdl(lu_panel2_kernel<T, PH, R, (Panel2W<T>::PW > PH)>, dim3(1), dim3(P2_T), smem, s, tm, B, ld, n,
                      k0, w, mv2, diag, Bp, mvp, kp0);
}

template <typename T, int PH>
static cudaError_t launch_panel2c(const CUtensorMap &tm, T *B, long long ld, int n, int k0, int w, int *mv2, T *diag,
                                  int CS, cudaStream_t s, const T *Bp = nullptr, const int *mvp = nullptr,
                                  int kp0 = 0) {
    constexpr bool TWO = Panel2W<T>::PW > PH;
    const size_t smem = (size_t)2 * P2_T * 128 + 1024;  // staging + the fused look-ahead's D0 rows
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(lu_panel2c_kernel<T, PH, TWO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e == cudaSuccess)  // clusters of 9..16 CTAs (m > 4096, the blocked getrf's panels)
            e = cudaFuncSetAttribute(lu_panel2c_kernel<T, PH, TWO>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    double wk = 0.0;
    for (int j = 0; j < w; ++j) wk += (double)(n - k0 - j - 1) * (1.0 + 2.0 * (w - j - 1));
    ProfScope ps(sizeof(T) == 8 ? "lu_panel2c<double>" : "lu_panel2c<double2>", s, wk * (sizeof(T) == 8 ? 1.0 : 4.0));
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2];
    cfg.gridDim = dim3((unsigned)CS);
    cfg.blockDim = dim3(P2_T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = (unsigned)CS;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    count_launch();
    return cudaLaunchKernelEx(&cfg, lu_panel2c_kernel<T, PH, TWO>, tm, B, ld, n, k0, w, mv2, diag, Bp, mvp, kp0);
}

template <typename T>
cudaError_t lu2_panel_inplace(const CUtensorMap &tm, T *A, long long lda, int n, int k0, int w, int *mv, T *diag,
                              cudaStream_t s) {
    constexpr int PH = Panel2W<T>::PH;
    const int m = n - k0;
    static_assert(MV2_INTS == MV_INTS && MV2_MAX == 2 * PW_MAX, "move-list layouts agree");
    if (m > lu2_panel_max_m() || m > P2C_MAX * P2_T) return cudaErrorInvalidValue;
    if (m > P2_T) return launch_panel2c<T, PH>(tm, A, lda, n, k0, w, mv, diag, (m + P2_T - 1) / P2_T, s);
    return launch_panel2<T, PH, 1>(tm, A, lda, n, k0, w, mv, diag, s);
}
template cudaError_t lu2_panel_inplace<double>(const CUtensorMap &, double *, long long, int, int, int, int *, double *,
                                               cudaStream_t);
template cudaError_t lu2_panel_inplace<double2>(const CUtensorMap &, double2 *, long long, int, int, int, int *,
                                                double2 *, cudaStream_t);

// ---------------------------------------------------------------------------------------
// EarlyInv (see lu.cuh): a lowest-priority auxiliary stream per device
static long long ld_of_ws(int n) { return ((long long)n + 7) / 8 * 8; }  // the callers' workspace ld
bool getrf_early_ok(int n) {
    static int mode = [] {
        const char *e = tuning_env("FROB_EARLY");
        return e ? atoi(e) : -1;
    }();
    return mode != 0 && n > LU2_MAX_N && n <= 2 * LU2_MAX_N;
}
int early_inv_h(int n) {
    static int mode = [] {
        const char *e = tuning_env("FROB_EARLY");
        return e ? atoi(e) : -1;
    }();
    static int frac = [] {  // h as a percentage of n (env FROB_EARLY_FRAC, A/B aid)
        const char *e = tuning_env("FROB_EARLY_FRAC");
        return e ? atoi(e) : 50;
    }();
    const int min_n = mode > 1 ? mode : 2048;  // (n = 1024: 3.16 ms with it, 3.10 without)
    if (mode == 0 || n < min_n || n > LU2_MAX_N) return 0;
    constexpr int PW = Panel2W<double>::PW;
    const int h = (int)((long long)n * frac / 100) / PW * PW;
    return (h > 0 && 2 * h <= n) ? h : 0;
}

// per-device streams: hi = 0 the lowest priority (EarlyInv work), 1 the highest (the LU's chain
// while EarlyInv work runs beside it: its panels take the SMs the auxiliary GEMMs free first)
static cudaError_t early_stream(int hi, cudaStream_t *out) {
    static std::mutex mu;
    static cudaStream_t st[2][64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 64) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(mu);
    if (!st[hi][dev]) {
        int least = 0, greatest = 0;
        if ((e = cudaDeviceGetStreamPriorityRange(&least, &greatest)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithPriority(&st[hi][dev], cudaStreamNonBlocking, hi ? greatest : least)) !=
            cudaSuccess)
            return e;
    }
    *out = st[hi][dev];
    return cudaSuccess;
}
static cudaError_t early_aux_stream(cudaStream_t *out) { return early_stream(0, out); }
// dst waits for everything enqueued on src so far
static cudaError_t stream_join(cudaStream_t dst, cudaStream_t src) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    e = cudaEventRecord(ev, src);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(dst, ev, 0);
    cudaEventDestroy(ev);
    return e;
}

// inv[pos[o]] = o: position -> original row after the snapshot's step
__global__ void invert_perm_kernel(const int *__restrict__ pos, int n, int *__restrict__ inv) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o < n) inv[pos[o]] = o;
}
// L21' rows [h, n), columns [0, h) in their order after step h / PW - 1 (at[j] = original row at
// position j then): column block b's multipliers sit in B_b at the original row's position after step b
__global__ void gather_l21_kernel(const double *__restrict__ B0, const double *__restrict__ B1, long long ld, int n,
                                  int h, int W, const int *__restrict__ at, const int *__restrict__ snap,
                                  double *__restrict__ out, long long ldo) {
    const long long total = (long long)(n - h) * h;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int j = h + (int)(idx / h), c = (int)(idx % h), b = c / W;
        const int p = snap[(long long)b * n + at[j]];
        out[(long long)j * ldo + c] = ((b & 1) ? B1 : B0)[(long long)p * ld + c];
    }
}

// split-K for the EarlyInv GEMMs: shorter CTA lifetimes beside the chain, whose cluster panels wait
// for whole SMs (n = 4096 Frobenius 31.42 -> 31.19 ms; env FROB_EARLY_SPLIT=0: off, A/B aid)
static int early_split() {
    static int v = [] {
        const char *e = tuning_env("FROB_EARLY_SPLIT");
        return e ? atoi(e) : 1;
    }();
    return v;
}

// the EarlyInv work of lu2_factor: fork from s after step h / PW - 1 is complete
static cudaError_t early_inv_launch(int n, const double *B0, const double *B1, long long ld, double *U, double *L,
                                    long long ldo, const int *perm, const int *snap, int *at, EarlyInv &ei,
                                    cudaStream_t s) {
    constexpr int PW = Panel2W<double>::PW;
    const int h = ei.h;
    cudaStream_t aux;
    cudaError_t e = early_aux_stream(&aux);
    if (e != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&ei.done, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = stream_join(aux, s)) != cudaSuccess) return e;
    EV_TRACE(30, 0, aux);
    {
        const long long total = (long long)h * n;
        const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
        count_launch();
        lu_assemble2_kernel<double><<<blocks, 256, 0, aux>>>(B0, B1, ld, n, PW, perm, snap, U, L, ldo, 0, h);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    EV_TRACE(31, 0, aux);
    if ((e = tri_inverses<double>(h, U, L, ldo, ei.vbuf, aux)) != cudaSuccess) return e;
    EV_TRACE(32, 0, aux);
    {
        GemmTag tag("gemm:tri_inv");
        auto p = gemm_params<double>(h, n - h, h, 1.0, U, ldo, U + h, ldo, 0.0, nullptr, ldo, ei.vbuf + h, ldo);
        p.triA = TRI_UPPER;
        p.force_split = early_split();
        if ((e = gemm_launch<double>(p, 1, aux)) != cudaSuccess) return e;
    }
    EV_TRACE(33, 0, aux);
    // W' = L21' L11^{-1} (rows in their order after step hstep - 1)
    const int *pos_h = snap + (long long)(h / PW - 1) * n;  // (snapshots of earlier steps stay valid)
    count_launch(2);
    invert_perm_kernel<<<(n + 255) / 256, 256, 0, aux>>>(pos_h, n, at);
    {
        const long long total = (long long)(n - h) * h;
        const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
        gather_l21_kernel<<<blocks, 256, 0, aux>>>(B0, B1, ld, n, h, PW, at, snap, ei.vbuf, ldo);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    {
        GemmTag tag("gemm:tri_inv");
        auto p = gemm_params<double>(n - h, h, h, 1.0, ei.vbuf + (long long)h * ldo, ldo, L, ldo, 0.0, nullptr, ldo,
                                     ei.vbuf + (long long)h * ldo + h, ldo);
        p.triB = TRI_LOWER;
        p.force_split = early_split();
        if ((e = gemm_launch<double>(p, 1, aux)) != cudaSuccess) return e;
    }
    // P11 = U11^{-1} L11^{-1}: the top-left block of the product's first term (vbuf's top-left block,
    // free again after the recursion)
    {
        GemmTag tag("gemm:product");
        auto p = gemm_params<double>(h, h, h, 1.0, U, ldo, L, ldo, 0.0, nullptr, ldo, ei.vbuf, ldo);
        p.triA = TRI_UPPER;
        p.triB = TRI_LOWER;
        p.force_split = early_split();
        if ((e = gemm_launch<double>(p, 1, aux)) != cudaSuccess) return e;
    }
    ei.pos_h = pos_h;
    ei.perm = perm;
    ei.wmap = nullptr;
    ei.ready = true;
    return cudaEventRecord(ei.done, aux);
}

// getrf's EarlyInv (see lu.cuh): A's first h rows hold U's rows and L11 (packed), rows [h, n) of its
// first h columns the multipliers L21 in their order before the tail's permutation
__global__ void early_extract_kernel(const double *__restrict__ A, long long lda, int n, int h,
                                     double *__restrict__ U, double *__restrict__ L, long long ld,
                                     double *__restrict__ l21, long long ldv) {
    const long long top = (long long)h * n, total = top + (long long)(n - h) * h;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        if (idx < top) {
            const int i = (int)(idx / n), j = (int)(idx % n);
            const double v = A[(long long)i * lda + j];
            U[(long long)i * ld + j] = (j >= i) ? v : 0.0;
            L[(long long)i * ld + j] = (j < i) ? v : ((j == i) ? 1.0 : 0.0);
        } else {
            const long long q = idx - top;
            const int i = h + (int)(q / h), j = (int)(q % h);
            l21[(long long)i * ldv + j] = A[(long long)i * lda + j];
        }
    }
}

cudaError_t getrf_early_launch(int n, const double *A, long long lda, int h, EarlyInv &ei, cudaStream_t s,
                               cudaEvent_t *l21_done) {
    cudaStream_t aux;
    cudaError_t e = early_aux_stream(&aux);
    if (e != cudaSuccess) return e;
    const long long ld = ld_of_ws(n);
    ei.h = h;
    if ((e = cudaEventCreateWithFlags(&ei.done, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(l21_done, cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = stream_join(aux, s)) != cudaSuccess) return e;
    EV_TRACE(30, 1, aux);
    {
        const long long total = (long long)h * n + (long long)(n - h) * h;
        count_launch();
        early_extract_kernel<<<(int)std::min<long long>((total + 255) / 256, 148LL * 8), 256, 0, aux>>>(
            A, lda, n, h, ei.U, ei.L, ld, ei.vbuf, ld);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = cudaEventRecord(*l21_done, aux)) != cudaSuccess) return e;
    }
    EV_TRACE(31, 1, aux);
    if ((e = tri_inverses<double>(h, ei.U, ei.L, ld, ei.vbuf, aux)) != cudaSuccess) return e;
    EV_TRACE(32, 1, aux);
    GemmTag tag("gemm:tri_inv");
    {   // V = U11^{-1} U12
        auto p = gemm_params<double>(h, n - h, h, 1.0, ei.U, ld, ei.U + h, ld, 0.0, nullptr, ld, ei.vbuf + h, ld);
        p.triA = TRI_UPPER;
        p.force_split = early_split();
        if ((e = gemm_launch<double>(p, 1, aux)) != cudaSuccess) return e;
    }
    {   // W' = L21' L11^{-1}
        auto p = gemm_params<double>(n - h, h, h, 1.0, ei.vbuf + (long long)h * ld, ld, ei.L, ld, 0.0, nullptr, ld,
                                     ei.vbuf + (long long)h * ld + h, ld);
        p.triB = TRI_LOWER;
        p.force_split = early_split();
        if ((e = gemm_launch<double>(p, 1, aux)) != cudaSuccess) return e;
    }
    {   // P11 = U11^{-1} L11^{-1}
        GemmTag ptag("gemm:product");
        auto p = gemm_params<double>(h, h, h, 1.0, ei.U, ld, ei.L, ld, 0.0, nullptr, ld, ei.vbuf, ld);
        p.triA = TRI_UPPER;
        p.triB = TRI_LOWER;
        p.force_split = early_split();
        if ((e = gemm_launch<double>(p, 1, aux)) != cudaSuccess) return e;
    }
    EV_TRACE(33, 1, aux);
    ei.pos_h = nullptr;
    ei.perm = nullptr;
    ei.ready = true;
    return cudaEventRecord(ei.done, aux);
}

// pipeline mode: 2 = fused look-ahead, 1 = separate NEXT kernels, 0 = panel -> full update per
// step (env FROB_LU2_LOOKAHEAD overrides, A/B aid).  Measured defaults (B200, n = 1024 / 4096):
// complex (8-column steps, 64 FMAs per row in the fused update) 2: 2.73 / 38.6 ms vs 3.00 / 44.1
// with mode 1; real (32-column steps: 1024 FMAs per row on the panel's one or few SMs) 1:
// 3.45 / 37.9 ms vs 3.88 / 38.9 with mode 2.
static int lu2_lookahead(bool cplx) {
    static int v = [] {
        const char *e = tuning_env("FROB_LU2_LOOKAHEAD");
        return e ? atoi(e) : -1;
    }();
    return v >= 0 ? v : ((cplx || Panel2W<double>::PW == Panel2W<double>::PH) ? 2 : 1);
}

// Look-ahead pipeline.  Step k (panel P_k at k0 = k PW) is followed by
//   BULK_k: the update of every column right of the NEXT panel's, launched AFTER P_{k+1} so that
//           it runs concurrently with it (P_{k+1} releases its dependents right after its own
//           wait; BULK_k does not wait at entry, its last CTA waits for P_{k+1} before exiting);
//   the update of the next panel's own PW columns is either fused into P_{k+1} (mode 2, the
//   default: P_{k+1} reads them from B_k and applies step k's update itself, see pre_update) or a
//   separate NEXT_k kernel between P_k and P_{k+1} (mode 1).
// Mode 2 stream order: P_0 | P_1 BULK_0 | P_2 BULK_1 | ...  P_{k+1} waits for BULK_{k-1}, whose
// completion implies P_k's; BULK_k is released only after that wait, so P_k and BULK_{k-1} are
// complete when it starts.  P_{k+1} writes columns [k0+PW, k0+2PW) of B_{k+1} (and the U rows of
// step k there), BULK_k the columns >= k0 + 2PW: disjoint.  BULK_k also applies step k's row moves
// to perm / iperm and takes the snapshot (in step order: the BULKs are serialised).
template <typename T>
static cudaError_t lu2_factor_on(int n, T *B0, T *B1, long long ld, T *U, T *L, long long ldo, int *perm, int *iw,
                                 T *diag, LuStats *stats, cudaStream_t s, EarlyInv *early, bool ew);

template <typename T>
cudaError_t lu2_factor(int n, T *B0, T *B1, long long ld, T *U, T *L, long long ldo, int *perm, int *iw, T *diag,
                       LuStats *stats, cudaStream_t s, EarlyInv *early) {
    constexpr int PW = Panel2W<T>::PW;
    if (n > LU2_MAX_N) return cudaErrorInvalidValue;
    // EarlyInv (real only): forked once step hstep - 1 is complete, i.e. behind BULK_{hstep-1}
    const bool ew = sizeof(T) == 8 && early && early->h > 0 && early->h < n && early->h % PW == 0 && early->vbuf;
    if (early && !ew) early->h = 0;
    static const int hi_mode = [] {
        const char *v = tuning_env("FROB_EARLY_HI");
        return v ? atoi(v) : 1;
    }();
    if (!ew || !hi_mode) return lu2_factor_on<T>(n, B0, B1, ld, U, L, ldo, perm, iw, diag, stats, s, early, ew);
    // the factorisation itself on the highest-priority stream, joined back into s
    cudaStream_t hs;
    cudaError_t e = early_stream(1, &hs);
    if (e == cudaSuccess) e = stream_join(hs, s);
    if (e == cudaSuccess) e = lu2_factor_on<T>(n, B0, B1, ld, U, L, ldo, perm, iw, diag, stats, hs, early, ew);
    const cudaError_t j = stream_join(s, hs);
    return e != cudaSuccess ? e : j;
}

template <typename T>
static cudaError_t lu2_factor_on(int n, T *B0, T *B1, long long ld, T *U, T *L, long long ldo, int *perm, int *iw,
                                 T *diag, LuStats *stats, cudaStream_t s, EarlyInv *early, bool ew) {
    constexpr int PW = Panel2W<T>::PW, PH = Panel2W<T>::PH;
    // fork step: 3/4 of the steps (the h rows are final from step h / PW; forking later leaves the
    // auxiliary GEMMs fewer of the chain's steps to slow: n = 4096 Frobenius 31.18 / 30.98 / 30.83 /
    // 31.05 ms at 50 / 70 / 75 / 80%; env FROB_EARLY_FORK: percent, A/B aid)
    static const int fork_pct = [] {
        const char *v = tuning_env("FROB_EARLY_FORK");
        return v ? atoi(v) : 75;
    }();
    const int nsteps = (n + PW - 1) / PW;
    const int hstep = ew ? std::min(nsteps - 1, std::max(early->h / PW, (int)((long long)nsteps * fork_pct / 100))) : -1;
    EV_TRACE(34, 0, s);
    const int steps = (n + PW - 1) / PW;
    const int ncb = (n + U2_TC - 1) / U2_TC + 1;
    int *iperm = iw;
    int *mvb = iw + n;
    int *snap = mvb + (size_t)steps * MV2_INTS;
    int *sync = iw + lu2_int_elems(n) - lu2_sync_ints(n);
    int *flagN = sync, *flagB = sync + ncb, *done = sync + 2 * ncb;
    const int nsync = (int)lu2_sync_ints(n);
    // TMA descriptors of the two ping-pong buffers (rows x 16-double boxes, 128B swizzle)
    const int E = (int)(sizeof(T) / 8);
    CUtensorMap tm[2];
    cudaError_t e = tma_map_rows128(&tm[0], B0, n, (long long)n * E, ld * E, 256);
    if (e == cudaSuccess) e = tma_map_rows128(&tm[1], B1, n, (long long)n * E, ld * E, 256);
    if (e != cudaSuccess) return e;
    e = launch_pdl(iota2_kernel, dim3((max(n, nsync) + 255) / 256), dim3(256), 0, s, perm, iperm, n, sync, nsync);
    if (e != cudaSuccess) return e;
    const int la = lu2_lookahead(sizeof(T) == 16);
    const char *nm_next = sizeof(T) == 8 ? "lu_next2<double>" : "lu_next2<double2>";
    const char *nm_bulk = sizeof(T) == 8 ? "lu_update2<double>" : "lu_update2<double2>";
    // update of step kk over columns [cb, ce); next: waits at entry + perm/iperm/snapshot work
    auto update = [&](int kk, int cb, int ce, bool next, bool doperm) -> cudaError_t {
        const int k0 = kk * PW, w = min(PW, n - k0), m = n - k0;
        const T *Bk = (kk & 1) ? B1 : B0;
        T *Bn = (kk & 1) ? B0 : B1;
        const int cols = max(0, ce - cb), rows = n - k0 - w;
        dim3 grid(max(1, (cols + U2_TC - 1) / U2_TC), max(1, (rows + U2_TR - 1) / U2_TR));
        if (cols == 0) grid = dim3(1, 1);
        // NEXT: one more row of CTAs for the perm / iperm / snapshot work (doperm = 2)
        const int dp = doperm ? (next ? 2 : 1) : 0;
        if (dp == 2) grid.y += 1;
        const double upd = ((double)(m - w) * 2.0 * w + (double)w * w) * (double)cols;  // GEMM + TRSM
        ProfScope ps(next ? nm_next : nm_bulk, s, upd * (sizeof(T) == 8 ? 1.0 : 4.0));
        return launch_pdl(lu_update2m_kernel<T, PW>, grid, dim3(U2_T), 0, s, Bk, Bn, ld, n, k0, w,
                          (const int *)(mvb + (size_t)kk * MV2_INTS), perm, iperm,
                          (doperm && kk + 1 < steps) ? snap + (size_t)kk * n : (int *)nullptr, next ? flagN : flagB,
                          kk + 1, cb, ce, dp, next ? 0 : 1, done + kk);
    };
    for (int k = 0; k < steps; ++k) {
        const int k0 = k * PW, w = min(PW, n - k0), m = n - k0;
        T *Bk = (k & 1) ? B1 : B0;
        int *mv2 = mvb + (size_t)k * MV2_INTS;
        // one CTA up to P2_T rows, else a cluster of ceil(m / P2_T) CTAs (measured: a 2-CTA cluster
        // beats one CTA with two rows per thread at 512 < m <= 1024)
        // fused look-ahead: P_k reads its columns from B_{k-1} and applies step k-1's update itself
        const bool fz = la == 2 && k > 0;
        const T *Bp = fz ? ((k & 1) ? B0 : B1) : nullptr;
        const int *mvp = fz ? mvb + (size_t)(k - 1) * MV2_INTS : nullptr;
        if (m > P2_T)
            e = launch_panel2c<T, PH>(tm[k & 1], Bk, ld, n, k0, w, mv2, diag, (m + P2_T - 1) / P2_T, s, Bp, mvp, k0 - PW);
        else e = launch_panel2<T, PH, 1>(tm[k & 1], Bk, ld, n, k0, w, mv2, diag, s, Bp, mvp, k0 - PW);
        if (e != cudaSuccess) return e;
        if (la == 0) {
            if ((e = update(k, k0 + w, n, true, true)) != cudaSuccess) return e;
            continue;
        }
        if (k >= 1) {  // BULK_{k-1}: the columns right of P_k's, concurrent with P_k
            const int cb = k0 + PW;
            if ((la == 1 && cb < n) || la == 2)
                if ((e = update(k - 1, min(cb, n), n, false, la == 2)) != cudaSuccess) return e;
        }
        if constexpr (sizeof(T) == 8) {
            if (k == hstep) EV_TRACE(36, 0, s);
            // (real steps use n / 32 of the n / 8 snapshot slots lu2_int_elems sizes for complex: the
            // position -> row map of EarlyInv lives behind them)
            if (k == hstep && (e = early_inv_launch(n, B0, B1, ld, U, L, ldo, perm, snap, snap + (size_t)steps * n,
                                                    *early, s)) != cudaSuccess)
                return e;
        }
        if (la == 1 && (e = update(k, k0 + w, min(n, k0 + w + PW), true, true)) != cudaSuccess) return e;  // NEXT_k
    }
    // fused mode: the last step's row moves still go to perm / iperm
    if (la == 2 && (e = update(steps - 1, n, n, true, true)) != cudaSuccess) return e;
    {
        const long long total = (long long)n * n;
        const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
        e = launch_pdl(lu_assemble2_kernel<T>, dim3(blocks), dim3(256), 0, s, (const T *)B0, (const T *)B1, ld, n,
                       PW, (const int *)perm, (const int *)snap, U, L, ldo, ew ? early->h : 0, n);
        if (e != cudaSuccess) return e;
    }
    if (stats) e = lu_stats_launch<T>(diag, n, stats, s);
    EV_TRACE(35, 0, s);
    return e;
}
template cudaError_t lu2_factor<double>(int, double *, double *, long long, double *, double *, long long, int *,
                                        int *, double *, LuStats *, cudaStream_t, EarlyInv *);
template cudaError_t lu2_factor<double2>(int, double2 *, double2 *, long long, double2 *, double2 *, long long,
                                         int *, int *, double2 *, LuStats *, cudaStream_t, EarlyInv *);

#ifdef FROB_TL
extern "C" int frob_tl_reset() {
    static unsigned long long s[5][1024], z[5][1024];
    for (auto &a : s) for (auto &v : a) v = ~0ull;
    for (auto &a : z) for (auto &v : a) v = 0ull;
    if (cudaMemcpyToSymbol(g_tl_start, s, sizeof(s)) != cudaSuccess) return 1;
    const int zero = 0;
    if (cudaMemcpyToSymbol(g_tl_call, &zero, sizeof(int)) != cudaSuccess) return 1;
    return cudaMemcpyToSymbol(g_tl_end, z, sizeof(z)) == cudaSuccess ? 0 : 1;
}
extern "C" int frob_nx_read(long long *out) {
    return cudaMemcpyFromSymbol(out, g_nx_tr, sizeof(g_nx_tr)) == cudaSuccess ? 0 : 1;
}
extern "C" int frob_tl_read(unsigned long long *start, unsigned long long *end) {
    if (cudaMemcpyFromSymbol(start, g_tl_start, sizeof(g_tl_start)) != cudaSuccess) return 1;
    return cudaMemcpyFromSymbol(end, g_tl_end, sizeof(g_tl_end)) == cudaSuccess ? 0 : 1;
}
#endif
}  // namespace frob
