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
#include <cstdio>
#include <utility>
#include <algorithm>
#include "lu.cuh"
#include "tma.cuh"

namespace frob {

constexpr int P2_T = 512;
constexpr int P2_WARPS = P2_T / 32;
constexpr int P2_STG = 18;  // staging row stride in doubles (16 + 2: 16-byte aligned, conflict free)

// panel width of one step: two 128-byte row halves (32 real / 16 complex columns)
template <typename T> struct Panel2W { static constexpr int PW = 32, PH = 16; };
template <> struct Panel2W<double2> { static constexpr int PW = 8, PH = 8; };  // one half: the two-half complex variant spills

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
                 int *__restrict__ mv2, T *__restrict__ diag) {
    pdl_trigger();
    extern __shared__ __align__(1024) unsigned char stgb[];  // R * P2_T rows x 128 B, 128B-swizzled (TMA)
    __shared__ __align__(8) unsigned long long tbar;
    if (threadIdx.x == 0) {
        mbar_init(smem_u32(&tbar), 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();
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

    // ---- half 0: TMA load -> registers; half 1 then streams into the staging buffer
    if (tid == 0) tma_half(0, 0u);
    __syncthreads();
    mbar_wait_cta(smem_u32(&tbar), 0u);
    T a[R][PH];
    int grow[R], pst[R];
    unsigned live = 0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
        grow[q] = q * P2_T + tid;
        pst[q] = -1;
        if (grow[q] < m) live |= 1u << q;
        row_from_stg(grow[q], a[q]);
    }
    __syncthreads();  // every thread has read its half-0 rows: the staging buffer is free
    if (two && tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_half(1, 1u);
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
        mbar_wait_cta(smem_u32(&tbar), 1u);
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
    P2T(21);
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

// Final U / L in final row order (see the file header).  snap[b * n + orig] = position of
// original row `orig` after step b.
template <typename T>
__global__ void lu_assemble2_kernel(const T *__restrict__ B0, const T *__restrict__ B1, long long ld, int n, int W,
                                    const int *__restrict__ perm, const int *__restrict__ snap, T *__restrict__ U,
                                    T *__restrict__ L, long long ldo) {
    pdl_trigger();
    pdl_wait();
    const long long total = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / n), c = (int)(idx - (long long)i * n);
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
        U[(long long)i * ldo + c] = uval;
        L[(long long)i * ldo + c] = lval;
    }
}

__global__ void iota2_kernel(int *p, int *q, int n) {
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { p[i] = i; q[i] = i; }
}

// ---------------------------------------------------------------------------------------
size_t lu2_int_elems(int n) {
    const int W = 8;  // smallest panel width (complex): most steps
    const size_t steps = (size_t)(n + W - 1) / W;
    return (size_t)n /* iperm */ + steps * MV2_INTS + steps * (size_t)n /* snapshots */;
}

template <typename T, int PH, int R>
static cudaError_t launch_panel2(const CUtensorMap &tm, T *B, long long ld, int n, int k0, int w, int *mv2, T *diag,
                                 cudaStream_t s) {
    const size_t smem = (size_t)R * P2_T * 128 + 1024;
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
                      k0, w, mv2, diag);
}

template <typename T>
cudaError_t lu2_factor(int n, T *B0, T *B1, long long ld, T *U, T *L, long long ldo, int *perm, int *iw, T *diag,
                       LuStats *stats, cudaStream_t s) {
    constexpr int PW = Panel2W<T>::PW, PH = Panel2W<T>::PH;
    if (n > LU2_MAX_N) return cudaErrorInvalidValue;
    const int steps = (n + PW - 1) / PW;
    int *iperm = iw;
    int *mvb = iw + n;
    int *snap = mvb + (size_t)steps * MV2_INTS;
    // TMA descriptors of the two ping-pong buffers (rows x 16-double boxes, 128B swizzle)
    const int E = (int)(sizeof(T) / 8);
    CUtensorMap tm[2];
    cudaError_t e = tma_map_rows128(&tm[0], B0, n, (long long)n * E, ld * E, 256);
    if (e == cudaSuccess) e = tma_map_rows128(&tm[1], B1, n, (long long)n * E, ld * E, 256);
    if (e != cudaSuccess) return e;
    e = launch_pdl(iota2_kernel, dim3((n + 255) / 256), dim3(256), 0, s, perm, iperm, n);
    if (e != cudaSuccess) return e;
    for (int k = 0; k < steps; ++k) {
        const int k0 = k * PW, w = min(PW, n - k0), m = n - k0;
        T *Bk = (k & 1) ? B1 : B0;
        T *Bn = (k & 1) ? B0 : B1;
        int *mv2 = mvb + (size_t)k * MV2_INTS;
        if (m <= P2_T) e = launch_panel2<T, PH, 1>(tm[k & 1], Bk, ld, n, k0, w, mv2, diag, s);
        else e = launch_panel2<T, PH, 2>(tm[k & 1], Bk, ld, n, k0, w, mv2, diag, s);
        if (e != cudaSuccess) return e;
        const int rest = n - k0 - w;
        dim3 grid(max(1, (rest + U2_TC - 1) / U2_TC), max(1, (rest + U2_TR - 1) / U2_TR));
        const double upd = ((double)(m - w) * 2.0 * w + (double)w * w) * (double)rest;  // GEMM + TRSM
        ProfScope ps(sizeof(T) == 8 ? "lu_update2<double>" : "lu_update2<double2>", s, upd * (sizeof(T) == 8 ? 1.0 : 4.0));
        e = launch_pdl(lu_update2_kernel<T, PW>, grid, dim3(U2_T), 0, s, (const T *)Bk, Bn, ld, n, k0, w,
                       (const int *)mv2, perm, iperm, k + 1 < steps ? snap + (size_t)k * n : (int *)nullptr);
        if (e != cudaSuccess) return e;
    }
    {
        const long long total = (long long)n * n;
        const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 8);
        e = launch_pdl(lu_assemble2_kernel<T>, dim3(blocks), dim3(256), 0, s, (const T *)B0, (const T *)B1, ld, n,
                       PW, (const int *)perm, (const int *)snap, U, L, ldo);
        if (e != cudaSuccess) return e;
    }
    if (stats) e = lu_stats_launch<T>(diag, n, stats, s);
    return e;
}
template cudaError_t lu2_factor<double>(int, double *, double *, long long, double *, double *, long long, int *,
                                        int *, double *, LuStats *, cudaStream_t);
template cudaError_t lu2_factor<double2>(int, double2 *, double2 *, long long, double2 *, double2 *, long long,
                                         int *, int *, double2 *, LuStats *, cudaStream_t);

}  // namespace frob
