// lu.cu -- LU panel / swap+TRSM / diagnostics kernels, the triangular-inverse
// recursion and the GEMM launcher.  See lu.cuh and DESIGN.md section "Kernels".
#include <cooperative_groups.h>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <type_traits>
#include <mutex>
#include <vector>
#include <string>
#include <algorithm>
#include "lu.cuh"
#include "tma.cuh"

namespace cg = cooperative_groups;

namespace frob {

// =====================================================================================
// GEMM launcher
// =====================================================================================
// algorithmic flops of a (paired, batched) launch: 2 M N K, halved per triangular operand
template <typename T>
static double gemm_work(const GemmPair<T> &pp, int b0, int b1) {
    auto one = [](const GemmParams<T> &p) {
        double f = 2.0 * p.M * (double)p.N * p.K;
        if (p.triA != TRI_NONE) f *= 0.5;
        if (p.triB != TRI_NONE) f *= (p.triA != TRI_NONE) ? (2.0 / 3.0) : 0.5;
        return f * (sizeof(T) == 8 ? 1.0 : 4.0);
    };
    return one(pp.q[0]) * b0 + (b1 > 0 ? one(pp.q[1]) * b1 : 0.0);
}

// split-K (cluster reduction, see gemm_tile) serves plain-store epilogues of non-persistent GEMMs
template <typename T>
static bool split_ok(const GemmParams<T> &p) {
    return !p.counter && p.epi == EPI_STORE;
}

template <typename T, bool VEC, int BIG>
static cudaError_t gemm_launch_cfg(const GemmPair<T> &pp, int batch0, int batch1, cudaStream_t s) {
    using Cf = GemmCfg<T, BIG>;
    constexpr size_t smem = gemm_smem_bytes<T, BIG>();
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(gemm_kernel<T, VEC, BIG, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if constexpr (!BIG)
            if (e == cudaSuccess)
                e = cudaFuncSetAttribute(gemm_kernel<T, VEC, BIG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    const GemmParams<T> &p0 = pp.q[0];
    if (p0.counter) {
        const int D = (p0.M + Cf::BM - 1) / Cf::BM;
        const int grid = min(D * D, 148 * 3);
        cudaError_t e = cudaMemsetAsync(p0.counter, 0, sizeof(int), s);
        if (e != cudaSuccess) return e;
        ProfScope ps(g_gemm_tag ? g_gemm_tag : sizeof(T) == 8 ? "gemm<double>" : "gemm<double2>", s, gemm_work(pp, batch0, batch1));
        return launch_pdl(gemm_kernel<T, VEC, BIG, false>, dim3(grid, 1, 1), dim3(Cf::WGM * Cf::WGN * 32), smem, s, pp);
    }
    int M = p0.M, N = p0.N;
    if (batch1 > 0) {
        M = max(M, pp.q[1].M);
        N = max(N, pp.q[1].N);
    }
    dim3 grid((N + Cf::BN - 1) / Cf::BN, (M + Cf::BM - 1) / Cf::BM, batch0 + batch1);
    GemmPair<T> q = pp;
    // split-K for grids far below the 148 SMs x 3 resident CTAs with long k-ranges: the S
    // k-chunks of a tile run as one (1, 1, S) cluster and are summed in DSMEM in chunk order
    {
        const long long tiles = (long long)grid.x * grid.y * grid.z;
        int S = 1;
        const int K = max(p0.K, batch1 > 0 ? pp.q[1].K : 0);
        const bool ok = !BIG && p0.epi == EPI_STORE && (batch1 == 0 || pp.q[1].epi == EPI_STORE) &&
                        split_ok(p0) && (batch1 == 0 || split_ok(pp.q[1]));
        if (ok && tiles * 2 <= 148LL * 3 && K >= 256) {
            S = (int)std::min<long long>(8, (148LL * 3) / tiles);
            S = std::min(S, K / 128);
        }
        if (ok && p0.force_split && K >= 512) S = std::max(S, std::min(4, K / 256));
        if (S > 1) {
            grid.z *= S;
            q.q[0].ksplit = q.q[1].ksplit = S;
        } else {
            q.q[0].ksplit = q.q[1].ksplit = 1;
        }
    }
    const long long ctas = (long long)grid.x * grid.y * grid.z;
    // policy (tuning aid, env FROB_PDL_GEMM): 0 = release after the main loop, 1 = early for
    // single-wave grids, 2 = always early; default 0 (measured best)
    static int policy = [] {
        const char *v = tuning_env("FROB_PDL_GEMM");
        return v ? atoi(v) : 0;
    }();
    const bool early = policy == 2 || (policy == 1 && ctas <= 148LL * (BIG ? 1 : 3));
    q.q[0].early_trigger = q.q[1].early_trigger = early ? 1 : 0;
    ProfScope ps(g_gemm_tag ? g_gemm_tag : sizeof(T) == 8 ? "gemm<double>" : "gemm<double2>", s, gemm_work(pp, batch0, batch1));
    if (!BIG && q.q[0].ksplit > 1)
        return launch_pdl_cluster_z(gemm_kernel<T, VEC, BIG, !BIG>, grid, dim3(Cf::WGM * Cf::WGN * 32), smem, s,
                                    q.q[0].ksplit, q);
    return launch_pdl(gemm_kernel<T, VEC, BIG, false>, grid, dim3(Cf::WGM * Cf::WGN * 32), smem, s, q);
}

template <typename T, bool VEC>
static cudaError_t gemm_launch_impl(const GemmPair<T> &pp, int batch0, int batch1, cudaStream_t s) {
    // 128 x 128 tiles when they fill >= 2 waves of the 148 SMs (real only)
    const GemmParams<T> &p0 = pp.q[0];
    long long tiles = (long long)((p0.M + 127) / 128) * ((p0.N + 127) / 128) * batch0;
    if (batch1 > 0) tiles += (long long)((pp.q[1].M + 127) / 128) * ((pp.q[1].N + 127) / 128) * batch1;
    // (measured: the 128 x 128 variant runs one CTA per SM and is slower than 3 x 64 x 64 per SM;
    //  kept compiled for experiments, not selected)
    if constexpr (sizeof(T) == 8) {
        if (!p0.counter && tiles >= (1LL << 40)) return gemm_launch_cfg<T, VEC, 1>(pp, batch0, batch1, s);
        // 64 x 128 tiles, two CTAs per SM, for long k-ranges once they fill two waves
        static const int wide_k = [] {  // env FROB_GEMM_WIDE_K: the k-range from which it is used (A/B aid)
            const char *v = tuning_env("FROB_GEMM_WIDE_K");
            return v ? atoi(v) : 1024;
        }();
        long long t2 = (long long)((p0.M + 63) / 64) * ((p0.N + 127) / 128) * batch0;
        if (batch1 > 0) t2 += (long long)((pp.q[1].M + 63) / 64) * ((pp.q[1].N + 127) / 128) * batch1;
        const int K = batch1 > 0 ? std::min(p0.K, pp.q[1].K) : p0.K;
        // (plain operands only: the coarser tiles waste more of a triangular k-range, and the B-row
        // gather's per-stage index loads double with BK = 8 -- both measured slower)
        auto plain = [](const GemmParams<T> &q) { return q.triA == TRI_NONE && q.triB == TRI_NONE && !q.browmap; };
        if (wide_k > 0 && !p0.counter && K >= wide_k && t2 >= 2LL * 148 * 2 && plain(p0) &&
            (batch1 == 0 || plain(pp.q[1])))
            return gemm_launch_cfg<T, VEC, 2>(pp, batch0, batch1, s);
    }
    return gemm_launch_cfg<T, VEC, 0>(pp, batch0, batch1, s);
}

static bool aligned16(const void *ptr) { return ((uintptr_t)ptr & 15u) == 0; }

template <typename T>
static bool gemm_vec_ok(const GemmParams<T> &p, int batch) {
    constexpr int E = 16 / sizeof(T);
    return aligned16(p.A) && aligned16(p.B) && (p.lda % E == 0) && (p.ldb % E == 0) &&
           (batch <= 1 || ((p.sA % E == 0) && (p.sB % E == 0)));
}

template <typename T>
cudaError_t gemm_launch(const GemmParams<T> &p, int batch, cudaStream_t s) {
    if (p.M <= 0 || p.N <= 0 || batch <= 0) return cudaSuccess;
    GemmPair<T> pp{};
    pp.q[0] = p;
    pp.q[1] = p;
    pp.zsplit = batch;
    return gemm_vec_ok(p, batch) ? gemm_launch_impl<T, true>(pp, batch, 0, s) : gemm_launch_impl<T, false>(pp, batch, 0, s);
}

// two independent problems (each possibly batched) in one launch
template <typename T>
cudaError_t gemm_launch2(const GemmParams<T> &p0, int b0, const GemmParams<T> &p1, int b1, cudaStream_t s) {
    if (p0.M <= 0 || p0.N <= 0 || b0 <= 0) return gemm_launch<T>(p1, b1, s);
    if (p1.M <= 0 || p1.N <= 0 || b1 <= 0) return gemm_launch<T>(p0, b0, s);
    GemmPair<T> pp{};
    pp.q[0] = p0;
    pp.q[1] = p1;
    pp.zsplit = b0;
    const bool vec = gemm_vec_ok(p0, b0) && gemm_vec_ok(p1, b1);
    return vec ? gemm_launch_impl<T, true>(pp, b0, b1, s) : gemm_launch_impl<T, false>(pp, b0, b1, s);
}
template cudaError_t gemm_launch<double>(const GemmParams<double> &, int, cudaStream_t);
template cudaError_t gemm_launch<double2>(const GemmParams<double2> &, int, cudaStream_t);

// =====================================================================================
// Panel factorisation: rows in REGISTERS, one CTA (or a thread-block cluster with DSMEM)
// =====================================================================================
// Thread t of cluster rank c owns panel rows rbeg + t + q*PANEL_T (q < R), rbeg = c*R*PANEL_T,
// all PW columns in registers.  The column loop is a compact runtime loop (a fully
// unrolled panel overflows the instruction cache); register indices stay static by
// ROTATING each row one slot per column: slot 0 always holds the current column, slots
// 1..PW-1-j the columns to its right, and the finished column (multiplier, or U entry for
// pivot rows) is rotated into slot PW-1.  Per column j:
//   local argmax (slot 0) -> warp-shuffle argmax; the winning lane publishes its whole row
//   next to the candidate -> ONE __syncthreads -> block argmax in every warp
//   [cluster: CTA winner + row to DSMEM, ONE cluster barrier, cluster argmax]
//   -> pivot row read with vector shared loads -> rank-1 update of own rows -> rotate.
// Rows never move during the panel; at the end each row is written to its final
// position and the row movement for the other columns is emitted.
constexpr int PANEL_T = 256;
constexpr int PANEL_W = PANEL_T / 32;

template <typename T, int PW>
FROB_DEV void store_row(T *dst, const T (&r)[PW]) {
    if constexpr (sizeof(T) == 8) {
#pragma unroll
        for (int c = 0; c < PW; c += 2)
            *reinterpret_cast<double2 *>(dst + c) = make_double2(r[c], r[c + 1]);
    } else {
#pragma unroll
        for (int c = 0; c < PW; ++c) dst[c] = r[c];
    }
}

template <typename T, int PW, int R>
FROB_DEV void store_row_sel(T *dst, const T (&a)[R][PW], int q) {
    switch (q) {
        case 0: store_row<T, PW>(dst, a[0]); break;
        case 1: if constexpr (R > 1) store_row<T, PW>(dst, a[1]); break;
        case 2: if constexpr (R > 2) store_row<T, PW>(dst, a[2]); break;
        default: if constexpr (R > 3) store_row<T, PW>(dst, a[R - 1]); break;
    }
}

template <typename T, int PW>
FROB_DEV void load_row(T (&u)[PW], const T *src) {
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

constexpr int PANEL_UNROLL = 4;

#ifdef FROB_PANEL_TRACE
__device__ long long g_panel_trace[64];
#define PTRACE(i) do { if (threadIdx.x == 0 && blockIdx.x == 0) g_panel_trace[i] = clock64(); } while (0)
#define PTRACEJ(j, i) do { if ((j) == 5) PTRACE(i); } while (0)
#else
#define PTRACE(i) do { } while (0)
#define PTRACEJ(j, i) do { } while (0)
#endif

// Coalesced staging of 256-row chunks of the panel through shared memory (row stride
// 18 doubles = 144 B: 16-byte aligned and conflict-free for per-thread 128-bit row access).
constexpr int STG_STRIDE = 18;

template <typename T, int PW, int R, bool CLUSTER>
__global__ void __launch_bounds__(PANEL_T)
lu_panel_kernel(T *__restrict__ P, long long lda, int m, int w, int CS, int k0, int *__restrict__ mv,
                T *__restrict__ diag, int cb, int ce, int *__restrict__ perm) {
    pdl_trigger();
    pdl_wait();
    constexpr int RW = PW * sizeof(T) / 8;  // row width in doubles (16)
    static_assert(RW == 16, "panel rows are 128 bytes");
    static_assert(PW % PANEL_UNROLL == 0, "PW must be a multiple of the unroll");
    extern __shared__ __align__(16) double stg[];  // R * PANEL_T rows x STG_STRIDE doubles
    __shared__ int sdst[R * PANEL_T];
    __shared__ unsigned long long wv[2][PANEL_W];
    __shared__ int wi[2][PANEL_W];
    __shared__ __align__(16) T wrow[2][PANEL_W][PW];  // each warp's candidate row (zero-padded)
    __shared__ T wip[2][PANEL_W];                     // and the reciprocal of its pivot value
    // cluster exchange (push model): slot [par][rank] written by CTA `rank`
    constexpr int CSMAX = CLUSTER ? 16 : 1;
    __shared__ unsigned long long rkey[2][CSMAX];
    __shared__ int ridx[2][CSMAX];
    __shared__ T rip[2][CSMAX];
    __shared__ __align__(16) T rrow[2][CSMAX][PW];
    __shared__ __align__(8) unsigned long long rbar[2];
    __shared__ int pivrows[PW];
    __shared__ T pvals[PW];
    __shared__ int vac[PW];
    __shared__ unsigned evm;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int crank = 0;
    if constexpr (CLUSTER) crank = (int)cg::this_cluster().block_rank();
    constexpr int RPC = R * PANEL_T;
    const int rbeg = crank * RPC;
    const long long ldd = lda * (long long)(sizeof(T) / 8);  // leading dim in doubles
    double *Pd = reinterpret_cast<double *>(P);
    const int wd = w * (int)(sizeof(T) / 8);                 // live doubles per row
    const bool vec = ((reinterpret_cast<uintptr_t>(Pd) & 15) == 0) && ((ldd & 1) == 0);

    if constexpr (CLUSTER) {
        if (tid == 0) {
            mbar_init(smem_u32(&rbar[0]), (unsigned)CS);
            mbar_init(smem_u32(&rbar[1]), (unsigned)CS);
            mbar_init_fence();
        }
        cg::this_cluster().sync();  // every CTA's barriers exist before anyone arrives on them
    }
    T *stgT = reinterpret_cast<T *>(stg);
    constexpr int STG_T = STG_STRIDE * 8 / (int)sizeof(T);  // row stride of the L buffer in T
    PTRACE(0);
    T a[R][PW];
    int grow[R], pidx[R];
    unsigned done = 0;
    // coalesced cp.async of all R*256 rows (8 threads per 128-byte row) into shared memory
#pragma unroll 4
    for (int idx = tid; idx < RPC * 8; idx += PANEL_T) {
        const int r = idx >> 3, c2 = (idx & 7) * 2;
        double *d = &stg[r * STG_STRIDE + c2];
        const int g = rbeg + r;
        if (vec && g < m && c2 + 1 < wd) {
            cp_async16(d, Pd + (long long)g * ldd + c2);
        } else if (g < m && c2 + 1 < wd) {
            d[0] = Pd[(long long)g * ldd + c2];
            d[1] = Pd[(long long)g * ldd + c2 + 1];
        } else {
            d[0] = (g < m && c2 < wd) ? Pd[(long long)g * ldd + c2] : 0.0;
            d[1] = 0.0;
        }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int q = 0; q < R; ++q) {
        grow[q] = rbeg + q * PANEL_T + tid;
        pidx[q] = -1;
        if (grow[q] >= m) done |= 1u << q;
        const double *row = &stg[(q * PANEL_T + tid) * STG_STRIDE];
        double t[16];
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
            const double2 v = *reinterpret_cast<const double2 *>(row + c);
            t[c] = v.x;
            t[c + 1] = v.y;
        }
#pragma unroll
        for (int c = 0; c < PW; ++c) {
            if constexpr (sizeof(T) == 8) a[q][c] = t[c];
            else a[q][c] = make_double2(t[2 * c], t[2 * c + 1]);
        }
    }
    PTRACE(1);

    // ---------------------------------------------------------------- column pipeline
    // publish(j, S): candidate of column j (current slot S) -- local argmax, warp argmax
    // (redux), candidate to wv/wi, the warp winner's row (zero-padded: rotated slot c is
    // live iff (c-S) mod PW < PW-j) and its reciprocal (computed speculatively by every
    // lane for its own candidate, overlapping the redux) to wrow[j&1][warp].
    // finish(j, S): barrier, block argmax (+ cluster argmax), pivot row, then the update
    // of the NEXT column's slot first, publish(j+1), and only then the other slots.
    int qb_next = 0;
    unsigned long long bv_next = 0;
    int bi_next = INT_MAX;
    T myip = zero_of(T());
    auto local_cand = [&](auto Sc) {
        constexpr int S = decltype(Sc)::value % PW;
        bv_next = 0;
        bi_next = INT_MAX;
        qb_next = 0;
        T myp = zero_of(T());
#pragma unroll
        for (int q = 0; q < R; ++q)
            if (!((done >> q) & 1u)) {
                const unsigned long long k = pkey_bits(a[q][S]);
                if (k > bv_next) { bv_next = k; bi_next = grow[q]; qb_next = q; myp = a[q][S]; }
            }
        // speculative reciprocal of this lane's candidate (used if it wins)
        if constexpr (sizeof(T) == 8) myip = is_zero(myp) ? zero_of(T()) : frcp(myp);
        else myip = is_zero(myp) ? zero_of(T()) : recip(myp);
    };
    auto publish = [&](const int j, auto Sc) {
        // Sc may be PANEL_UNROLL (first column after the next rotation): the row is then
        // stored already rotated so that it matches the frame the consumer will use.
        constexpr int V = decltype(Sc)::value;
        constexpr int K = (V >= PANEL_UNROLL) ? PANEL_UNROLL : 0;
        constexpr int SN = V - K;  // slot of column j after the rotation
        const int par = j & 1;
        const ArgMaxK wa = warp_argmax_key(bv_next, bi_next);
        if (lane == 0) { wv[par][warp] = wa.k; wi[par][warp] = wa.i; }
        if (bi_next == wa.i && bi_next != INT_MAX) {
#pragma unroll
            for (int q = 0; q < R; ++q)
                if (q == qb_next) {
                    T r[PW];
#pragma unroll
                    for (int c = 0; c < PW; ++c)
                        r[c] = a[q][(c + K) % PW];  // finished slots are already zero
                    store_row<T, PW>(wrow[par][warp], r);
                    wip[par][warp] = myip;
                }
        }
    };
    auto finish = [&](const int j, auto Sc) {
        constexpr int S = decltype(Sc)::value % PW;
        constexpr int S1 = (decltype(Sc)::value + 1) % PW;
        const int par = j & 1;
        PTRACEJ(j, 50);
        __syncthreads();
        PTRACEJ(j, 51);
        const ArgMaxK ca = warp_argmax_key(lane < PANEL_W ? wv[par][lane] : 0ull,
                                           lane < PANEL_W ? wi[par][lane] : INT_MAX);
        PTRACEJ(j, 52);
        const int cw = (ca.i == INT_MAX) ? 0 : ((ca.i - rbeg) % PANEL_T) >> 5;  // warp holding the CTA winner
        int gp;
        T u[PW];
        T ip;
        if constexpr (!CLUSTER) {
            gp = ca.i;
            load_row<T, PW>(u, wrow[par][cw]);
            ip = wip[par][cw];
        } else {
            // push the CTA winner (key, index, reciprocal, row) into every CTA of the cluster,
            // then one remote mbarrier arrive per target; wait on the local barrier
            if (warp == 0 && lane < CS) {
                const unsigned tgt = (unsigned)lane;
                const T *wr = wrow[par][cw];
                const unsigned rowa = mapa_u32(smem_u32(&rrow[par][crank][0]), tgt);
#pragma unroll
                for (int c = 0; c < PW; ++c) st_cluster(rowa + c * (unsigned)sizeof(T), wr[c]);
                st_cluster(mapa_u32(smem_u32(&rkey[par][crank]), tgt), ca.k);
                st_cluster(mapa_u32(smem_u32(&ridx[par][crank]), tgt), ca.i);
                st_cluster(mapa_u32(smem_u32(&rip[par][crank]), tgt), wip[par][cw]);
                mbar_remote_arrive(mapa_u32(smem_u32(&rbar[par]), tgt));
            }
            mbar_wait_parity(smem_u32(&rbar[par]), (unsigned)((j >> 1) & 1));
            const ArgMaxK ga = warp_argmax_key(lane < CS ? rkey[par][lane] : 0ull, lane < CS ? ridx[par][lane] : INT_MAX);
            gp = ga.i;
            const int owner = gp / RPC;
            load_row<T, PW>(u, rrow[par][owner]);
            ip = rip[par][owner];
        }
        const T piv = u[S];
        const bool zp = is_zero(piv);
        PTRACEJ(j, 53);
        if (tid == 0) { pivrows[j] = gp; pvals[j] = piv; }
        T l[R];
        bool act[R];
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const bool live = !((done >> q) & 1u);
            if (live && grow[q] == gp) { done |= 1u << q; pidx[q] = j; }
            act[q] = live && grow[q] != gp && !zp;
            l[q] = act[q] ? mul(a[q][S], ip) : a[q][S];
            if (act[q] && S1 != S) a[q][S1] = msub(a[q][S1], l[q], u[S1]);
        }
        if (j + 1 < w) {
            local_cand(std::integral_constant<int, decltype(Sc)::value + 1>{});
        }
        PTRACEJ(j, 54);
#pragma unroll
        for (int q = 0; q < R; ++q) {
            if (act[q]) {
#pragma unroll
                for (int c = 0; c < PW; ++c)
                    if (c != S && c != S1) a[q][c] = msub(a[q][c], l[q], u[c]);
            }
            // multiplier of a live non-pivot row -> L buffer; its register slot becomes 0 so a
            // published pivot row never carries finished columns (no masking needed)
            if (!((done >> q) & 1u)) {
                stgT[(q * PANEL_T + tid) * STG_T + j] = l[q];
                a[q][S] = zero_of(T());
            }
        }
        PTRACEJ(j, 55);
        if (j + 1 < w) publish(j + 1, std::integral_constant<int, decltype(Sc)::value + 1>{});
        PTRACE(2 + j);
    };
    auto rotate = [&](auto Kc) {
        constexpr int K = decltype(Kc)::value;
#pragma unroll
        for (int q = 0; q < R; ++q) {
            T t[PW];
#pragma unroll
            for (int c = 0; c < PW; ++c) t[c] = a[q][(c + K) % PW];
#pragma unroll
            for (int c = 0; c < PW; ++c) a[q][c] = t[c];
        }
    };

    local_cand(std::integral_constant<int, 0>{});
    publish(0, std::integral_constant<int, 0>{});
    int j = 0;
#pragma unroll 1
    for (; j + PANEL_UNROLL <= w; j += PANEL_UNROLL) {
        finish(j + 0, std::integral_constant<int, 0>{});
        finish(j + 1, std::integral_constant<int, 1>{});
        finish(j + 2, std::integral_constant<int, 2>{});
        finish(j + 3, std::integral_constant<int, 3>{});
        rotate(std::integral_constant<int, PANEL_UNROLL>{});
    }
    // tail (w % 4 columns, last panel only), then restore the original slot order
    const int jt = j;
    if (j < w) { finish(j, std::integral_constant<int, 0>{}); ++j; }
    if (j < w) { finish(j, std::integral_constant<int, 1>{}); ++j; }
    if (j < w) { finish(j, std::integral_constant<int, 2>{}); ++j; }
    const int rem = (PW - jt) % PW;  // slots still to rotate so that slot c holds column c
#pragma unroll 1
    for (int r = 0; r < rem; ++r) rotate(std::integral_constant<int, 1>{});
    __syncthreads();
    PTRACE(40);

    // final positions: pivot j -> row j; evicted rows (< w, not pivots) fill the rows
    // vacated by pivots that came from below (>= w), in pivot order.
    if (warp == 0) {
        bool rp = false;
        if (lane < w)
            for (int q = 0; q < w; ++q) rp |= (pivrows[q] == lane);
        const unsigned pivmask = __ballot_sync(0xffffffffu, rp);
        const unsigned wmask = (w >= 32) ? 0xffffffffu : ((1u << w) - 1u);
        const unsigned evmask = wmask & ~pivmask;
        const int gpj = lane < w ? pivrows[lane] : -1;
        const bool isv = lane < w && gpj >= w;
        const unsigned vb = __ballot_sync(0xffffffffu, isv);
        if (isv) vac[__popc(vb & ((1u << lane) - 1u))] = gpj;
        if (lane == 0) evm = evmask;
        __syncwarp();
        if (crank == 0) {
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
                mv[1 + q] = k0 + vac[__popc(evmask & ((1u << lane) - 1u))];
                mv[1 + 2 * PW_MAX + q] = k0 + lane;
            }
            if (lane == 0) mv[0] = nm + __popc(evmask);
            if (lane < w) diag[k0 + lane] = pvals[lane];
        }
    }
    __syncthreads();
    // write back through the staging buffer, coalesced, each row to its final position
#pragma unroll
    for (int q = 0; q < R; ++q) {
        const int g = grow[q];
        int dst = g;
        if (pidx[q] >= 0) dst = pidx[q];
        else if (g < w) dst = vac[__popc(evm & ((1u << g) - 1u))];
        sdst[q * PANEL_T + tid] = (g < m) ? dst : -1;
        // columns before the row's pivot step hold L multipliers (already in the buffer);
        // a pivot row keeps its U part (columns >= its step) in registers
        const int jp = (pidx[q] >= 0) ? pidx[q] : PW;
        T *row = stgT + (q * PANEL_T + tid) * STG_T;
#pragma unroll
        for (int c = 0; c < PW; ++c)
            if (c >= jp) row[c] = a[q][c];
    }
    __syncthreads();
#pragma unroll 4
    for (int idx = tid; idx < RPC * 8; idx += PANEL_T) {
        const int r = idx >> 3, c2 = (idx & 7) * 2;
        const int d = sdst[r];
        if (d < 0 || c2 >= wd) continue;
        double *out = Pd + (long long)d * ldd + c2;
        const double2 v = *reinterpret_cast<const double2 *>(&stg[r * STG_STRIDE + c2]);
        if (c2 + 1 < wd) {
            if (vec) *reinterpret_cast<double2 *>(out) = v;
            else { out[0] = v.x; out[1] = v.y; }
        } else {
            out[0] = v.x;
        }
    }
    PTRACE(41);
    // ---- fused: row movement of this panel + U12 = L11^{-1} A12 on the other columns of
    // the block [cb, ce) (the two-level LU's inner update), once every CTA's rows are back
    const int ncol = ce - cb - w;
    if (ncol > 0) {
        __shared__ T Ls[PW][PW + 1];
        __shared__ int srcr[PW], xdst[PW], xsrc[PW];
        __shared__ int nx_s;
        if constexpr (CLUSTER) cg::this_cluster().sync();  // release/acquire: the writeback is visible
        else __syncthreads();
        T *A = P - (long long)k0 * lda - k0;  // matrix origin
        if (tid == 0) {
            int nx = 0;
            for (int i = 0; i < w; ++i) srcr[i] = k0 + pivrows[i];
            for (int r = 0; r < w; ++r)
                if ((evm >> r) & 1u) {
                    xdst[nx] = k0 + vac[__popc(evm & ((1u << r) - 1u))];
                    xsrc[nx] = k0 + r;
                    ++nx;
                }
            nx_s = nx;
        }
        if (crank == 0 && warp == 0 && perm) {  // perm[dst] = perm[src] for the moved rows
            int d = -1, v = 0;
            if (lane < w && pivrows[lane] != lane) { d = k0 + lane; v = perm[k0 + pivrows[lane]]; }
            int d2 = -1, v2 = 0;
            if (lane < w && ((evm >> lane) & 1u)) {
                d2 = k0 + vac[__popc(evm & ((1u << lane) - 1u))];
                v2 = perm[k0 + lane];
            }
            __syncwarp();
            if (d >= 0) perm[d] = v;
            if (d2 >= 0) perm[d2] = v2;
        }
        for (int idx = tid; idx < w * w; idx += PANEL_T) {
            const int i = idx / w, q = idx - i * w;
            Ls[i][q] = A[(long long)(k0 + i) * lda + k0 + q];
        }
        __syncthreads();
        const int nx = nx_s;
        for (int v = crank * PANEL_T + tid; v < ncol; v += CS * PANEL_T) {
            const int c = (cb + v < k0) ? cb + v : cb + v + w;
            T x[PW], y[PW];
#pragma unroll
            for (int i = 0; i < PW; ++i) x[i] = (i < w) ? A[(long long)srcr[i] * lda + c] : zero_of(T());
#pragma unroll
            for (int i = 0; i < PW; ++i) y[i] = (i < nx) ? A[(long long)xsrc[i] * lda + c] : zero_of(T());
            if (c >= k0 + w) {
#pragma unroll
                for (int i = 1; i < PW; ++i) {
                    if (i < w) {
                        T acc = x[i];
#pragma unroll
                        for (int q = 0; q < i; ++q) acc = msub(acc, Ls[i][q], x[q]);
                        x[i] = acc;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < PW; ++i)
                if (i < w) A[(long long)(k0 + i) * lda + c] = x[i];
#pragma unroll
            for (int i = 0; i < PW; ++i)
                if (i < nx) A[(long long)xdst[i] * lda + c] = y[i];
        }
    }
    if constexpr (CLUSTER) cg::this_cluster().sync();  // no CTA leaves while its smem may still be read
}

// =====================================================================================
// Row movement on the other columns + U12 = L11^{-1} A12 (unit lower forward solve)
// =====================================================================================
constexpr int SWP_COLS = 32;

// One thread per column outside the panel.  Rows k0..k0+w-1 of column c are gathered
// straight from their source rows (srcrow), the other moved rows (evicted -> vacated)
// are copied; for c right of the panel the gathered top rows then get
// U12 = L11^{-1} A12 (unit lower forward substitution in registers).  Every load of a
// column is issued before its first store.
template <typename T, int PW>
__global__ void __launch_bounds__(SWP_COLS)
lu_swap_trsm_kernel(T *__restrict__ A, long long lda, int cb, int ce, int k0, int w, const int *__restrict__ mv,
                    int *__restrict__ perm) {
    pdl_trigger();
    pdl_wait();
    __shared__ T Ls[PW][PW + 1];
    __shared__ int srcrow[PW];
    __shared__ int xdst[PW], xsrc[PW];  // moves with destination outside the top w rows
    __shared__ int nx_s;
    __shared__ int ptmp[2 * PW];
    const int tid = threadIdx.x;
    const int cnt = mv[0];
    const int *dst = mv + 1, *src = mv + 1 + 2 * PW_MAX;
    if (tid == 0) {
        for (int i = 0; i < w; ++i) srcrow[i] = k0 + i;
        int nx = 0;
        for (int q = 0; q < cnt; ++q) {
            const int d = dst[q];
            if (d < k0 + w) srcrow[d - k0] = src[q];
            else { xdst[nx] = d; xsrc[nx] = src[q]; ++nx; }
        }
        nx_s = nx;
    }
    if (perm && blockIdx.x == 0) {
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
    if (v >= ce - cb - w) return;
    const int c = (cb + v < k0) ? cb + v : cb + v + w;
    const int nx = nx_s;
    T x[PW], y[PW];
#pragma unroll
    for (int i = 0; i < PW; ++i) x[i] = (i < w) ? A[(long long)srcrow[i] * lda + c] : zero_of(T());
#pragma unroll
    for (int i = 0; i < PW; ++i) y[i] = (i < nx) ? A[(long long)xsrc[i] * lda + c] : zero_of(T());
    if (c >= k0 + w) {
#pragma unroll
        for (int i = 1; i < PW; ++i) {
            if (i < w) {
                T acc = x[i];
#pragma unroll
                for (int q = 0; q < i; ++q) acc = msub(acc, Ls[i][q], x[q]);
                x[i] = acc;
            }
        }
    }
#pragma unroll
    for (int i = 0; i < PW; ++i)
        if (i < w) A[(long long)(k0 + i) * lda + c] = x[i];
#pragma unroll
    for (int i = 0; i < PW; ++i)
        if (i < nx) A[(long long)xdst[i] * lda + c] = y[i];
}

// Apply nlists consecutive panel row movements (lists at mv0 + l*MV_INTS) to the columns
// [ca0, ca1) and [cb0, cb1): one thread per column, lists in order, every load of a list
// before its stores.
constexpr int SWM_COLS = 64;
template <typename T, int PW>
__global__ void __launch_bounds__(SWM_COLS)
lu_swap_multi_kernel(T *__restrict__ A, long long lda, int ca0, int ca1, int cb0, int cb1,
                     const int *__restrict__ mv0, int nlists) {
    pdl_trigger();
    pdl_wait();
    const int v = blockIdx.x * SWM_COLS + threadIdx.x;
    const int na = ca1 - ca0;
    if (v >= na + (cb1 - cb0)) return;
    const int c = (v < na) ? ca0 + v : cb0 + (v - na);
    for (int l = 0; l < nlists; ++l) {
        const int *mv = mv0 + (long long)l * MV_INTS;
        const int cnt = mv[0];
        const int *dst = mv + 1, *src = mv + 1 + 2 * PW_MAX;
        T val[2 * PW];
#pragma unroll
        for (int q = 0; q < 2 * PW; ++q)
            if (q < cnt) val[q] = A[(long long)src[q] * lda + c];
#pragma unroll
        for (int q = 0; q < 2 * PW; ++q)
            if (q < cnt) A[(long long)dst[q] * lda + c] = val[q];
    }
}

template <typename T>
__global__ void copy_block_kernel(const T *__restrict__ src, long long lds, T *__restrict__ dst, long long ldd,
                                  int rows, int cols) {
    pdl_trigger();
    pdl_wait();
    const long long total = (long long)rows * cols;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / cols), j = (int)(idx - (long long)i * cols);
        dst[(long long)i * ldd + j] = src[(long long)i * lds + j];
    }
}

// Linv = (unit lower triangle of the W x W block at L, ld) extracted with unit diagonal
template <typename T>
__global__ void extract_unit_lower_kernel(const T *__restrict__ L, long long ld, int W, T *__restrict__ Li,
                                          long long ldi) {
    pdl_trigger();
    pdl_wait();
    const long long total = (long long)W * W;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / W), j = (int)(idx - (long long)i * W);
        Li[(long long)i * ldi + j] = (j < i) ? L[(long long)i * ld + j] : ((i == j) ? one_of(T()) : zero_of(T()));
    }
}

// =====================================================================================
// Pivot diagnostics (reading R2): rho, singular column, non-finite
// =====================================================================================
template <typename T>
__global__ void __launch_bounds__(1024) lu_stats_kernel(const T *__restrict__ diag, int n, LuStats *st) {
    pdl_trigger();
    pdl_wait();
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
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

// =====================================================================================
// getrf driver
// =====================================================================================
// panel width: 16 real / 8 complex columns (16 doubles per row in registers)
template <typename T> struct PanelW { static constexpr int PW = 16; };
template <> struct PanelW<double2> { static constexpr int PW = 8; };
constexpr int PANEL_MAX_CS = 16;

template <typename T, int PW, int R>
static cudaError_t launch_panel_r(T *P, long long lda, int m, int w, int k0, int *mv, T *diag, int CS,
                                  cudaStream_t s, int cb = 0, int ce = 0, int *perm = nullptr) {
    const size_t smem = (size_t)R * PANEL_T * STG_STRIDE * sizeof(double);
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_set[dev]) {
        cudaError_t e = cudaFuncSetAttribute(lu_panel_kernel<T, PW, R, false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(lu_panel_kernel<T, PW, R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(lu_panel_kernel<T, PW, R, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr_set[dev] = true;
    }
    double wk = 0.0;
    for (int j = 0; j < w; ++j) wk += (double)(m - j - 1) * (1.0 + 2.0 * (w - j - 1));
    ProfScope ps(sizeof(T) == 8 ? "lu_panel<double>" : "lu_panel<double2>", s, wk * (sizeof(T) == 8 ? 1.0 : 4.0));
    if (CS == 1) {
        return launch_pdl(lu_panel_kernel<T, PW, R, false>, dim3(1), dim3(PANEL_T), smem, s, P, lda, m, w, 1, k0,
                          mv, diag, cb, ce, perm);
    }
    auto kern = lu_panel_kernel<T, PW, R, true>;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[2];
    cfg.gridDim = dim3(CS, 1, 1);
    cfg.blockDim = dim3(PANEL_T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    count_launch();
    return cudaLaunchKernelEx(&cfg, kern, P, lda, m, w, CS, k0, mv, diag, cb, ce, perm);
}

template <typename T, int PW>
static cudaError_t launch_panel(T *P, long long lda, int m, int w, int k0, int *mv, T *diag, cudaStream_t s,
                                int cb = 0, int ce = 0, int *perm = nullptr) {
    // single CTA up to 1024 rows; beyond, a cluster with as few rows per CTA as 16 CTAs allow
    // (the push-model exchange makes more, lighter CTAs cheaper per column)
    if (m <= PANEL_T) return launch_panel_r<T, PW, 1>(P, lda, m, w, k0, mv, diag, 1, s, cb, ce, perm);
    if (m <= 2 * PANEL_T) return launch_panel_r<T, PW, 2>(P, lda, m, w, k0, mv, diag, 1, s, cb, ce, perm);
    if (m <= 4 * PANEL_T) return launch_panel_r<T, PW, 4>(P, lda, m, w, k0, mv, diag, 1, s, cb, ce, perm);
    if (m <= 16 * PANEL_T) return launch_panel_r<T, PW, 1>(P, lda, m, w, k0, mv, diag, (m + PANEL_T - 1) / PANEL_T, s, cb, ce, perm);
    if (m <= 32 * PANEL_T)
        return launch_panel_r<T, PW, 2>(P, lda, m, w, k0, mv, diag, (m + 2 * PANEL_T - 1) / (2 * PANEL_T), s, cb, ce, perm);
    return launch_panel_r<T, PW, 4>(P, lda, m, w, k0, mv, diag, (m + 4 * PANEL_T - 1) / (4 * PANEL_T), s, cb, ce, perm);
}

// =====================================================================================
// Triangular inverses: U^{-1} (non-unit upper) and L^{-1} (unit lower)
// =====================================================================================
constexpr int TRI_LEAF = 32;

// U = triu(lu) (zeros below), L = tril(lu, -1) + I (zeros above)
template <typename T>
__global__ void extract_ul_kernel(const T *__restrict__ lu, long long ld, int n, T *__restrict__ U,
                                  T *__restrict__ L, int r0, int r1) {  // rows [r0, r1)
    const long long total = (long long)(r1 - r0) * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = r0 + (int)(idx / n), j = (int)(idx % n);
        const T v = lu[(long long)i * ld + j];
        const T z = zero_of(T());
        U[(long long)i * ld + j] = (j >= i) ? v : z;
        L[(long long)i * ld + j] = (j < i) ? v : ((j == i) ? one_of(T()) : z);
    }
}

template <typename T>
cudaError_t extract_ul(int n, const T *lu, long long ld, T *U, T *L, cudaStream_t s) {
    const long long total = (long long)n * n;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    count_launch();
    extract_ul_kernel<T><<<blocks, 256, 0, s>>>(lu, ld, n, U, L, 0, n);
    return cudaGetLastError();
}
template cudaError_t extract_ul<double>(int, const double *, long long, double *, double *, cudaStream_t);
template cudaError_t extract_ul<double2>(int, const double2 *, long long, double2 *, double2 *, cudaStream_t);

// blockIdx.y == 0: invert upper diagonal blocks of U in place; == 1: unit-lower blocks of L.
// One thread per row of U^{-1} (column of L^{-1}); the recurrences are evaluated "right-looking":
// once X[i][k] is known it is added into the accumulators of every later entry (independent
// FMAs in registers) instead of each entry re-reading a dependent dot product, with the same
// terms in the same order (k increasing): bit-identical to the dot-product form for real T (a
// complex product's mul/add pairs may contract to FMAs differently: ~1e-14 relative).
template <typename T>
__global__ void __launch_bounds__(TRI_LEAF) tri_leaf_kernel(T *__restrict__ U, T *__restrict__ L,
                                                            long long ld, int n, int lower_only = 0) {
    pdl_trigger();
    pdl_wait();
    __shared__ T S[TRI_LEAF][TRI_LEAF + 1];
    __shared__ T X[TRI_LEAF][TRI_LEAF + 1];
    __shared__ T R[TRI_LEAF];
    const int b0 = blockIdx.x * TRI_LEAF;
    const int sz = min(TRI_LEAF, n - b0);
    const bool upper = (blockIdx.y == 0) && !lower_only;
    T *M = upper ? U : L;
    const int tid = threadIdx.x;
    const T z = zero_of(T());
    for (int i = 0; i < TRI_LEAF; ++i) S[i][tid] = (i < sz && tid < sz) ? M[(long long)(b0 + i) * ld + b0 + tid] : z;
    __syncthreads();
    R[tid] = (upper && tid < sz) ? recip(S[tid][tid]) : z;
    __syncthreads();
    T acc[TRI_LEAF];
#pragma unroll
    for (int j = 0; j < TRI_LEAF; ++j) acc[j] = z;
    if (upper) {
        // row i = tid of U^{-1}: X[i][i] = 1/u_ii; X[i][j] = -(sum_{k=i}^{j-1} X[i][k] u_kj)/u_jj
        const int i = tid;
#pragma unroll
        for (int k = 0; k < TRI_LEAF; ++k) {
            T xk = z;
            if (k == i) xk = R[k];
            else if (k > i) xk = neg(mul(acc[k], R[k]));
            X[i][k] = xk;
            if (k >= i) {
#pragma unroll
                for (int j = k + 1; j < TRI_LEAF; ++j) acc[j] = madd(acc[j], xk, S[k][j]);
            }
        }
    } else {
        // column j = tid of L^{-1}: Y[j][j] = 1; Y[i][j] = -sum_{k=j}^{i-1} l_ik Y[k][j]
        const int j = tid;
#pragma unroll
        for (int k = 0; k < TRI_LEAF; ++k) {
            T yk = z;
            if (k == j) yk = one_of(T());
            else if (k > j) yk = neg(acc[k]);
            X[k][j] = yk;
            if (k >= j) {
#pragma unroll
                for (int i = k + 1; i < TRI_LEAF; ++i) acc[i] = madd(acc[i], S[i][k], yk);
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
                             cudaStream_t st, bool do_upper = true, bool do_lower = true) {
    const long long stride = 2LL * s * (ld + 1);
    cudaError_t e;
#ifdef FROB_TUNING  // per-level profiler tags (tools/profile_n.py), tuning builds only
    static const char *lvl[] = {"gemm:tri_inv_s32", "gemm:tri_inv_s64", "gemm:tri_inv_s128", "gemm:tri_inv_s256",
                                "gemm:tri_inv_s512", "gemm:tri_inv_s1024", "gemm:tri_inv_s2048", "gemm:tri_inv_s4096",
                                "gemm:tri_inv_s8192"};
    int li = 0;
    while ((32 << li) < s && li < 8) ++li;
    GemmTag ltag(g_gemm_tag && std::string(g_gemm_tag) == "gemm:tri_inv" ? lvl[li] : g_gemm_tag);
#endif
    // step 1 -- upper: W = U12 * inv(U22);  lower: W = L21 * inv(L11)   (one launch)
    auto pu = gemm_params<T>(s, s2, s2, 1.0, U + (long long)o * ld + o + s, ld,
                             U + (long long)(o + s) * ld + o + s, ld, 0.0, nullptr, ld,
                             tmp + (long long)o * ld + o + s, ld);
    pu.triB = TRI_UPPER; pu.sA = pu.sB = pu.sC = stride; pu.sD = 0;
    auto pl = gemm_params<T>(s2, s, s, 1.0, L + (long long)(o + s) * ld + o, ld,
                             L + (long long)o * ld + o, ld, 0.0, nullptr, ld,
                             tmp + (long long)(o + s) * ld + o, ld);
    pl.triB = TRI_LOWER; pl.sA = pl.sB = pl.sC = stride; pl.sD = 0;
    if (!do_lower) {
        if ((e = gemm_launch<T>(pu, batch, st)) != cudaSuccess) return e;
    } else if ((e = gemm_launch2<T>(pl, batch, pu, do_upper ? batch : 0, st)) != cudaSuccess) {
        return e;
    }
    // step 2 -- upper: U12 <- -inv(U11) * W;  lower: L21 <- -inv(L22) * W
    auto qu = gemm_params<T>(s, s2, s, -1.0, U + (long long)o * ld + o, ld,
                             tmp + (long long)o * ld + o + s, ld, 0.0, nullptr, ld,
                             U + (long long)o * ld + o + s, ld);
    qu.triA = TRI_UPPER; qu.sA = qu.sB = qu.sC = stride; qu.sD = 0;
    auto ql = gemm_params<T>(s2, s, s2, -1.0, L + (long long)(o + s) * ld + o + s, ld,
                             tmp + (long long)(o + s) * ld + o, ld, 0.0, nullptr, ld,
                             L + (long long)(o + s) * ld + o, ld);
    ql.triA = TRI_LOWER; ql.sA = ql.sB = ql.sC = stride; ql.sD = 0;
    if (!do_lower) return gemm_launch<T>(qu, batch, st);
    return gemm_launch2<T>(ql, batch, qu, do_upper ? batch : 0, st);
}

template <typename T>
cudaError_t inv_from_lu(int n, T *lu, long long ld, T *U, T *L, T *out, long long ldo,
                        const int *colperm, int *counter, cudaStream_t s, EarlyInv *early) {
    cudaError_t e;
    // (EarlyInv from getrf: the first h rows of U and L are in place already)
    const int r0 = (early && early->ready) ? early->h : 0;
    {
        long long total = (long long)(n - r0) * n;
        long long nb = (total + 255) / 256; int blocks = (int)(nb < 148LL * 16 ? nb : 148LL * 16);
        count_launch();
        extract_ul_kernel<T><<<blocks, 256, 0, s>>>(lu, ld, n, U, L, r0, n);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    return inv_from_ul<T>(n, U, L, ld, lu, out, ldo, colperm, counter, s, early);  // the LU factors are scratch now
}

// U <- U^{-1}, L <- L^{-1} in place (32 x 32 diagonal inverses + log-depth recursion)
template <typename T>
cudaError_t tri_inverses(int n, T *U, T *L, long long ld, T *tmp, cudaStream_t s) {
    cudaError_t e;
    GemmTag tag("gemm:tri_inv");
    const bool lower = L != nullptr;  // L == nullptr: invert the upper triangle U only
    if ((e = launch_pdl(tri_leaf_kernel<T>, dim3((n + TRI_LEAF - 1) / TRI_LEAF, lower ? 2 : 1), dim3(TRI_LEAF), 0, s,
                        U, lower ? L : U, ld, n, 0)) != cudaSuccess)
        return e;
    for (int sz = TRI_LEAF; sz < n; sz *= 2) {
        const int full = n / (2 * sz);
        if (full > 0 && (e = tri_level<T>(U, lower ? L : U, tmp, ld, sz, 0, sz, full, s, true, lower)) != cudaSuccess)
            return e;
        const int o = full * 2 * sz;
        if (o + sz < n) {
            if ((e = tri_level<T>(U, lower ? L : U, tmp, ld, sz, o, n - o - sz, 1, s, true, lower)) != cudaSuccess)
                return e;
        }
    }
    return cudaSuccess;
}
template cudaError_t tri_inverses<double>(int, double *, double *, long long, double *, cudaStream_t);
template cudaError_t tri_inverses<double2>(int, double2 *, double2 *, long long, double2 *, cudaStream_t);

// out[i][c] = Wp[pos_h[perm[h + i]] - h][c]: EarlyInv's W' rows in the final order (i < n - h, c < h)
// (getrf's EarlyInv: out[i][c] = Wp[wmap[i]][c])
template <typename T>
__global__ void gather_w_kernel(const T *__restrict__ Wp, long long ld, const int *__restrict__ perm,
                                const int *__restrict__ pos_h, const int *__restrict__ wmap, int n, int h,
                                T *__restrict__ out, long long ldo) {
    const long long total = (long long)(n - h) * h;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / h), c = (int)(idx % h);
        const int src = wmap ? wmap[i] : pos_h[perm[h + i]] - h;
        out[(long long)i * ldo + c] = Wp[(long long)src * ld + c];
    }
}

template <typename T>
cudaError_t inv_from_ul(int n, T *U, T *L, long long ld, T *tmp, T *out, long long ldo, const int *colperm,
                        int *counter, cudaStream_t s, EarlyInv *early) {
    cudaError_t e;
    if (early && early->h > 0 && early->done) {
        // U11^{-1}, L11^{-1} and V = U11^{-1} U12 came from lu2_factor's auxiliary stream (EarlyInv)
        const int h = early->h, r = n - h;
        EV_TRACE(20, 0, s);
        e = cudaStreamWaitEvent(s, early->done, 0);
        cudaEventDestroy(early->done);  // released once the recorded work completes
        early->done = nullptr;
        if (e != cudaSuccess) return e;
        T *U22 = U + (long long)h * ld + h, *L22 = L + (long long)h * ld + h;
        EV_TRACE(21, 0, s);
        if ((e = tri_inverses<T>(r, U22, L22, ld, tmp + (long long)h * ld + h, s)) != cudaSuccess) return e;
        EV_TRACE(22, 0, s);
        GemmTag tag("gemm:tri_inv");
        const T *V = reinterpret_cast<const T *>(early->vbuf) + h;
        // W = L21 L11^{-1} in the final row order: W'[pos_h(perm[i]) - h] (into tmp rows [h, n), columns [0, h))
        {
            const long long total = (long long)r * h;
            count_launch();
            gather_w_kernel<T><<<(int)std::min<long long>((total + 255) / 256, 148LL * 8), 256, 0, s>>>(
                reinterpret_cast<const T *>(early->vbuf) + (long long)h * ld + h, ld, early->perm, early->pos_h,
                early->wmap, n, h, tmp + (long long)h * ld, ld);
            if ((e = cudaGetLastError()) != cudaSuccess) return e;
        }
        // U12 <- -V U22^{-1}  and  L21 <- -L22^{-1} W: one launch
        auto pu = gemm_params<T>(h, r, r, -1.0, V, ld, U22, ld, 0.0, nullptr, ld, U + h, ld);
        pu.triB = TRI_UPPER;
        auto ql = gemm_params<T>(r, h, r, -1.0, L22, ld, tmp + (long long)h * ld, ld, 0.0, nullptr, ld,
                                 L + (long long)h * ld, ld);
        ql.triA = TRI_LOWER;
        if ((e = gemm_launch2<T>(ql, 1, pu, 1, s)) != cudaSuccess) return e;
        EV_TRACE(23, 0, s);
    } else {
        EV_TRACE(20, 1, s);
        if ((e = tri_inverses<T>(n, U, L, ld, tmp, s)) != cudaSuccess) return e;
        EV_TRACE(23, 1, s);
    }
    if (early && early->ready && early->h > 0) {
        // X = U^{-1} L^{-1} by blocks, P11 = U11^{-1} L11^{-1} formed early (EarlyInv, vbuf's top-left):
        //   X11 = U12' L21' + P11,  X12 = U12' L22',  X21 = U22' L21',  X22 = U22' L22'
        const int h = early->h, r = n - h;
        const T *P11 = reinterpret_cast<const T *>(early->vbuf);
        const T *U12 = U + h, *U22 = U + (long long)h * ld + h, *L21 = L + (long long)h * ld,
                *L22 = L + (long long)h * ld + h;
        T *o21 = out + (long long)h * ldo;
        auto blk = [&](int M, int N, int K, const T *A, const T *B, const T *D, T *Cb, int col0, int ta, int tb) {
            auto q = gemm_params<T>(M, N, K, 1.0, A, ld, B, ld, D ? 1.0 : 0.0, D, ld, colperm ? Cb : Cb + col0, ldo);
            q.colperm = colperm ? colperm + col0 : nullptr;
            q.triA = ta;
            q.triB = tb;
            return q;
        };
        GemmTag tag("gemm:product");
        const auto x11 = blk(h, h, r, U12, L21, P11, out, 0, TRI_NONE, TRI_NONE);
        const auto x22 = blk(r, r, r, U22, L22, nullptr, o21, h, TRI_UPPER, TRI_LOWER);
        if ((e = gemm_launch2<T>(x11, 1, x22, 1, s)) != cudaSuccess) return e;
        const auto x12 = blk(h, r, r, U12, L22, nullptr, out, h, TRI_NONE, TRI_LOWER);
        const auto x21 = blk(r, h, r, U22, L21, nullptr, o21, 0, TRI_UPPER, TRI_NONE);
        e = gemm_launch2<T>(x12, 1, x21, 1, s);
        early->ready = false;
        EV_TRACE(24, 0, s);
        return e;
    }
    // X = U^{-1} L^{-1}: (upper) x (lower) -> k from max(row0, col0)
    auto p = gemm_params<T>(n, n, n, 1.0, U, ld, L, ld, 0.0, nullptr, ld, out, ldo);
    p.triA = TRI_UPPER;
    p.triB = TRI_LOWER;
    p.colperm = colperm;
    // persistent CTAs, longest k-range first (tile (0,0) has k = 0..n): only when the tile
    // count is comparable to the resident CTAs; larger products balance by themselves
    // product schedule: n <= 1024 split-K (the 1024-long k-range of the corner tile dominates
    // otherwise; measured 236 -> 220 us real, 597 -> 529 us complex at n = 1024), n <= 2048
    // persistent longest-first CTAs, beyond a plain grid (env FROB_PRODUCT=0/1 forces one)
    static int prod_mode = [] {
        const char *v = tuning_env("FROB_PRODUCT");
        return v ? atoi(v) : -1;
    }();
    const int mode = prod_mode >= 0 ? prod_mode : (n <= 1024 ? 1 : 0);
    p.counter = (n <= 2048 && mode == 0) ? counter : nullptr;
    if (mode == 1) p.force_split = 1;
    GemmTag tag("gemm:product");
    e = gemm_launch<T>(p, 1, s);
    EV_TRACE(24, 0, s);
    return e;
}
template cudaError_t inv_from_ul<double>(int, double *, double *, long long, double *, double *, long long, const int *, int *, cudaStream_t, EarlyInv *);
template cudaError_t inv_from_ul<double2>(int, double2 *, double2 *, long long, double2 *, double2 *, long long, const int *, int *, cudaStream_t, EarlyInv *);

template <typename T>
cudaError_t lu_stats_launch(const T *diag, int n, LuStats *st, cudaStream_t s) {
    return launch_pdl(lu_stats_kernel<T>, dim3(1), dim3(1024), 0, s, diag, n, st);
}
template cudaError_t lu_stats_launch<double>(const double *, int, LuStats *, cudaStream_t);
template cudaError_t lu_stats_launch<double2>(const double2 *, int, LuStats *, cudaStream_t);

template cudaError_t inv_from_lu<double>(int, double *, long long, double *, double *, double *, long long, const int *, int *, cudaStream_t, EarlyInv *);
template cudaError_t inv_from_lu<double2>(int, double2 *, long long, double2 *, double2 *, double2 *, long long, const int *, int *, cudaStream_t, EarlyInv *);


// =====================================================================================
// getrf: two-level blocked right-looking LU with look-ahead
// =====================================================================================
// Outer blocks of LuNB<T>::N columns; inside a block, PW-column register panels with narrow
// swap/TRSM/GEMM updates restricted to the block.  After a block, its row movements,
// U12 = L11^{-1} A12 (L11^{-1} by the triangular recursion, so the TRSM is a K = LuNB
// GEMM) and the K = LuNB trailing GEMM are applied: first to the NEXT block's columns on
// the caller's stream (look-ahead), and for all other columns on an internal auxiliary
// stream, where they overlap the next block's panel chain.
// below this order the single-level LU (full-width K = PW trailing updates) is faster
constexpr int LU_TWO_LEVEL_MIN = 2048;

struct AuxCtx {
    cudaStream_t st = nullptr;  // far-column updates, lowest priority
    cudaStream_t hi = nullptr;  // the panel chain, highest priority (its CTAs are dispatched first)
    cudaEvent_t ev[6];
    bool ok = false;
    std::mutex mu;
};
static AuxCtx &aux_ctx(cudaError_t &err) {
    static AuxCtx ctx[64];
    static std::mutex gmu;
    int dev = 0;
    cudaGetDevice(&dev);
    AuxCtx &c = ctx[dev & 63];
    std::lock_guard<std::mutex> g(gmu);
    err = cudaSuccess;
    if (!c.ok) {
        int least = 0, greatest = 0;
        err = cudaDeviceGetStreamPriorityRange(&least, &greatest);
        if (err == cudaSuccess) err = cudaStreamCreateWithPriority(&c.st, cudaStreamNonBlocking, least);
        if (err == cudaSuccess) err = cudaStreamCreateWithPriority(&c.hi, cudaStreamNonBlocking, greatest);
        for (auto &e : c.ev)
            if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        c.ok = (err == cudaSuccess);
    }
    return c;
}

static long long ld8(int n) { return ((long long)n + 7) / 8 * 8; }

// the real blocked LU hands its last trailing matrix (m <= LU2_MAX_N rows) to lu2: two compact
// m x m ping-pong buffers + lu2's ints + the sub-permutation (n = 8192 LU 26.3 -> 23.6 ms; for
// complex matrices lu2's 8-column steps at m = 4096 are slower than the blocked steps: not used)
template <typename T> struct GetrfTail { static constexpr bool on = sizeof(T) == 8; };
static size_t getrf_tail_m(int n) { return (size_t)std::min(n, LU2_MAX_N); }
template <typename T>
static size_t getrf_tail_elems(int n) {
    if (!GetrfTail<T>::on) return 0;
    const size_t m = getrf_tail_m(n), ints = lu2_int_elems((int)m) + 2 * m;
    return 2 * m * (size_t)ld8((int)m) + (ints * sizeof(int) + sizeof(T) - 1) / sizeof(T) + 64;
}
template <typename T>
size_t getrf_work_elems(int n) {
    if (n <= LuNB<T>::N) return 1;
    return 3 * (size_t)LuNB<T>::N * LuNB<T>::N + 2 * (size_t)LuNB<T>::N * ld8(n) + getrf_tail_elems<T>(n);
}
template size_t getrf_work_elems<double>(int);
template size_t getrf_work_elems<double2>(int);

size_t lu_mv_ints(int n) { return ((size_t)(n + 7) / 8 + 1) * MV_INTS; }

static int ew_grid(long long total) {
    long long nb = (total + 255) / 256;
    return (int)(nb < 148LL * 8 ? nb : 148LL * 8);
}

// rows [r0, r0 + m) of columns [c0, c0 + nc) gathered by a row permutation: dst[i][j] = A[r0 + p[i]][c0 + j]
template <typename T>
__global__ void gather_rows_kernel(const T *__restrict__ A, long long lda, int r0, int c0, int m, int nc,
                                   const int *__restrict__ p, T *__restrict__ dst, long long ldd) {
    pdl_trigger();
    pdl_wait();
    const long long total = (long long)m * nc;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx / nc), j = (int)(idx - (long long)i * nc);
        dst[(long long)i * ldd + j] = A[(long long)(r0 + p[i]) * lda + c0 + j];
    }
}
// perm[r0 + i] = perm[r0 + p[i]] (through tmp)
__global__ void perm_gather_kernel(int *__restrict__ perm, int r0, int m, const int *__restrict__ p,
                                   int *__restrict__ tmp, int phase) {
    pdl_trigger();
    pdl_wait();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        if (phase == 0) tmp[i] = perm[r0 + p[i]];
        else perm[r0 + i] = tmp[i];
    }
}

// one panel step restricted to the column range [cb, ce) (the panel lies inside it)
template <typename T, int PW>
static cudaError_t panel_step(int n, T *A, long long lda, int cb, int ce, int k0, int *perm, int *list, T *diag,
                              cudaStream_t s) {
    cudaError_t e;
    const int w = min(PW, ce - k0), m = n - k0;
    const bool fused = (ce - cb) <= LuNB<T>::N;  // inner step of the two-level LU: swap+TRSM fused into the panel
    if ((e = launch_panel<T, PW>(A + (long long)k0 * lda + k0, lda, m, w, k0, list, diag, s, fused ? cb : 0,
                                 fused ? ce : 0, fused ? perm : nullptr)) != cudaSuccess)
        return e;
    const int ncols = ce - cb - w;
    if (!fused || ncols <= 0) {
        ProfScope ps(sizeof(T) == 8 ? "lu_swap_trsm<double>" : "lu_swap_trsm<double2>", s);
        if ((e = launch_pdl(lu_swap_trsm_kernel<T, PW>, dim3(max(1, (ncols + SWP_COLS - 1) / SWP_COLS)),
                            dim3(SWP_COLS), 0, s, A, lda, cb, ce, k0, w, list, perm)) != cudaSuccess)
            return e;
    }
    const int rest = ce - k0 - w;
    if (rest > 0 && m - w > 0) {
        T *a21 = A + (long long)(k0 + w) * lda + k0;
        T *a12 = A + (long long)k0 * lda + k0 + w;
        T *a22 = A + (long long)(k0 + w) * lda + k0 + w;
        auto p = gemm_params<T>(m - w, rest, w, -1.0, a21, lda, a12, lda, 1.0, a22, lda, a22, lda);
        GemmTag tag("gemm:lu_inner");
        if ((e = gemm_launch<T>(p, 1, s)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// The same step with lu2's 32-column panel kernels (one CTA, or a cluster of <= 8 CTAs with a
// DSMEM pivot exchange) for m <= LU2_PANEL_MAX_M: panel in place, then row movement + TRSM on the
// other columns of [cb, ce) and the trailing GEMM inside [cb, ce).  Returns the width taken.
template <typename T>
static cudaError_t panel_step2(int n, T *A, long long lda, const CUtensorMap &tm, int cb, int ce, int k0, int *perm,
                               int *list, T *diag, cudaStream_t s, int &w) {
    constexpr int PW2 = Panel2W<T>::PW;
    cudaError_t e;
    w = min(PW2, ce - k0);
    const int m = n - k0;
    if ((e = lu2_panel_inplace<T>(tm, A, lda, n, k0, w, list, diag, s)) != cudaSuccess) return e;
    const int ncols = ce - cb - w;
    if (ncols > 0) {
        ProfScope ps(sizeof(T) == 8 ? "lu_swap_trsm<double>" : "lu_swap_trsm<double2>", s);
        if ((e = launch_pdl(lu_swap_trsm_kernel<T, PW2>, dim3((ncols + SWP_COLS - 1) / SWP_COLS), dim3(SWP_COLS), 0, s,
                            A, lda, cb, ce, k0, w, (const int *)list, perm)) != cudaSuccess)
            return e;
    } else if (perm) {
        // no other columns: the permutation still has to follow the panel's moves
        if ((e = launch_pdl(lu_swap_trsm_kernel<T, PW2>, dim3(1), dim3(SWP_COLS), 0, s, A, lda, cb, ce, k0, w,
                            (const int *)list, perm)) != cudaSuccess)
            return e;
    }
    const int rest = ce - k0 - w;
    if (rest > 0 && m - w > 0) {
        T *a21 = A + (long long)(k0 + w) * lda + k0;
        T *a12 = A + (long long)k0 * lda + k0 + w;
        T *a22 = A + (long long)(k0 + w) * lda + k0 + w;
        auto p = gemm_params<T>(m - w, rest, w, -1.0, a21, lda, a12, lda, 1.0, a22, lda, a22, lda);
        GemmTag tag("gemm:lu_inner");
        if ((e = gemm_launch<T>(p, 1, s)) != cudaSuccess) return e;
    }
    return cudaSuccess;
}
// new panels unless env FROB_GETRF_PANEL=old (A/B measurement aid)
static bool getrf_new_panels() {
    static bool v = [] {
        const char *e = tuning_env("FROB_GETRF_PANEL");
        return !(e && e[0] == 'o');
    }();
    return v;
}

// Host-side event timeline of getrf (-DFROB_TL builds only; tools/getrf_timeline.py): timing
// events recorded on the chain and far-column streams at the points named by `kind`, read back
// as ms relative to the first one.  Events on two streams do not serialise the kernels.
#ifdef FROB_TL
static std::vector<std::pair<int, cudaEvent_t>> g_evt;
static std::mutex g_evt_mu;
void ev_trace(int kind, int t, cudaStream_t st) {
    std::lock_guard<std::mutex> g(g_evt_mu);
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, st);
    g_evt.emplace_back(kind * 100000 + t, e);
}
extern "C" int frob_evtrace_reset() {
    std::lock_guard<std::mutex> g(g_evt_mu);
    for (auto &p : g_evt) cudaEventDestroy(p.second);
    g_evt.clear();
    return 0;
}
extern "C" int frob_evtrace_read(int *codes, float *ms, int cap) {
    std::lock_guard<std::mutex> g(g_evt_mu);
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    const int cnt = (int)std::min<size_t>(g_evt.size(), (size_t)cap);
    for (int i = 0; i < cnt; ++i) {
        codes[i] = g_evt[i].first;
        if (cudaEventElapsedTime(&ms[i], g_evt[0].second, g_evt[i].second) != cudaSuccess) ms[i] = -1.f;
    }
    return cnt;
}
#endif

// outer update of columns [c0, c1) by block (K0, W): U12 = Linv * A12 -> Tb, A22 -= L21 * Tb, A12 <- Tb
template <typename T>
static cudaError_t outer_update(int n, T *A, long long lda, int K0, int W, int c0, int c1, const T *Linv, T *Tb,
                                long long ldT, cudaStream_t s) {
    cudaError_t e;
    const int nc = c1 - c0;
    if (nc <= 0) return cudaSuccess;
    GemmTag tag("gemm:lu_outer");
    auto p = gemm_params<T>(W, nc, W, 1.0, Linv, LuNB<T>::N, A + (long long)K0 * lda + c0, lda, 0.0, nullptr, ldT,
                            Tb + c0, ldT);
    p.triA = TRI_LOWER;
    if ((e = gemm_launch<T>(p, 1, s)) != cudaSuccess) return e;
    EV_TRACE(10, K0 / LuNB<T>::N + (c1 == n ? 0 : 50000), s);
    const int mr = n - K0 - W;
    if (mr > 0) {
        T *c = A + (long long)(K0 + W) * lda + c0;
        auto q = gemm_params<T>(mr, nc, W, -1.0, A + (long long)(K0 + W) * lda + K0, lda, Tb + c0, ldT, 1.0, c, lda,
                                c, lda);
        if ((e = gemm_launch<T>(q, 1, s)) != cudaSuccess) return e;
    }
    EV_TRACE(11, K0 / LuNB<T>::N + (c1 == n ? 0 : 50000), s);
    return launch_pdl(copy_block_kernel<T>, dim3(ew_grid((long long)W * nc)), dim3(256), 0, s, Tb + c0, ldT,
                      A + (long long)K0 * lda + c0, lda, W, nc);
}

// lu2 for the last trailing matrix unless env FROB_GETRF_TAIL=0 (A/B measurement aid)
static bool getrf_tail() {
    static bool v = [] {
        const char *e = tuning_env("FROB_GETRF_TAIL");
        return !(e && e[0] == '0');
    }();
    return v;
}

// chain / far-column stream priorities unless env FROB_LU_PRIO=0 (A/B measurement aid)
static bool getrf_prio() {
    static bool v = [] {
        const char *e = tuning_env("FROB_LU_PRIO");
        return !(e && e[0] == '0');
    }();
    return v;
}


template <typename T>
cudaError_t getrf(int n, T *A, long long lda, int *perm, int *mv, T *diag, LuStats *stats, T *work,
                  cudaStream_t s, EarlyInv *early) {
    constexpr int PW = PanelW<T>::PW, PW2 = Panel2W<T>::PW;
    cudaError_t e = launch_pdl(iota_kernel, dim3((n + 255) / 256), dim3(256), 0, s, perm, n);
    if (e != cudaSuccess) return e;
    // lu2's panels stage rows with TMA and 16-byte vector stores: 16-byte aligned rows only
    const bool np = getrf_new_panels() && ((lda * (long long)sizeof(T)) % 16 == 0) &&
                    ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    CUtensorMap tm;
    if (np) {
        const int E = (int)(sizeof(T) / 8);
        if ((e = tma_map_rows128(&tm, A, n, (long long)n * E, lda * E, 256)) != cudaSuccess) return e;
    }
    // one panel step at k0 inside [cb, ce); its move list goes to the next slot of mv
    int slot = 0;
    cudaStream_t cs = s;  // the panel chain's stream
    auto step = [&](int cb, int ce, int k0, int &w) -> cudaError_t {
        int *list = mv + (long long)slot * MV_INTS;
        ++slot;
        if (np && n - k0 <= lu2_panel_max_m()) return panel_step2<T>(n, A, lda, tm, cb, ce, k0, perm, list, diag, cs, w);
        w = min(PW, ce - k0);
        return panel_step<T, PW>(n, A, lda, cb, ce, k0, perm, list, diag, cs);
    };
    if (n < LU_TWO_LEVEL_MIN || !work) {
        for (int k0 = 0, w = 0; k0 < n; k0 += w)
            if ((e = step(0, n, k0, w)) != cudaSuccess) return e;
    } else {
        AuxCtx &ax = aux_ctx(e);
        if (e != cudaSuccess) return e;
        std::lock_guard<std::mutex> guard(ax.mu);
        const long long ldT = ld8(n);
        T *Linv[2] = {work, work + (size_t)LuNB<T>::N * LuNB<T>::N};
        T *tmp = work + 2 * (size_t)LuNB<T>::N * LuNB<T>::N;
        T *Tb[2] = {tmp + (size_t)LuNB<T>::N * LuNB<T>::N, tmp + (size_t)LuNB<T>::N * LuNB<T>::N + (size_t)LuNB<T>::N * ldT};
        cudaEvent_t evL = ax.ev[0], evR[2] = {ax.ev[1], ax.ev[2]}, evJ = ax.ev[3];
        // the chain (panels, L11^{-1}, look-ahead block) on a high-priority stream, the far
        // columns on a low-priority one: the chain's CTAs take the SMs the far-column GEMM frees
        // first instead of queueing behind its remaining tiles (env FROB_LU_PRIO=0: caller's stream)
        const bool prio = getrf_prio();
        if (prio) {
            if ((e = cudaEventRecord(ax.ev[4], s)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(ax.hi, ax.ev[4], 0)) != cudaSuccess) return e;
            cs = ax.hi;
        }
        int t = 0;
        int Ktail = n;  // the trailing matrix from here on goes to lu2
        for (int K0 = 0; K0 < n; K0 += LuNB<T>::N, ++t) {
            if (GetrfTail<T>::on && K0 > 0 && n - K0 <= lu2_max_n() && getrf_tail()) {
                Ktail = K0;
                break;
            }
            const int W = min(LuNB<T>::N, n - K0);
            const int slot0 = slot;
            EV_TRACE(0, t, cs);
            for (int k0 = K0, w = 0; k0 < K0 + W; k0 += w)
                if ((e = step(K0, K0 + W, k0, w)) != cudaSuccess) return e;
            const int cn0 = K0 + W, cn1 = min(n, K0 + 2 * W);
            const int nl = slot - slot0;
            const int *lists = mv + (long long)slot0 * MV_INTS;
            T *Li = Linv[t & 1];
            EV_TRACE(1, t, cs);
            if (cn0 < n) {
                // L11^{-1} (W x W unit lower) by the triangular recursion
                if ((e = launch_pdl(extract_unit_lower_kernel<T>, dim3(ew_grid((long long)W * W)), dim3(256), 0, cs,
                                    A + (long long)K0 * lda + K0, lda, W, Li, (long long)LuNB<T>::N)) != cudaSuccess)
                    return e;
                if ((e = launch_pdl(tri_leaf_kernel<T>, dim3((W + TRI_LEAF - 1) / TRI_LEAF, 1), dim3(TRI_LEAF), 0, cs,
                                    Li, Li, (long long)LuNB<T>::N, W, 1)) != cudaSuccess)
                    return e;
                GemmTag tag("gemm:lu_Linv");
                for (int sz = TRI_LEAF; sz < W; sz *= 2) {
                    const int full = W / (2 * sz);
                    if (full > 0 && (e = tri_level<T>(Li, Li, tmp, LuNB<T>::N, sz, 0, sz, full, cs, false)) != cudaSuccess)
                        return e;
                    const int o = full * 2 * sz;
                    if (o + sz < W && (e = tri_level<T>(Li, Li, tmp, LuNB<T>::N, sz, o, W - o - sz, 1, cs, false)) !=
                                          cudaSuccess)
                        return e;
                }
            }
            EV_TRACE(2, t, cs);
            if ((e = cudaEventRecord(evL, cs)) != cudaSuccess) return e;
            // ---- auxiliary stream: left columns + columns beyond the look-ahead block
            if ((e = cudaStreamWaitEvent(ax.st, evL, 0)) != cudaSuccess) return e;
            EV_TRACE(3, t, ax.st);
            {
                const int ncol = K0 + (n - cn1);
                if (ncol > 0) {
                    if ((e = launch_pdl(lu_swap_multi_kernel<T, PW2>, dim3((ncol + SWM_COLS - 1) / SWM_COLS),
                                        dim3(SWM_COLS), 0, ax.st, A, lda, 0, K0, cn1, n, lists, nl)) != cudaSuccess)
                        return e;
                }
                if (cn1 < n && (e = outer_update<T>(n, A, lda, K0, W, cn1, n, Li, Tb[t & 1], ldT, ax.st)) != cudaSuccess)
                    return e;
            }
            EV_TRACE(4, t, ax.st);
            if ((e = cudaEventRecord(evR[t & 1], ax.st)) != cudaSuccess) return e;
            // ---- caller's stream: look-ahead block [cn0, cn1)
            if (cn0 < n) {
                if (t > 0 && (e = cudaStreamWaitEvent(cs, evR[(t - 1) & 1], 0)) != cudaSuccess) return e;
                EV_TRACE(5, t, cs);
                if ((e = launch_pdl(lu_swap_multi_kernel<T, PW2>, dim3((cn1 - cn0 + SWM_COLS - 1) / SWM_COLS),
                                    dim3(SWM_COLS), 0, cs, A, lda, cn0, cn1, 0, 0, lists, nl)) != cudaSuccess)
                    return e;
                if ((e = outer_update<T>(n, A, lda, K0, W, cn0, cn1, Li, Tb[t & 1], ldT, cs)) != cudaSuccess) return e;
                EV_TRACE(6, t, cs);
            }
        }
        // join the auxiliary stream
        if ((e = cudaEventRecord(evJ, ax.st)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(cs, evJ, 0)) != cudaSuccess) return e;
        EV_TRACE(7, 0, cs);
        // EarlyInv (real, Ktail <= n / 2): U's first Ktail rows and L11 are final now; the tail's
        // left-column permutation below must not overwrite L21 before the auxiliary stream copied it
        cudaEvent_t l21_done = nullptr;
        if constexpr (sizeof(T) == 8) {
            if (early && early->vbuf && early->U && early->L && Ktail < n && Ktail > 0 && 2 * Ktail <= n) {
                if ((e = getrf_early_launch(n, A, lda, Ktail, *early, cs, &l21_done)) != cudaSuccess) return e;
            } else if (early) {
                early->h = 0;
                early->ready = false;
            }
        }
        if (Ktail < n) {
            // ---- the trailing m x m matrix (fully updated, all earlier row moves applied to every
            // column) factored by lu2 into compact buffers, assembled packed back in place; its
            // row permutation then applied to the L columns on the left and to perm
            const int m = n - Ktail;
            const long long ldm = ld8(m);
            T *tb = work + 3 * (size_t)LuNB<T>::N * LuNB<T>::N + 2 * (size_t)LuNB<T>::N * ld8(n);
            tb = reinterpret_cast<T *>((reinterpret_cast<uintptr_t>(tb) + 255) & ~(uintptr_t)255);
            T *B0 = tb, *B1 = tb + (size_t)m * ldm;
            int *iw2 = reinterpret_cast<int *>(B1 + (size_t)m * ldm);
            int *psub = iw2 + lu2_int_elems(m), *ptmp = psub + m;
            if constexpr (sizeof(T) == 8) {
                if (early && early->ready) early->wmap = psub;  // W[i] = W'[psub[i]] once the tail is done
            }
            T *A22 = A + (long long)Ktail * lda + Ktail;
            if ((e = launch_pdl(copy_block_kernel<T>, dim3(ew_grid((long long)m * m)), dim3(256), 0, cs, (const T *)A22,
                                lda, B0, ldm, m, m)) != cudaSuccess)
                return e;
            if ((e = lu2_factor<T>(m, B0, B1, ldm, A22, A22, lda, psub, iw2, diag + Ktail, nullptr, cs)) != cudaSuccess)
                return e;
            EV_TRACE(8, 0, cs);
            if (l21_done) {
                e = cudaStreamWaitEvent(cs, l21_done, 0);
                cudaEventDestroy(l21_done);
                if (e != cudaSuccess) return e;
            }
            for (int c0 = 0; c0 < Ktail; c0 += m) {  // left columns in chunks of m through B1
                const int nc = min(m, Ktail - c0);
                if ((e = launch_pdl(gather_rows_kernel<T>, dim3(ew_grid((long long)m * nc)), dim3(256), 0, cs,
                                    (const T *)A, lda, Ktail, c0, m, nc, (const int *)psub, B1, ldm)) != cudaSuccess)
                    return e;
                if ((e = launch_pdl(copy_block_kernel<T>, dim3(ew_grid((long long)m * nc)), dim3(256), 0, cs,
                                    (const T *)B1, ldm, A + (long long)Ktail * lda + c0, lda, m, nc)) != cudaSuccess)
                    return e;
            }
            for (int ph = 0; ph < 2; ++ph)
                if ((e = launch_pdl(perm_gather_kernel, dim3((m + 255) / 256), dim3(256), 0, cs, perm, Ktail, m,
                                    (const int *)psub, ptmp, ph)) != cudaSuccess)
                    return e;
        }
        EV_TRACE(9, 0, cs);
        if (prio) {
            if ((e = cudaEventRecord(ax.ev[5], cs)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(s, ax.ev[5], 0)) != cudaSuccess) return e;
        }
    }
    if (stats) {
        e = launch_pdl(lu_stats_kernel<T>, dim3(1), dim3(1024), 0, s, diag, n, stats);
    }
    return e;
}
template cudaError_t getrf<double>(int, double *, long long, int *, int *, double *, LuStats *, double *, cudaStream_t,
                                   EarlyInv *);
template cudaError_t getrf<double2>(int, double2 *, long long, int *, int *, double2 *, LuStats *, double2 *,
                                    cudaStream_t, EarlyInv *);

}  // namespace frob
