// gemm.cuh -- FP64 tensor-core (DMMA) GEMM engine for the Frobenius path.
//
//   C = alpha * op_A * op_B + beta * D          (row-major, fp64 or complex fp64)
//
// Used for: LU trailing updates (Alg 3 line 1), the triangular-inverse recursion and
// the product U^{-1} L^{-1} (Alg 3 lines 2-3), and the three Frobenius GEMMs
// C = X^{-1} Y, M = X + Y C, Im = -C Re (Alg 1).
//
// Design (B200 / sm_100a): FP64 has no tcgen05 kind, so the tensor path is the
// warp-level DMMA (mma.sync.m8n8k4.f64).  Operands are staged global -> shared memory
// with a multi-stage cp.async (LDGSTS) pipeline; each warp owns a register tile of
// 8x8 accumulators.  Shared-memory row strides are padded (real: +4 doubles, complex:
// +4 / +2 elements) so every fragment load is bank-conflict free.
// Extras fused into the kernel:
//   - triangular operands: per-tile k-range restriction (skips all-zero blocks),
//   - B row gather (rows of P*B without materialising it),
//   - output column scatter (the column interchanges of A^{-1} = X P),
//   - the final Frobenius epilogue: X[i][perm[j]] = (Re'[i][j], -(C Re')[i][j]) written
//     interleaved (branch S1), or (Im', -Re') for branch S2.
#pragma once
#include "common.cuh"

namespace frob {

enum { TRI_NONE = 0, TRI_UPPER = 1, TRI_LOWER = 2 };
enum { EPI_STORE = 0, EPI_FROB_A = 1, EPI_FROB_B = 2 };

template <typename T>
struct GemmParams {
    int M, N, K;
    const T *A; long long lda, sA;
    const T *B; long long ldb, sB;
    T *C; long long ldc, sC;         // EPI_FROB_*: C is reinterpreted as double2 (interleaved out)
    const T *D; long long ldd, sD;   // beta input (may alias C) / Re' for EPI_FROB_*
    double alpha, beta;
    const int *browmap;              // nullable: row k of B is B[browmap[k]]
    const int *colperm;              // nullable: output column j goes to colperm[j]
    int triA, triB, epi;
    int triC;                        // TRI_UPPER: tiles strictly below the diagonal are skipped (their
                                     // output is not needed: symmetric trailing updates, SYRK-style)
    int *counter;                    // non-null: persistent CTAs take tiles from this counter,
                                     // longest k-range first (square triangular products)
    int early_trigger;               // set by the launcher: release dependents at entry
                                     // (single-wave grids) instead of after the main loop
    double mu;                       // EPI_FROB_*: output scaled by (1 + mu i) (Alg 5 line 5)
    const int *dbranch;              // EPI_FROB_*, nullable: branch read on the device (*dbranch == 2
                                     // -> EPI_FROB_B, else EPI_FROB_A; AUTO decided on the device)
    int force_split;                 // request split-K even above the tile-count threshold
    int ksplit;                      // set by the launcher: > 1 = split-K over a (1, 1, ksplit)
                                     // cluster; the partials meet in distributed shared memory
                                     // and are summed in chunk order (deterministic)
};

// Up to two independent problems in one launch (blockIdx.z < zsplit -> q[0], else q[1]).
template <typename T>
struct GemmPair {
    GemmParams<T> q[2];
    int zsplit;
};

// BIG = 0: 64 x 64 tiles (4 warps of 32 x 32), several CTAs per SM -- small / medium problems;
// BIG = 1: 128 x 128 tiles (8 warps of 64 x 32), one CTA per SM, fewer shared loads per DMMA --
// large problems (>= 2 waves of tiles).
template <typename T, int BIG = 0> struct GemmCfg;
#ifndef FROB_GEMM_BK      // A/B build knobs (tools/build_variant.sh); the library uses the defaults
#define FROB_GEMM_BK 16
#endif
#ifndef FROB_GEMM_STAGES
#define FROB_GEMM_STAGES 3
#endif
template <> struct GemmCfg<double, 0> {
    static constexpr int BM = 64, BN = 64, BK = FROB_GEMM_BK, WGM = 2, WGN = 2, STAGES = FROB_GEMM_STAGES;
    static constexpr int PADA = 4, PADB = 4;
};
template <> struct GemmCfg<double, 1> {
    static constexpr int BM = 128, BN = 128, BK = 16, WGM = 2, WGN = 4, STAGES = 3;
    static constexpr int PADA = 4, PADB = 4;
};
// BIG = 2: 64 x 128 tiles (4 warps of 32 x 64), two CTAs per SM: 12 fragment loads per 32 DMMA
// instead of 8 per 16, and 0.094 instead of 0.125 staged bytes per flop -- large real problems
// with long k-ranges (BK = 8 x 4 stages: the BK = 16 version spilled in its main loop)
#ifndef FROB_WIDE_BK
#define FROB_WIDE_BK 8
#endif
#ifndef FROB_WIDE_STAGES
#define FROB_WIDE_STAGES 4
#endif
template <> struct GemmCfg<double, 2> {
    static constexpr int BM = 64, BN = 128, BK = FROB_WIDE_BK, WGM = 2, WGN = 2, STAGES = FROB_WIDE_STAGES;
    static constexpr int PADA = 4, PADB = 4;
};
template <int BIG> struct GemmCfg<double2, BIG> {
    static constexpr int BM = 64, BN = 64, BK = 8, WGM = 2, WGN = 4, STAGES = 3;
    static constexpr int PADA = 4, PADB = 2;
};

template <typename T, int BIG = 0>
constexpr size_t gemm_smem_bytes() {
    using C = GemmCfg<T, BIG>;
    // (the split-K cluster reduction reuses the stages for one BM x (BN + pad) partial)
    const size_t st = (size_t)C::STAGES * ((size_t)C::BM * (C::BK + C::PADA) + (size_t)C::BK * (C::BN + C::PADB)) * sizeof(T);
    const size_t part = (size_t)C::BM * (C::BN + (sizeof(T) == 8 ? 4 : 0)) * sizeof(T);
    return st > part ? st : part;
}

// ---------------------------------------------------------------- MMA micro-kernels
template <int MT, int NT>
FROB_DEV void mma_tile(double (&acc)[MT][NT][2], const double (&a)[MT], const double (&b)[NT]) {
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
}
// complex: acc[..][0..1] real part, acc[..][2..3] imaginary part
template <int MT, int NT>
FROB_DEV void mma_tile(double (&acc)[MT][NT][4], const double2 (&a)[MT], const double2 (&b)[NT]) {
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        double nai = -a[i].y;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            dmma(acc[i][j][0], acc[i][j][1], a[i].x, b[j].x);
            dmma(acc[i][j][0], acc[i][j][1], nai, b[j].y);
            dmma(acc[i][j][2], acc[i][j][3], a[i].x, b[j].y);
            dmma(acc[i][j][2], acc[i][j][3], a[i].y, b[j].x);
        }
    }
}

template <typename T> struct AccW { static constexpr int V = 2; };
template <> struct AccW<double2> { static constexpr int V = 4; };

FROB_DEV double acc_val(const double (&c)[2], int e) { return c[e]; }
FROB_DEV double acc_re(double v) { return v; }
FROB_DEV double acc_re(double2 v) { return v.x; }
FROB_DEV double acc_im(double2 v) { return v.y; }
FROB_DEV double2 acc_val(const double (&c)[4], int e) { return make_double2(c[e], c[2 + e]); }

// Split-K cluster reduction (see gemm_tile): out of line so that its registers do not add to the
// main loop's allocation.  P = this CTA's BM x PS partial in shared memory.
template <typename T, int BM, int BN, int PS, int NTH>
FROB_DEV void split_reduce(const int S, const int M, const int N, const double alpha, const double beta,
                                          const T *__restrict__ D, const long long ldd, T *Cp, const long long ldc,
                                          const int *__restrict__ colperm, const int row0, const int col0,
                                          const T *P) {
    cluster_sync_all();
    const int tid = threadIdx.x;
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const unsigned pbase = smem_u32(P);
    constexpr int TILE = BM * BN, SMAX = 8;
    const int per = (TILE + S - 1) / S;
    const int lo = (int)rank * per, hi = min(TILE, lo + per);
    for (int idx = lo + tid; idx < hi; idx += NTH) {
        // all S remote loads in flight before the adds; summed in rank (= chunk) order
        const unsigned off = pbase + (unsigned)(((idx / BN) * PS + idx % BN) * sizeof(T));
        T part[SMAX];
#pragma unroll
        for (int q = 0; q < SMAX; ++q)
            if (q < S) part[q] = ld_cluster(mapa_u32(off, (unsigned)q), T());
        const int row = row0 + idx / BN, col = col0 + idx % BN;
        if (row >= M || col >= N) continue;
        T v = part[0];
#pragma unroll
        for (int q = 1; q < SMAX; ++q)
            if (q < S) v = add(v, part[q]);
        v = scal(v, alpha);
        if (beta != 0.0) v = add(v, scal(D[(long long)row * ldd + col], beta));
        Cp[(long long)row * ldc + (colperm ? colperm[col] : col)] = v;
    }
    cluster_sync_all();  // keep this CTA's partial alive until every reader is done
}

template <typename T, bool VEC, int BIG, bool SPLIT>
FROB_DEV void gemm_tile(const GemmParams<T> &p, const long long bz, const int row0, const int col0, T *As, T *Bs) {
    using Cf = GemmCfg<T, BIG>;
    constexpr int BM = Cf::BM, BN = Cf::BN, BK = Cf::BK, STAGES = Cf::STAGES;
    constexpr int NTH = Cf::WGM * Cf::WGN * 32;
    constexpr int WM = BM / Cf::WGM, WN = BN / Cf::WGN, MT = WM / 8, NT = WN / 8;
    constexpr int E = 16 / sizeof(T);
    constexpr int SA = BK + Cf::PADA, SB = BN + Cf::PADB;
    constexpr int V = AccW<T>::V;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm0 = (warp / Cf::WGN) * WM, wn0 = (warp % Cf::WGN) * WN;
    const T *__restrict__ A = p.A + bz * p.sA;
    const T *__restrict__ B = p.B + bz * p.sB;
    const int M = p.M, N = p.N, K = p.K;
    if (row0 >= M || col0 >= N) return;

    int kb = 0, ke = K;
    if (p.triA == TRI_UPPER) kb = max(kb, row0);
    else if (p.triA == TRI_LOWER) ke = min(ke, row0 + BM);
    if (p.triB == TRI_UPPER) ke = min(ke, col0 + BN);
    else if (p.triB == TRI_LOWER) kb = max(kb, col0);
    kb = (kb / BK) * BK;
    if (SPLIT) {
        const int tot = (ke > kb) ? (ke - kb + BK - 1) / BK : 0;
        const int per = (tot + p.ksplit - 1) / p.ksplit;
        const int c = (int)(blockIdx.z % p.ksplit);
        const int b2 = kb + c * per * BK;
        ke = min(ke, b2 + per * BK);
        kb = b2;  // an empty chunk still joins the cluster reduction (adds zero)
    }
    const int nk = (ke > kb) ? (ke - kb + BK - 1) / BK : 0;

    double acc[MT][NT][V];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < V; ++e) acc[i][j][e] = 0.0;

    // Fast path (interior tile, 16-byte aligned operands): every thread's chunks keep the same
    // (row, column) offsets in each stage, so their global addresses are computed once and
    // advanced by a constant per stage; no bounds checks.  The checked path below serves edge
    // tiles and the ragged last stage (K or a triangular k-range not a multiple of BK).
    constexpr int ACH = BM * BK / E, BCH = BK * BN / E;
    constexpr int APT = (ACH + NTH - 1) / NTH, BPT = (BCH + NTH - 1) / NTH;
    static_assert(ACH % NTH == 0 && BCH % NTH == 0, "whole chunks per thread");
    // chunk c = tid + u * NTH of a stage sits at row c / (chunks per row): the column is the same for
    // every u and the row advances by a constant, so one base address per operand serves all u
    static_assert(NTH % (BK / E) == 0 && NTH % (BN / E) == 0, "affine chunk rows");
    constexpr int ARS = NTH / (BK / E), BRS = NTH / (BN / E);  // row step per u
    const bool fast = VEC && row0 + BM <= M && col0 + BN <= N;
    const int ar0 = tid / (BK / E), acc0 = (tid % (BK / E)) * E;
    const int br0 = tid / (BN / E), bcc0 = (tid % (BN / E)) * E;
    const T *asrc0 = A + (long long)(row0 + ar0) * p.lda + kb + acc0;
    const unsigned adst0 = (unsigned)(ar0 * SA + acc0);
    const int boff0 = col0 + bcc0, bdst0 = br0 * SB + bcc0;
    auto load_stage = [&](int s, int kt) {
        const int k0 = kb + kt * BK;
        if (fast && k0 + BK <= K) {
            T *as = As + s * BM * SA + adst0;
            T *bs = Bs + s * BK * SB + bdst0;
            const T *ag = asrc0 + kt * BK;
#pragma unroll
            for (int u = 0; u < APT; ++u) cp_async16(as + u * ARS * SA, ag + (long long)u * ARS * p.lda);
            if (p.browmap) {
#pragma unroll
                for (int u = 0; u < BPT; ++u)
                    cp_async16(bs + u * BRS * SB, B + (long long)p.browmap[k0 + br0 + u * BRS] * p.ldb + boff0);
            } else {
                const T *bg = B + (long long)(k0 + br0) * p.ldb + boff0;
#pragma unroll
                for (int u = 0; u < BPT; ++u) cp_async16(bs + u * BRS * SB, bg + (long long)u * BRS * p.ldb);
            }
            return;
        }
        T *as = As + s * BM * SA;
        T *bs = Bs + s * BK * SB;
#pragma unroll 2
        for (int c = tid; c < ACH; c += NTH) {
            const int r = c / (BK / E), cc = (c % (BK / E)) * E;
            const int gr = row0 + r, gk = k0 + cc;
            T *dst = as + r * SA + cc;
            if (VEC && gr < M && gk + E <= K) {
                cp_async16(dst, A + (long long)gr * p.lda + gk);
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e)
                    dst[e] = (gr < M && gk + e < K) ? A[(long long)gr * p.lda + gk + e] : zero_of(T());
            }
        }
#pragma unroll 2
        for (int c = tid; c < BCH; c += NTH) {
            const int r = c / (BN / E), cc = (c % (BN / E)) * E;
            const int gk = k0 + r, gc = col0 + cc;
            T *dst = bs + r * SB + cc;
            if (gk < K) {
                const long long brow = p.browmap ? (long long)p.browmap[gk] : (long long)gk;
                const T *src = B + brow * p.ldb + gc;
                if (VEC && gc + E <= N) {
                    cp_async16(dst, src);
                } else {
#pragma unroll
                    for (int e = 0; e < E; ++e) dst[e] = (gc + e < N) ? src[e] : zero_of(T());
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e] = zero_of(T());
            }
        }
    };

    auto compute_stage = [&](int kt) {
        const T *as = As + (kt % STAGES) * BM * SA;
        const T *bs = Bs + (kt % STAGES) * BK * SB;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            T a[MT], b[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i) a[i] = as[(wm0 + i * 8 + g) * SA + kk + t];
#pragma unroll
            for (int j = 0; j < NT; ++j) b[j] = bs[(kk + t) * SB + wn0 + j * 8 + g];
            mma_tile<MT, NT>(acc, a, b);
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nx = kt + STAGES - 1;
            if (nx < nk) load_stage(nx % STAGES, nx);
            cp_async_commit();
        }
        compute_stage(kt);
    }
    cp_async_wait<0>();
    if (!p.counter && !p.early_trigger) pdl_trigger();

    // ------------------------------------------------------------ epilogue
    // All reads of D (which may alias C) and of colperm are issued before any store so
    // the memory latency is paid once, not once per element.
    const T *__restrict__ D = p.D ? p.D + bz * p.sD : nullptr;
    T *Cp = p.C + bz * p.sC;
    if constexpr (SPLIT) {
        // deterministic split-K: the cluster's S CTAs hold the partials of one tile; each writes
        // its partial to its own shared memory, then reduces 1/S of the tile over all S partials
        // (read through DSMEM in rank order, so the summation order is fixed) and stores it
        constexpr int PS = BN + (sizeof(T) == 8 ? 4 : 0);
        static_assert((size_t)BM * PS * sizeof(T) <= gemm_smem_bytes<T, BIG>(), "partial fits the stages");
        T *P = As;
        __syncthreads();  // all warps done with the stage buffers
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    P[(wm0 + i * 8 + g) * PS + wn0 + j * 8 + 2 * t + e] = acc_val(acc[i][j], e);
        split_reduce<T, BM, BN, PS, NTH>(p.ksplit, M, N, p.alpha, p.beta, D, p.ldd, Cp, p.ldc, p.colperm, row0, col0, P);
        return;
    }
    if constexpr (sizeof(T) == 8) {
        // fast path: interior tile, plain store, 16-byte aligned rows -> vector D/C access
        const bool interior = (row0 + BM <= M) && (col0 + BN <= N) && p.epi == EPI_STORE && !p.colperm &&
                              ((p.ldc & 1) == 0) && (!D || (p.ldd & 1) == 0) &&
                              ((reinterpret_cast<uintptr_t>(Cp) & 15) == 0) &&
                              (!D || (reinterpret_cast<uintptr_t>(D) & 15) == 0);
        if (interior) {
            const double alpha = p.alpha, beta = p.beta;
#pragma unroll
            for (int i = 0; i < MT; ++i) {
                // D loads of one row group are issued together, before its stores
                double2 dv2[NT];
                if (beta != 0.0) {
#pragma unroll
                    for (int j = 0; j < NT; ++j)
                        dv2[j] = *reinterpret_cast<const double2 *>(
                            D + (long long)(row0 + wm0 + i * 8 + g) * p.ldd + col0 + wn0 + j * 8 + 2 * t);
                }
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    double2 v = make_double2(alpha * acc[i][j][0], alpha * acc[i][j][1]);
                    if (beta != 0.0) {
                        v.x = fma(beta, dv2[j].x, v.x);
                        v.y = fma(beta, dv2[j].y, v.y);
                    }
                    *reinterpret_cast<double2 *>(Cp + (long long)(row0 + wm0 + i * 8 + g) * p.ldc + col0 + wn0 +
                                                 j * 8 + 2 * t) = v;
                }
            }
            return;
        }
    }
    const bool needD = (p.epi != EPI_STORE) || (p.beta != 0.0);
    int oc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int col = col0 + wn0 + j * 8 + 2 * t + e;
            oc[j][e] = (p.colperm && col < N) ? p.colperm[col] : col;
        }
#pragma unroll
    for (int i = 0; i < MT; ++i) {
        const int row = row0 + wm0 + i * 8 + g;
        if (row >= M) continue;
        T dv[NT][2];
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = col0 + wn0 + j * 8 + 2 * t + e;
                dv[j][e] = (needD && col < N) ? D[(long long)row * p.ldd + col] : zero_of(T());
            }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = col0 + wn0 + j * 8 + 2 * t + e;
                if (col >= N) continue;
                T v = scal(acc_val(acc[i][j], e), p.alpha);
                if constexpr (sizeof(T) == 8) {
                    if (p.epi != EPI_STORE) {
                        const double d = dv[j][e];
                        double2 *X = reinterpret_cast<double2 *>(Cp);
                        const int epi = p.dbranch ? (*p.dbranch == 2 ? EPI_FROB_B : EPI_FROB_A) : p.epi;
                        double2 o = (epi == EPI_FROB_A) ? make_double2(d, v) : make_double2(v, -d);
                        if (p.mu != 0.0) o = make_double2(o.x - p.mu * o.y, p.mu * o.x + o.y);
                        X[(long long)row * p.ldc + oc[j][e]] = o;
                        continue;
                    }
                }
                if (p.beta != 0.0) v = add(v, scal(dv[j][e], p.beta));
                Cp[(long long)row * p.ldc + oc[j][e]] = v;
            }
        }
    }
}

// SPLIT: the split-K instantiation (cluster launch, see gemm_tile); a separate kernel so that its
// reduction code does not raise the register allocation of the plain GEMM
template <typename T, bool VEC, int BIG, bool SPLIT>
__global__ void __launch_bounds__(GemmCfg<T, BIG>::WGM * GemmCfg<T, BIG>::WGN * 32)
gemm_kernel(GemmPair<T> pp) {
    using Cf = GemmCfg<T, BIG>;
    constexpr int SA = Cf::BK + Cf::PADA;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T *As = reinterpret_cast<T *>(smem_raw);
    T *Bs = As + Cf::STAGES * Cf::BM * SA;
    // multi-wave grids release dependents only after the main loop (see gemm_tile): releasing
    // them at entry lets the next grid's waiting CTAs occupy SM slots this GEMM still needs
    if (pp.q[0].early_trigger) pdl_trigger();
    pdl_wait();
    const int z = SPLIT ? blockIdx.z / pp.q[0].ksplit : blockIdx.z;  // ksplit is equal in both problems
    const GemmParams<T> &p = (z < pp.zsplit) ? pp.q[0] : pp.q[1];
    const long long bz = (z < pp.zsplit) ? z : z - pp.zsplit;
    if (SPLIT || !p.counter) {
        // grouped tile order: consecutive CTAs walk GROUP_M tile rows column by column, so the ~444
        // resident CTAs cover a ~16 x 28 block of tiles and share their A and B k-slabs in L2
        // (row-major order made the resident wave span all tile columns: every B panel was re-read
        // from DRAM once per tile row -- 557 GB per 16384^3 GEMM, ncu)
        constexpr int GROUP_M = 16;
        const int tn = gridDim.x, tm = gridDim.y;
        const int lin = blockIdx.y * tn + blockIdx.x;
        const int first = (lin / (GROUP_M * tn)) * GROUP_M;
        const int gm = min(tm - first, GROUP_M);
        const int rem = lin - first * tn;
        int ty = first + rem % gm, tx = rem / gm;
        // longest triangular k-ranges first (the tail wave then holds short tiles): n = 4096 / 8192
        // Frobenius 32.84 -> 32.67 / 190.2 -> 189.5 ms
        if (p.triB == TRI_UPPER) tx = tn - 1 - tx;
        if (p.triA == TRI_LOWER) ty = tm - 1 - ty;
        if (p.triC == TRI_UPPER && ty * Cf::BM >= (tx + 1) * Cf::BN) return;
        gemm_tile<T, VEC, BIG, SPLIT>(p, bz, ty * Cf::BM, tx * Cf::BN, As, Bs);
        return;
    }
    // persistent: tiles in order of max(I, J) = 0, 1, ... (longest k-range first for
    // upper x lower products); t -> d = isqrt(t), r = t - d^2: (d, r) or (r - d - 1, d)
    __shared__ int tile_s;
    const int D = (p.M + Cf::BM - 1) / Cf::BM;
    const int total = D * D;
    for (;;) {
        __syncthreads();  // previous tile done with the shared stages
        if (threadIdx.x == 0) tile_s = atomicAdd(p.counter, 1);
        __syncthreads();
        const int tt = tile_s;
        if (tt >= total) { pdl_trigger(); break; }
        int d = (int)sqrtf((float)tt);
        while (d * d > tt) --d;
        while ((d + 1) * (d + 1) <= tt) ++d;
        const int r = tt - d * d;
        const int I = (r <= d) ? d : r - d - 1;
        const int J = (r <= d) ? r : d;
        gemm_tile<T, VEC, BIG, false>(p, bz, I * Cf::BM, J * Cf::BN, As, Bs);
    }
}

}  // namespace frob
