// lu.cuh -- blocked LU with partial pivoting (Alg 3 line 1) and the explicit
// inverse from the LU factors (Alg 3 lines 2-3), for real (double) and
// complex (double2) matrices, row-major.
//
// Panel: one thread-block CLUSTER owns the m x PW panel in shared memory (rows split
// across the CTAs).  Per column: each thread scans its rows, warp-shuffle argmax,
// block argmax through shared memory, cluster argmax through DSMEM (one cluster
// barrier per column), then every CTA applies the rank-1 update to its rows.  Rows are
// never moved during the panel ("physical rows" + done flags); at the end each row is
// written straight to its final position and the row movement list is emitted for the
// rest of the matrix.
#pragma once
#include <cuda.h>
#include "common.cuh"
#include "gemm.cuh"

namespace frob {

// device-side pivot diagnostics of one LU (filled by lu_stats_kernel)
struct LuStats {
    double rho;      // max|u_ii| / min|u_ii|
    double umax;     // max|u_ii|
    int info;        // 0 or 1-based first singular pivot column (reading R2)
    int nonfinite;   // 1 if any pivot is NaN/Inf
};

// Early triangular inverses (real lu2): the first h rows of U and the block L11 are final once lu2's
// step h / PW has been applied, while the rest of the LU -- its chain-bound tail, which leaves most
// SMs idle -- is still running.  lu2_factor then assembles them on a low-priority auxiliary stream,
// inverts U11 and L11 in place (tri_inverses) and forms V = U11^{-1} U12 into rows [0, h), columns
// [h, n) of vbuf (its top-left h x h block is that recursion's scratch); inv_from_ul waits for that
// work and finishes with the order-(n - h) blocks and the top-level products
//   U^{-1} = [U11^{-1}, -V U22^{-1}; 0, U22^{-1}],  L^{-1} = [L11^{-1}, 0; -L22^{-1} W, L22^{-1}],  W = L21 L11^{-1}.
// vbuf: n x ldo doubles, untouched by anything else from lu2_factor's start until inv_from_ul returns.
// L21 is not final at that point (later pivots move its rows), but its rows are only permuted:
// W' = L21' L11^{-1} is formed early on the rows in their order after step h / PW - 1 (vbuf rows
// [h, n): L21' in columns [0, h), W' in columns [h, 2h)) and gathered into the final order at the end
// (W[i] = W'[pos_h(perm[h + i]) - h], pos_h = that step's row-position snapshot).
// The blocked LU (getrf, 4096 < n <= 8192) does the same during its lu2 tail: when the blocked part
// has reached h = Ktail (<= n / 2), U's first h rows and L11 are final and L21 only awaits the tail's
// row permutation psub (W[i] = W'[psub[i]]); U and L are then the inverse's split buffers.
struct EarlyInv {
    int h = 0;                    // lu2: the split row (0: not used); getrf sets it
    double *vbuf = nullptr;
    double *U = nullptr, *L = nullptr;  // getrf only: where the inverse's split factors go
    cudaEvent_t done = nullptr;   // recorded on the auxiliary stream after V, W' and P11
    const int *pos_h = nullptr;   // lu2: original row -> position after step h / PW - 1
    const int *perm = nullptr;    // lu2: the final permutation (valid after the LU)
    const int *wmap = nullptr;    // getrf: W[i] = W'[wmap[i]] (the tail's psub, valid after the LU)
    bool ready = false;           // the early blocks were launched (the product takes the block path)
};

// Row movement produced by one panel: rows src[q] -> dst[q] (global indices), q < cnt.
// Layout in an int buffer: [cnt, dst[0..2PWMAX), src[0..2PWMAX)].
constexpr int PW_MAX = 32;
constexpr int MV_INTS = 1 + 4 * PW_MAX;

// Outer block width of the two-level LU (real 256: K = 256 outer GEMMs, n = 8192 LU 27.6 ->
// 26.3 ms; complex 128, where 256 measured slower)
#ifndef FROB_LUNB_D  // A/B build knob (tools/build_variant.sh): outer block of the blocked real LU
#define FROB_LUNB_D 256
#endif
template <typename T> struct LuNB { static constexpr int N = sizeof(T) == 8 ? FROB_LUNB_D : 128; };
// ints needed for the per-panel row-movement lists (mv) of an order-n LU
size_t lu_mv_ints(int n);
// elements of T workspace for the outer update (L11^{-1} x2, recursion scratch, U12 x2)
template <typename T>
size_t getrf_work_elems(int n);

template <typename T>
cudaError_t getrf(int n, T *A, long long lda, int *perm, int *mv, T *diag, LuStats *stats, T *work,
                  cudaStream_t s, EarlyInv *early = nullptr);
// getrf takes EarlyInv for 4096 < n <= 8192 (env FROB_EARLY=0: off, A/B aid)
bool getrf_early_ok(int n);
// getrf's EarlyInv work (lu2.cu): forked from s at the tail (A's first h rows final); l21_done is
// recorded once L21 has been copied out (the tail's left-column permutation must wait for it)
cudaError_t getrf_early_launch(int n, const double *A, long long lda, int h, EarlyInv &ei, cudaStream_t s,
                               cudaEvent_t *l21_done);

// From an LU in `lu` (ld): Xinv = U^{-1} L^{-1} (un-permuted: A^{-1} = Xinv P).
// Work buffers U, L (n x ld each) are overwritten; `lu` may be used as the
// recursion scratch (it is destroyed) when lu_is_scratch.
// counter: device int scratch for the persistent product scheduler (nullable = static grid)
template <typename T>
cudaError_t inv_from_lu(int n, T *lu, long long ld, T *U, T *L, T *out, long long ldo,
                        const int *colperm, int *counter, cudaStream_t s, EarlyInv *early = nullptr);

// Latency-oriented LU for n <= LU2_MAX_N (lu2.cu): B0 holds A on entry and is destroyed,
// B1 is scratch (n x ld); the factors come out split: U (upper, zeros below), L (unit lower,
// zeros above), ldo; perm[i] = original row at position i; iw = lu2_int_elems(n) ints.
constexpr int LU2_MAX_N = 4096;  // single CTA up to 1024 rows, then a cluster of <= 8 CTAs
size_t lu2_int_elems(int n);
// orders that take lu2 (LU2_MAX_N; env FROB_LU2_MAX lowers it: A/B measurement aid)
int lu2_max_n();
// lu2's panel width: one or two 128-byte row halves (real 16 or 32 columns; complex 8 -- the
// two-half complex variant spills).  Real 16-column steps with the fused look-ahead measured
// 3.37 / 9.11 / 38.96 ms at n = 1024 / 2048 / 4096 against 3.33 / 9.02 / 37.22 for 32-column
// steps with the NEXT kernel: 32 stays.
#ifndef PANEL2_REAL_PW
#define PANEL2_REAL_PW 32
#endif
template <typename T> struct Panel2W { static constexpr int PW = PANEL2_REAL_PW, PH = 16; };
template <> struct Panel2W<double2> { static constexpr int PW = 8, PH = 8; };
// lu2's panel kernels used IN PLACE by the blocked getrf: rows [k0, n) x columns [k0, k0 + w) of A
// (lda; tm = tma_map_rows128 of A with 256-row boxes) factored, rows written to their final
// positions, the move list (MV_INTS layout) to mv, pivots to diag[k0..]; n - k0 <= lu2_panel_max_m()
// (LU2_PANEL_MAX_M: a cluster of up to 16 CTAs x 512 rows; env FROB_P2C_MAX=8 lowers it to 4096)
constexpr int LU2_PANEL_MAX_M = 8192;
int lu2_panel_max_m();
template <typename T>
cudaError_t lu2_panel_inplace(const CUtensorMap &tm, T *A, long long lda, int n, int k0, int w, int *mv, T *diag,
                              cudaStream_t s);
// h for an order-n lu2 factorisation (0 below the size where it pays; env FROB_EARLY=0: off, A/B aid)
int early_inv_h(int n);
template <typename T>
cudaError_t lu2_factor(int n, T *B0, T *B1, long long ld, T *U, T *L, long long ldo, int *perm, int *iw, T *diag,
                       LuStats *stats, cudaStream_t s, EarlyInv *early = nullptr);
template <typename T>
cudaError_t lu_stats_launch(const T *diag, int n, LuStats *st, cudaStream_t s);
// U = triu(lu) (zeros below), L = tril(lu, -1) + I (zeros above)
template <typename T>
cudaError_t extract_ul(int n, const T *lu, long long ld, T *U, T *L, cudaStream_t s);
// U <- U^{-1} (upper), L <- L^{-1} (unit lower) in place; tmp: n x ld scratch
template <typename T>
cudaError_t tri_inverses(int n, T *U, T *L, long long ld, T *tmp, cudaStream_t s);
// Xinv = U^{-1} L^{-1} from split factors (U, L destroyed; scratch n x ld)
template <typename T>
cudaError_t inv_from_ul(int n, T *U, T *L, long long ld, T *scratch, T *out, long long ldo, const int *colperm,
                        int *counter, cudaStream_t s, EarlyInv *early = nullptr);

// host-side event timeline (-DFROB_TL builds: tools/getrf_timeline.py, tools/early_timeline.py)
#ifdef FROB_TL
void ev_trace(int kind, int t, cudaStream_t st);
#define EV_TRACE(kind, t, st) ev_trace(kind, t, st)
#else
#define EV_TRACE(kind, t, st) do { } while (0)
#endif

template <typename T>
cudaError_t gemm_launch(const GemmParams<T> &p, int batch, cudaStream_t s);
template <typename T>
cudaError_t gemm_launch2(const GemmParams<T> &p0, int b0, const GemmParams<T> &p1, int b1, cudaStream_t s);

template <typename T>
GemmParams<T> gemm_params(int M, int N, int K, double alpha, const T *A, long long lda,
                          const T *B, long long ldb, double beta, const T *D, long long ldd,
                          T *C, long long ldc) {
    GemmParams<T> p{};
    p.M = M; p.N = N; p.K = K;
    p.A = A; p.lda = lda; p.B = B; p.ldb = ldb;
    p.C = C; p.ldc = ldc; p.D = D; p.ldd = ldd;
    p.alpha = alpha; p.beta = beta;
    p.triA = TRI_NONE; p.triB = TRI_NONE; p.triC = TRI_NONE; p.epi = EPI_STORE;
    return p;
}

}  // namespace frob
