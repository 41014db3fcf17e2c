// lu2_probe.cu -- correctness + timing probe of the latency-oriented LU (lu2.cu) against the
// blocked getrf (lu.cu).  Debug tool, not the product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/lu2_probe tools/lu2_probe.cu
#include "../paper_2208_01239_b200/csrc/lu.cu"
#include "../paper_2208_01239_b200/csrc/tma.cu"
#include "../paper_2208_01239_b200/csrc/lu2.cu"
#include "lu3_experiment.cu"
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>
using namespace frob;
unsigned long long &frob::launch_counter() { static unsigned long long c = 0; return c; }
bool frob::prof_enabled() { return false; }
void frob::prof_record(const char *, cudaStream_t, bool, double) {}
thread_local const char *frob::g_gemm_tag = nullptr;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

template <typename T> double re_of(T v);
template <> double re_of(double v) { return v; }
template <> double re_of(double2 v) { return v.x; }

template <typename T>
void run(int n, int reps, bool use3 = false) {
    const bool cplx = sizeof(T) == 16;
    const long long ld = (n + 7) / 8 * 8;
    const int E = sizeof(T) / 8;
    std::vector<double> h((size_t)n * ld * E, 0.0);
    std::mt19937_64 g(7 + n);
    std::normal_distribution<double> nd;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n * E; ++j) h[(size_t)i * ld * E + j] = nd(g);
    for (int i = 0; i < n; ++i) h[(size_t)i * ld * E + (size_t)i * E] += std::sqrt((double)n);
    T *B0, *B1, *U, *L, *diag, *O;
    int *perm, *iw;
    LuStats *st;
    const size_t bytes = (size_t)n * ld * sizeof(T);
    CK(cudaMalloc(&B0, bytes)); CK(cudaMalloc(&B1, bytes)); CK(cudaMalloc(&U, bytes)); CK(cudaMalloc(&L, bytes));
    CK(cudaMalloc(&O, bytes));
    CK(cudaMalloc(&diag, n * sizeof(T))); CK(cudaMalloc(&perm, n * 4)); CK(cudaMalloc(&iw, std::max(lu2_int_elems(n), lu3_int_elems(n)) * 4));
    CK(cudaMalloc(&st, sizeof(LuStats)));
    cudaMemset(B1, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaMemcpy(B0, h.data(), bytes, cudaMemcpyHostToDevice));
        cudaEventRecord(e0);
        if (use3) CK(lu3_factor<T>(n, B0, ld, U, L, perm, iw, diag, st, 0));
        else CK(lu2_factor<T>(n, B0, B1, ld, U, L, ld, perm, iw, diag, st, 0));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    CK(cudaGetLastError());
    // residual || P A - L U ||_F / ||A||_F on the host
    std::vector<double> hU((size_t)n * ld * E), hL((size_t)n * ld * E);
    std::vector<int> hp(n);
    CK(cudaMemcpy(hU.data(), U, bytes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hL.data(), L, bytes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hp.data(), perm, n * 4, cudaMemcpyDeviceToHost));
    std::vector<int> seen(n, 0);
    bool pok = true;
    for (int i = 0; i < n; ++i) { if (hp[i] < 0 || hp[i] >= n || seen[hp[i]]++) pok = false; }
    double num = 0, den = 0, maxl = 0;
    const int stride = std::max(1, n / 128);
    for (int i = 0; i < n; i += stride) {
        for (int j = 0; j < n; ++j) {
            double sr = 0, si = 0;
            for (int k = 0; k <= std::min(i, j); ++k) {
                const double *l = &hL[(size_t)i * ld * E + (size_t)k * E];
                const double *u = &hU[(size_t)k * ld * E + (size_t)j * E];
                if (cplx) { sr += l[0] * u[0] - l[1] * u[1]; si += l[0] * u[1] + l[1] * u[0]; }
                else sr += l[0] * u[0];
            }
            const double *a = &h[(size_t)hp[i] * ld * E + (size_t)j * E];
            num += (sr - a[0]) * (sr - a[0]) + (cplx ? (si - a[1]) * (si - a[1]) : 0.0);
            den += a[0] * a[0] + (cplx ? a[1] * a[1] : 0.0);
            if (j < i) maxl = std::max(maxl, std::fabs(hL[(size_t)i * ld * E + (size_t)j * E]));
        }
    }
    // reference: blocked getrf on the same input, compare pivots
    int *perm0, *mv; T *work, *diag0;
    CK(cudaMalloc(&perm0, n * 4)); CK(cudaMalloc(&mv, lu_mv_ints(n) * 4));
    CK(cudaMalloc(&work, std::max<size_t>(1, getrf_work_elems<T>(n)) * sizeof(T))); CK(cudaMalloc(&diag0, n * sizeof(T)));
    float best0 = 1e30f;
    for (int r = 0; r < reps; ++r) {
        CK(cudaMemcpy(B0, h.data(), bytes, cudaMemcpyHostToDevice));
        cudaEventRecord(e0);
        CK(getrf<T>(n, B0, ld, perm0, mv, diag0, st, work, 0));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        best0 = std::min(best0, ms);
    }
    std::vector<int> hp0(n);
    CK(cudaMemcpy(hp0.data(), perm0, n * 4, cudaMemcpyDeviceToHost));
    int pdiff = 0;
    for (int i = 0; i < n; ++i) pdiff += hp0[i] != hp[i];
    // inverse timing from the split factors
    CK(cudaMemcpy(B0, h.data(), bytes, cudaMemcpyHostToDevice));
    float bi = 1e30f;
    for (int r = 0; r < reps; ++r) {
        if (use3) CK(lu3_factor<T>(n, B0, ld, U, L, perm, iw, diag, st, 0));
        else CK(lu2_factor<T>(n, B0, B1, ld, U, L, ld, perm, iw, diag, st, 0));
        cudaEventRecord(e0);
        CK(inv_from_ul<T>(n, U, L, ld, B0, O, ld, perm, nullptr, 0));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        bi = std::min(bi, ms);
        CK(cudaMemcpy(B0, h.data(), bytes, cudaMemcpyHostToDevice));
    }
    // X A = I check on sampled rows
    std::vector<double> hO((size_t)n * ld * E);
    CK(cudaMemcpy(hO.data(), O, bytes, cudaMemcpyDeviceToHost));
    double rres = 0;
    for (int i = 0; i < n; i += stride)
        for (int j = 0; j < n; ++j) {
            double sr = 0, si = 0;
            for (int k = 0; k < n; ++k) {
                const double *x = &hO[(size_t)i * ld * E + (size_t)k * E];
                const double *a = &h[(size_t)k * ld * E + (size_t)j * E];
                if (cplx) { sr += x[0] * a[0] - x[1] * a[1]; si += x[0] * a[1] + x[1] * a[0]; }
                else sr += x[0] * a[0];
            }
            sr -= (i == j);
            rres += sr * sr + si * si;
        }
    printf("%s %s n=%5d  lu %8.1f us  getrf %8.1f us  | rel(PA-LU) %.2e  perm %s  maxL %.2f  pivdiff %d | inv_from_ul %7.1f us  rowsample ||XA-I|| %.2e\n",
           use3 ? "LU3" : "LU2", cplx ? "cplx" : "real", n, best * 1e3, best0 * 1e3, std::sqrt(num / den), pok ? "ok" : "BAD", maxl, pdiff,
           bi * 1e3, std::sqrt(rres));
    cudaFree(B0); cudaFree(B1); cudaFree(U); cudaFree(L); cudaFree(O); cudaFree(diag); cudaFree(perm); cudaFree(iw);
    cudaFree(perm0); cudaFree(mv); cudaFree(work); cudaFree(diag0); cudaFree(st);
}

template <typename T>
void pieces(int n) {
    constexpr int PW = Panel2W<T>::PW, PH = Panel2W<T>::PH;
    const long long ld = (n + 7) / 8 * 8;
    const size_t bytes = (size_t)n * ld * sizeof(T);
    std::vector<double> h(bytes / 8);
    std::mt19937_64 g(3);
    std::normal_distribution<double> nd;
    for (auto &x : h) x = nd(g);
    T *B0, *B1, *diag; int *iw, *perm, *iperm;
    CK(cudaMalloc(&B0, bytes)); CK(cudaMalloc(&B1, bytes)); CK(cudaMalloc(&diag, n * sizeof(T)));
    CK(cudaMalloc(&iw, lu2_int_elems(n) * 4)); CK(cudaMalloc(&perm, n * 4)); CK(cudaMalloc(&iperm, n * 4));
    CK(cudaMemcpy(B0, h.data(), bytes, cudaMemcpyHostToDevice));
    iota2_kernel<<<(n + 255) / 256, 256>>>(perm, iperm, n, nullptr, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    auto tm = [&](const char *nm, auto fn, int reps) {
        for (int r = 0; r < 3; ++r) fn();
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r) fn();
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        printf("  %s n=%d: %-40s %8.2f us\n", sizeof(T) == 8 ? "real" : "cplx", n, nm, ms * 1e3 / reps);
    };
    // the panel kernel re-factors the same (already factored) panel: timing only
    CUtensorMap tmap;
    CK(tma_map_rows128(&tmap, B0, n, (long long)n * (sizeof(T) / 8), ld * (sizeof(T) / 8), 256));
    if (n <= 2 * P2_T) tm("panel2 (m=n) x20", [&] {
        if (n <= P2_T) launch_panel2<T, PH, 1>(tmap, B0, ld, n, 0, PW, iw, diag, 0);
        else launch_panel2c<T, PH>(tmap, B0, ld, n, 0, PW, iw, diag, (n + P2_T - 1) / P2_T, 0);
    }, 20);
#ifdef FROB_P2_TRACE
    if (n <= 2 * P2_T) {
        long long tr[64];
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpyFromSymbol(tr, g_p2_trace, sizeof(tr)));
        printf("   trace: load %lld | cols:", tr[1] - tr[0]);
        for (int j = 0; j < PW; ++j) printf(" %lld", tr[2 + j] - (j ? tr[1 + j] : tr[1]));
        printf(" | tail %lld | store %lld\n", tr[20] - tr[1 + PW], tr[21] - tr[20]);
        printf("   transition: wait %lld  fill+solve %lld  update+swap %lld | half1 %lld | tail %lld\n", tr[31] - tr[30],
               tr[33] - tr[31], tr[34] - tr[33], tr[20] - tr[34], tr[21] - tr[20]);
        printf("   col5: pre-bar %lld bar %lld argmax+row %lld l+next %lld cand+redux %lld rest %lld publish %lld\n",
               tr[40] - tr[6], tr[41] - tr[40], tr[42] - tr[41], tr[43] - tr[42], tr[44] - tr[43], tr[45] - tr[44], tr[7] - tr[45]);
    }
#endif

    if (n > P2_T) {
        tm("panel2c cluster (m=n) x20", [&] {
            launch_panel2c<T, PH>(tmap, B0, ld, n, 0, PW, iw, diag, (n + P2_T - 1) / P2_T, 0);
        }, 20);
#ifdef FROB_P2_TRACE
        long long tr[64];
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpyFromSymbol(tr, g_p2_trace, sizeof(tr)));
        printf("   trace: load %lld half0 %lld trans %lld half1 %lld tail %lld | cols(half1):", tr[1] - tr[0], tr[19] - tr[1],
               tr[18] - tr[19], tr[20] - tr[18], tr[21] - tr[20]);
        for (int j = 1; j < PH; ++j) printf(" %lld", tr[2 + j] - tr[1 + j]);
        printf("\n   trans: obox %lld push %lld hwait %lld solve %lld update %lld",
               tr[22] - tr[19], tr[23] - tr[22], tr[24] - tr[23], tr[25] - tr[24], tr[18] - tr[25]);
        printf("\n   col5: pre-bar %lld push %lld deferred %lld wait %lld argmax+row %lld mult %lld cand+pub %lld\n",
               tr[40] - tr[6], tr[41] - tr[40], tr[42] - tr[41], tr[43] - tr[42], tr[44] - tr[43], tr[45] - tr[44], tr[7] - tr[45]);
#endif
    }
    const int rest = n - PW;
    dim3 grid(max(1, (rest + U2_TC - 1) / U2_TC), max(1, (rest + U2_TR - 1) / U2_TR));
    tm("update2 step 0 x20", [&] {
        launch_pdl(lu_update2_kernel<T, PW>, grid, dim3(U2_T), 0, (cudaStream_t)0, (const T *)B0, B1, ld, n, 0, PW,
                   (const int *)iw, perm, iperm, (int *)nullptr);
    }, 20);
    tm("panel2+update2 alternating x20", [&] {
        if (n <= P2_T) launch_panel2<T, PH, 1>(tmap, B0, ld, n, 0, PW, iw, diag, 0);
        else launch_panel2c<T, PH>(tmap, B0, ld, n, 0, PW, iw, diag, (n + P2_T - 1) / P2_T, 0);
        launch_pdl(lu_update2_kernel<T, PW>, grid, dim3(U2_T), 0, (cudaStream_t)0, (const T *)B0, B1, ld, n, 0, PW,
                   (const int *)iw, perm, iperm, (int *)nullptr);
    }, 20);
    tm("empty-ish: iota x20", [&] { launch_pdl(iota2_kernel, dim3(1), dim3(32), 0, (cudaStream_t)0, perm, iperm, 1, (int *)nullptr, 0); }, 20);
    CK(cudaGetLastError());
    cudaFree(B0); cudaFree(B1); cudaFree(diag); cudaFree(iw); cudaFree(perm); cudaFree(iperm);
}

int main(int argc, char **argv) {
    if (argc > 1 && argv[1][0] == 'w') {  // wide cluster panels of the blocked getrf (m > 4096: 9..16 CTAs)
        pieces<double>(4096); pieces<double>(6000); pieces<double>(8192); pieces<double2>(8192);
        return 0;
    }
    if (argc > 1 && argv[1][0] == 'p') {
        pieces<double>(1024); pieces<double>(512); pieces<double2>(1024);
        pieces<double>(2048); pieces<double>(4096); pieces<double2>(4096);
        return 0;
    }
    if (argc > 1 && argv[1][0] == 't') {
#ifdef FROB_L3_TRACE
        for (int n : {1024}) {
            long long z[16] = {0};
            run<double>(n, 1, true);
            CK(cudaMemcpyToSymbol(g_l3_trace, z, sizeof(z)));
            run<double>(n, 1, true);
            long long tr[16];
            CK(cudaMemcpyFromSymbol(tr, g_l3_trace, sizeof(tr)));
            const int nb = n / 16;
            printf("col trace: cand+shfl %lld push %lld wait %lld argmax+row %lld update %lld\n", tr[9] - tr[8], tr[10] - tr[9], tr[11] - tr[10], tr[12] - tr[11], tr[13] - tr[12]);
            printf("n=%d per step (cycles): wait %lld  lookahead %lld  columns %lld (%lld/col)  publish %lld\n", n, tr[0] / nb,
                   tr[1] / nb, tr[2] / nb, tr[2] / n, tr[3] / nb);
        }
#endif
        return 0;
    }
    if (argc > 1 && argv[1][0] == 'c') {  // cluster panel sizes (m > 512 rows)
        int szc[] = {513, 777, 1024, 1025, 1500, 2048, 3001, 4096};
        run<double>(2048, 5);  // warm-up (clocks)
        for (int n : szc) run<double>(n, 5);
        for (int n : szc) run<double2>(n, 3);
        return 0;
    }
    if (argc > 1 && argv[1][0] == '3') {
        int sz3[] = {1, 5, 16, 17, 100, 256, 300, 512, 513, 777, 1000, 1024};
        for (int n : sz3) run<double>(n, n >= 512 ? 5 : 2, true);
        for (int n : sz3) run<double2>(n, n >= 512 ? 5 : 2, true);
        return 0;
    }
    int sizes[] = {1, 5, 16, 17, 100, 256, 300, 512, 513, 777, 1024};
    for (int n : sizes) run<double>(n, n >= 512 ? 5 : 2);
    for (int n : sizes) run<double2>(n, n >= 512 ? 5 : 2);
    return 0;
}
