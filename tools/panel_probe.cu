// panel_probe.cu -- cycle-level probe of the LU kernels (debug tool, not the product).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DFROB_PANEL_TRACE -o tools/panel_probe tools/panel_probe.cu
#include "../paper_2208_01239_b200/csrc/lu.cu"
#include <vector>
#include <random>
#include <algorithm>
using namespace frob;
unsigned long long &frob::launch_counter() { static unsigned long long c = 0; return c; }
bool frob::prof_enabled() { return false; }
void frob::prof_record(const char *, cudaStream_t, bool, double) {}

int main(int argc, char **argv) {
    int n = argc > 1 ? atoi(argv[1]) : 1024;
    long long ld = n;
    std::vector<double> h((size_t)n * n);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    for (auto &x : h) x = nd(g);
    for (int i = 0; i < n; ++i) h[(size_t)i * n + i] += 32.0;
    double *A, *diag;
    int *perm, *mv;
    cudaMalloc(&A, h.size() * 8);
    cudaMalloc(&diag, n * 8);
    cudaMalloc(&perm, n * 4);
    cudaMalloc(&mv, lu_mv_ints(n) * 4);
    double *work; cudaMalloc(&work, getrf_work_elems<double>(n) * 8);
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    // 1) one panel at k0 = 0 (m = n), traced
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        launch_panel<double, 16>(A, ld, n, 16, 0, mv, diag, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long tr[64];
        cudaMemcpyFromSymbol(tr, g_panel_trace, sizeof(tr));
        printf("panel m=%d: %.2f us | load %lld | cols:", n, ms * 1e3, tr[1] - tr[0]);
        for (int j = 0; j < 16; ++j) printf(" %lld", tr[2 + j] - (j ? tr[1 + j] : tr[1]));
        printf(" | tail %lld | store %lld\n", tr[40] - tr[17], tr[41] - tr[40]);
        printf("   col5: pre-bar %lld, bar %lld, bargmax %lld, u-load %lld, next-slot+cand %lld, rest-update %lld, publish %lld\n", tr[50] - tr[6], tr[51] - tr[50], tr[52] - tr[51], tr[53] - tr[52], tr[54] - tr[53], tr[55] - tr[54], tr[7] - tr[55]);
    }
    // 1a) traced cluster panel (R1, CS = n/256)
    if (n > 1024) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
            launch_panel_r<double, 16, 1>(A, ld, n, 16, 0, mv, diag, (n + 255) / 256, 0);
            cudaDeviceSynchronize();
            long long tr[64];
            cudaMemcpyFromSymbol(tr, g_panel_trace, sizeof(tr));
            printf("cluster panel: load %lld | cols:", tr[1] - tr[0]);
            for (int j = 0; j < 16; ++j) printf(" %lld", tr[2 + j] - (j ? tr[1 + j] : tr[1]));
            printf(" | store %lld\n   col5: bar %lld, bargmax %lld, ->push %lld, push %lld, wait %lld, after-wait->u %lld\n",
                   tr[41] - tr[40], tr[51] - tr[50], tr[52] - tr[51], tr[60] - tr[52], tr[61] - tr[60], tr[62] - tr[61], tr[53] - tr[62]);
        }
    }
    // 1b) cluster variants for the same panel
    {
        auto tp = [&](const char *nm, auto fn) {
            float ms2;
            for (int r = 0; r < 3; ++r) fn();
            cudaEventRecord(e0);
            for (int r = 0; r < 20; ++r) fn();
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms2, e0, e1);
            printf("  %-28s %.2f us  (%s)\n", nm, ms2 * 1e3 / 20, cudaGetErrorString(cudaGetLastError()));
        };
        if (n <= 1024) tp("R4 CS1", [&] { launch_panel_r<double, 16, 4>(A, ld, n, 16, 0, mv, diag, 1, 0); });
        if (n <= 1024) tp("R2 CS2", [&] { launch_panel_r<double, 16, 2>(A, ld, n, 16, 0, mv, diag, 2, 0); });
        if (n <= 1024) tp("R1 CS4", [&] { launch_panel_r<double, 16, 1>(A, ld, n, 16, 0, mv, diag, 4, 0); });
        if (n <= 512) tp("R1 CS2", [&] { launch_panel_r<double, 16, 1>(A, ld, n, 16, 0, mv, diag, 2, 0); });
        if (n <= 2048) tp("R1 CS8", [&] { launch_panel_r<double, 16, 1>(A, ld, n, 16, 0, mv, diag, (n + 255) / 256, 0); });
        if (n > 1024) tp("R4 CSn", [&] { launch_panel_r<double, 16, 4>(A, ld, n, 16, 0, mv, diag, (n + 1023) / 1024, 0); });
        if (n > 1024 && n <= 8192) tp("R2 CSn", [&] { launch_panel_r<double, 16, 2>(A, ld, n, 16, 0, mv, diag, (n + 511) / 512, 0); });
        if (n > 1024 && n <= 4096) tp("R1 CSn", [&] { launch_panel_r<double, 16, 1>(A, ld, n, 16, 0, mv, diag, (n + 255) / 256, 0); });
    }
    // 2) kernel-only timings of the LU pieces
    cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    iota_kernel<<<(n + 255) / 256, 256>>>(perm, n);
    float ms;
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch_panel<double, 16>(A, ld, n, 16, 0, mv, diag, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("panel x20 avg %.2f us\n", ms * 1e3 / 20);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) lu_swap_trsm_kernel<double, 16><<<(n - 16 + SWP_COLS - 1) / SWP_COLS, SWP_COLS>>>(A, ld, 0, n, 0, 16, mv, perm);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("swap_trsm x20 avg %.2f us\n", ms * 1e3 / 20);
    auto p = gemm_params<double>(n - 16, n - 16, 16, -1.0, A + 16 * ld, ld, A + 16, ld, 1.0, A + 16 * ld + 16, ld, A + 16 * ld + 16, ld);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) gemm_launch<double>(p, 1, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("trailing gemm K=16 x20 avg %.2f us\n", ms * 1e3 / 20);
    auto q = gemm_params<double>(n, n, n, 1.0, A, ld, A, ld, 0.0, nullptr, ld, A + 0, ld);
    double *C; cudaMalloc(&C, h.size() * 8); q.C = C;
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) gemm_launch<double>(q, 1, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("gemm nnn x10 avg %.2f us = %.2f TF\n", ms * 1e3 / 10, 2.0 * n * n * (double)n / (ms / 10 * 1e-3) / 1e12);
    // full getrf
    LuStats *st; cudaMalloc(&st, sizeof(LuStats));
    for (int r = 0; r < 2; ++r) {
        cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        cudaEventRecord(e0);
        getrf<double>(n, A, ld, perm, mv, diag, st, work, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("getrf n=%d: %.1f us (%lld launches so far)\n", n, ms * 1e3, launch_counter());
    }
    {
        double *U, *L, *O;
        cudaMalloc(&U, h.size() * 8); cudaMalloc(&L, h.size() * 8); cudaMalloc(&O, h.size() * 8);
        for (int r = 0; r < 3; ++r) {
            getrf<double>(n, A, ld, perm, mv, diag, st, work, 0);
            cudaEventRecord(e0);
            inv_from_lu<double>(n, A, ld, U, L, O, ld, perm, nullptr, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            printf("inv_from_lu n=%d: %.1f us\n", n, ms * 1e3);
        }
        // pieces
        long long total = (long long)n * n;
        cudaEventRecord(e0);
        extract_ul_kernel<double><<<(int)std::min<long long>((total + 255) / 256, 148LL * 16), 256>>>(A, ld, n, U, L);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("  extract %.1f us\n", ms * 1e3);
        cudaEventRecord(e0);
        tri_leaf_kernel<double><<<dim3((n + TRI_LEAF - 1) / TRI_LEAF, 2), TRI_LEAF>>>(U, L, ld, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("  leaf %.1f us\n", ms * 1e3);
        for (int sz = TRI_LEAF; sz < n; sz *= 2) {
            const int full = n / (2 * sz);
            cudaEventRecord(e0);
            tri_level<double>(U, L, A, ld, sz, 0, sz, full, 0);
            cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
            printf("  level s=%d (x%d) %.1f us\n", sz, full, ms * 1e3);
        }
        auto pp = gemm_params<double>(n, n, n, 1.0, U, ld, L, ld, 0.0, nullptr, ld, O, ld);
        pp.triA = TRI_UPPER; pp.triB = TRI_LOWER; pp.colperm = perm;
        cudaEventRecord(e0);
        gemm_launch<double>(pp, 1, 0);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("  product %.1f us\n", ms * 1e3);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
