// getrf_probe.cu -- time one LU (and inv_from_lu) at order n, for launch-list profiling.
#include "../paper_2208_01239_b200/csrc/lu.cu"
#include <vector>
#include <random>
using namespace frob;
unsigned long long &frob::launch_counter() { static unsigned long long c = 0; return c; }
bool frob::prof_enabled() { return false; }
void frob::prof_record(const char *, cudaStream_t, bool, double) {}
int main(int argc, char **argv) {
    int n = argc > 1 ? atoi(argv[1]) : 4096;
    int reps = argc > 2 ? atoi(argv[2]) : 2;
    long long ld = n;
    std::vector<double> h((size_t)n * n);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    for (auto &x : h) x = nd(g);
    for (int i = 0; i < n; ++i) h[(size_t)i * n + i] += sqrt((double)n);
    double *A, *diag, *work, *U, *L, *O;
    int *perm, *mv;
    LuStats *st;
    int *cnt;
    cudaMalloc(&cnt, 16);
    cudaMalloc(&A, h.size() * 8); cudaMalloc(&U, h.size() * 8); cudaMalloc(&L, h.size() * 8); cudaMalloc(&O, h.size() * 8);
    cudaMalloc(&diag, n * 8); cudaMalloc(&perm, n * 4); cudaMalloc(&mv, lu_mv_ints(n) * 4);
    cudaMalloc(&work, getrf_work_elems<double>(n) * 8); cudaMalloc(&st, sizeof(LuStats));
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&e2);
    for (int r = 0; r < reps; ++r) {
        cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        unsigned long long l0 = launch_counter();
        cudaEventRecord(e0);
        getrf<double>(n, A, ld, perm, mv, diag, st, work, 0);
        cudaEventRecord(e1);
        inv_from_lu<double>(n, A, ld, U, L, O, ld, perm, cnt, 0);
        cudaEventRecord(e2);
        cudaEventSynchronize(e2);
        float ms1, ms2;
        cudaEventElapsedTime(&ms1, e0, e1);
        cudaEventElapsedTime(&ms2, e1, e2);
        printf("n=%d getrf %.1f us, inv_from_lu %.1f us, launches %llu\n", n, ms1 * 1e3, ms2 * 1e3, launch_counter() - l0);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
