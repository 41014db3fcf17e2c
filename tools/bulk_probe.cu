// bulk_probe.cu -- standalone timing of lu2's BULK trailing update (lu_update2m_kernel, look-ahead
// mode) at the trailing sizes of an n = 4096 LU, against a plain device copy of the same bytes.
// Debug tool, not the product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/bulk_probe tools/bulk_probe.cu -lcuda
#include "../paper_2208_01239_b200/csrc/lu.cu"
#include "../paper_2208_01239_b200/csrc/tma.cu"
#include "../paper_2208_01239_b200/csrc/lu2.cu"
#include <vector>
#include <random>
#include <algorithm>
using namespace frob;
unsigned long long &frob::launch_counter() { static unsigned long long c = 0; return c; }
bool frob::prof_enabled() { return false; }
void frob::prof_record(const char *, cudaStream_t, bool, double) {}
thread_local const char *frob::g_gemm_tag = nullptr;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

// the body with an explicit streaming switch (the product kernel streams for n > 2048)
template <int PW>
__global__ void __launch_bounds__(U2_T, 3)
bulk_nostream(const double *Bk, double *Bn, long long ld, int n, int k0, int w, const int *mv2, int *u12f, int tag,
              int cbeg, int cend) {
    update2m_body<double, PW>(Bk, Bn, ld, n, k0, w, mv2, nullptr, nullptr, nullptr, u12f, tag, cbeg, cend, 0, false);
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 4096;
    constexpr int PW = 32;
    const long long ld = n;
    const size_t bytes = (size_t)n * ld * sizeof(double);
    double *B0, *B1;
    CK(cudaMalloc(&B0, bytes));
    CK(cudaMalloc(&B1, bytes));
    std::vector<double> h((size_t)n * ld);
    std::mt19937_64 g(1);
    std::normal_distribution<double> nd;
    for (auto &v : h) v = nd(g);
    CK(cudaMemcpy(B0, h.data(), bytes, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B1, h.data(), bytes, cudaMemcpyHostToDevice));
    int *mv, *flags, *done;
    CK(cudaMalloc(&mv, MV2_INTS * sizeof(int)));
    CK(cudaMalloc(&flags, 4096 * sizeof(int)));
    CK(cudaMalloc(&done, 4096 * sizeof(int)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int k0 : {0, 256, 768, 1280, 2304, 3072}) {
        const int m = n - k0, w = PW;
        // the move list of a panel: top row k0 + j <-> a distinct pivot row below
        std::vector<int> mvh(MV2_INTS, 0), piv;
        std::uniform_int_distribution<int> ud(k0 + PW, n - 1);
        while ((int)piv.size() < PW) {
            int p = ud(g);
            if (std::find(piv.begin(), piv.end(), p) == piv.end()) piv.push_back(p);
        }
        mvh[0] = 2 * PW;
        for (int j = 0; j < PW; ++j) {
            mvh[1 + j] = k0 + j; mvh[1 + MV2_MAX + j] = piv[j];
            mvh[1 + PW + j] = piv[j]; mvh[1 + MV2_MAX + PW + j] = k0 + j;
        }
        CK(cudaMemcpy(mv, mvh.data(), MV2_INTS * sizeof(int), cudaMemcpyHostToDevice));
        const int cb = k0 + 2 * PW, cols = n - cb, rows = m - w;
        dim3 grid((cols + U2_TC - 1) / U2_TC, (rows + U2_TR - 1) / U2_TR);
        const int reps = 20;
        auto timeit = [&](auto launch) {
            CK(cudaMemset(flags, 0, 4096 * sizeof(int)));
            CK(cudaMemset(done, 0, 4096 * sizeof(int)));
            launch(1);
            CK(cudaDeviceSynchronize());
            CK(cudaEventRecord(e0));
            for (int r = 0; r < reps; ++r) launch(r + 2);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            return ms * 1000.f / reps;
        };
        const float t_prod = timeit([&](int tag) {
            lu_update2m_kernel<double, PW><<<grid, U2_T>>>(B0, B1, ld, n, k0, w, mv, nullptr, nullptr, nullptr, flags, tag,
                                                           cb, n, 0, 1, done + tag);
        });
        const float t_ns = timeit([&](int tag) {
            bulk_nostream<PW><<<grid, U2_T>>>(B0, B1, ld, n, k0, w, mv, flags, tag, cb, n);
        });
        const float t_cp = timeit([&](int) {
            CK(cudaMemcpy2DAsync(B1 + (size_t)(k0 + w) * ld + cb, ld * 8, B0 + (size_t)(k0 + w) * ld + cb, ld * 8,
                                 (size_t)cols * 8, rows, cudaMemcpyDeviceToDevice));
        });
        CK(cudaGetLastError());
        const double mb = 2.0 * rows * (double)cols * 8 / 1e6;
        printf("n=%d k0=%d m=%d grid %dx%d: BULK %.1f us (%.2f TB/s)  no-stream %.1f us  copy2D %.1f us (%.2f TB/s)\n", n,
               k0, m, grid.x, grid.y, t_prod, mb / t_prod, t_ns, t_cp, mb / t_cp);
    }
    return 0;
}
