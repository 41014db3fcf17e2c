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
#include <cmath>
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

// Candidate: persistent streaming BULK with U12 precomputed (in Bn's top rows, as NEXT would
// publish it).  Each CTA walks tiles t = blockIdx.x + i * gridDim.x (column block fastest); the
// next tile's L21 / U12 slabs (cp.async, 2 stages) and C fragments (registers) are in flight while
// the current tile is multiplied and stored.
template <int PW>
__global__ void __launch_bounds__(U2_T, 3)
bulk_stream(const double *__restrict__ Bk, double *__restrict__ Bn, long long ld, int n, int k0, int w,
            const int *__restrict__ mv2, int cbeg, int cend, int ntc, int ntiles) {
    constexpr int SP = 4;
    constexpr int WM = U2_TR / U2M_WGM, WN = U2_TC / U2M_WGN, MT = WM / 8, NT = WN / 8;
    __shared__ int mdst[MV2_MAX], msrc[MV2_MAX];
    __shared__ int nmv_s;
    __shared__ int rmap[2][U2_TR];
    extern __shared__ __align__(16) double dsm[];
    auto Ls = reinterpret_cast<double (*)[U2_TR][PW + SP]>(dsm);
    auto Us = reinterpret_cast<double (*)[PW][U2_TC + SP]>(dsm + 2 * U2_TR * (PW + SP));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int wm0 = (warp / U2M_WGN) * WM, wn0 = (warp % U2M_WGN) * WN;
    if (tid < MV2_MAX) {
        const int nm = mv2[0];
        if (tid == 0) nmv_s = nm;
        mdst[tid] = tid < nm ? mv2[1 + tid] : -1;
        msrc[tid] = tid < nm ? mv2[1 + MV2_MAX + tid] : -1;
    }
    __syncthreads();
    const int nm = nmv_s;
    const int rbase = k0 + w;
    auto tile_rc = [&](int t, int &r0, int &c0, int &nc) {
        const int ty = t / ntc, tx = t % ntc;
        r0 = rbase + ty * U2_TR;
        c0 = cbeg + tx * U2_TC;
        nc = min(U2_TC, cend - c0);
    };
    // rmap of tile t into slot sl (identity, then the step's moves)
    auto make_rmap = [&](int t, int sl) {
        int r0, c0, nc;
        tile_rc(t, r0, c0, nc);
        if (tid < U2_TR) rmap[sl][tid] = r0 + tid;
        __syncthreads();
        if (tid < nm) {
            const int d = mdst[tid];
            if (d >= r0 && d < r0 + U2_TR) rmap[sl][d - r0] = msrc[tid];
        }
    };
    auto issue_slabs = [&](int t, int st) {
        int r0, c0, nc;
        tile_rc(t, r0, c0, nc);
        for (int idx = tid; idx < U2_TR * (PW / 2); idx += U2_T) {
            const int r = idx / (PW / 2), e = (idx % (PW / 2)) * 2;
            if (r0 + r < n) cp_async16(&Ls[st][r][e], Bk + (long long)(r0 + r) * ld + k0 + e);
        }
        for (int idx = tid; idx < PW * (U2_TC / 2); idx += U2_T) {
            const int i = idx / (U2_TC / 2), e = (idx % (U2_TC / 2)) * 2;
            if (e < nc) cp_async16(&Us[st][i][e], Bn + (long long)(k0 + i) * ld + c0 + e);
        }
        cp_async_commit();
    };
    double acc[MT][NT][2], nxt[MT][NT][2];
    auto load_c = [&](double (&a)[MT][NT][2], int t, int sl) {
        int r0, c0, nc;
        tile_rc(t, r0, c0, nc);
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int rr = wm0 + i * 8 + g;
            const bool ok = r0 + rr < n;
            const double *src = Bk + (long long)(ok ? rmap[sl][rr] : 0) * ld + c0;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int cc = wn0 + j * 8 + 2 * t4;
                if (ok && cc + 1 < nc) {
                    const double2 v = *reinterpret_cast<const double2 *>(src + cc);
                    a[i][j][0] = v.x; a[i][j][1] = v.y;
                } else {
                    a[i][j][0] = (ok && cc < nc) ? src[cc] : 0.0;
                    a[i][j][1] = 0.0;
                }
            }
        }
    };
    int t = blockIdx.x;
    if (t >= ntiles) return;
    make_rmap(t, 0);
    issue_slabs(t, 0);
    __syncthreads();
    load_c(acc, t, 0);
    int st = 0;
    for (; t < ntiles; t += gridDim.x) {
        const int tn = t + gridDim.x;
        if (tn < ntiles) {
            make_rmap(tn, st ^ 1);
            issue_slabs(tn, st ^ 1);
            __syncthreads();
            load_c(nxt, tn, st ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < PW; kk += 4) {
            double a[MT], b[NT];
#pragma unroll
            for (int i = 0; i < MT; ++i) a[i] = -Ls[st][wm0 + i * 8 + g][kk + t4];
#pragma unroll
            for (int j = 0; j < NT; ++j) b[j] = Us[st][kk + t4][wn0 + j * 8 + g];
            mma_tile<MT, NT>(acc, a, b);
        }
        int r0, c0, nc;
        tile_rc(t, r0, c0, nc);
#pragma unroll
        for (int i = 0; i < MT; ++i) {
            const int r = r0 + wm0 + i * 8 + g;
            if (r >= n) continue;
            double *dst = Bn + (long long)r * ld + c0;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int cc = wn0 + j * 8 + 2 * t4;
                if (cc + 1 < nc) *reinterpret_cast<double2 *>(dst + cc) = make_double2(acc[i][j][0], acc[i][j][1]);
                else if (cc < nc) dst[cc] = acc[i][j][0];
            }
        }
        __syncthreads();  // stage st and rmap slot st free for reuse
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) { acc[i][j][0] = nxt[i][j][0]; acc[i][j][1] = nxt[i][j][1]; }
        st ^= 1;
    }
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
        // reference output of the product kernel (U12 published in B1's top rows by it)
        std::vector<double> ref((size_t)rows * cols), got((size_t)rows * cols);
        CK(cudaMemcpy2D(ref.data(), cols * 8, B1 + (size_t)(k0 + w) * ld + cb, ld * 8, cols * 8, rows,
                        cudaMemcpyDeviceToHost));
        const int ntc = (cols + U2_TC - 1) / U2_TC, ntr = (rows + U2_TR - 1) / U2_TR, ntiles = ntc * ntr;
        float t_st[3];
        const int gsz[3] = {148 * 2, 148 * 3, ntiles};
        const int dsmem = (2 * U2_TR * (PW + 4) + 2 * PW * (U2_TC + 4)) * 8;
        CK(cudaFuncSetAttribute(bulk_stream<PW>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem));
        for (int q = 0; q < 3; ++q) {
            const int G = std::min(gsz[q], ntiles);
            CK(cudaMemset2D(B1 + (size_t)(k0 + w) * ld + cb, ld * 8, 0, cols * 8, rows));
            t_st[q] = timeit([&](int) {
                bulk_stream<PW><<<G, U2_T, dsmem>>>(B0, B1, ld, n, k0, w, mv, cb, n, ntc, ntiles);
            });
        }
        CK(cudaMemcpy2D(got.data(), cols * 8, B1 + (size_t)(k0 + w) * ld + cb, ld * 8, cols * 8, rows,
                        cudaMemcpyDeviceToHost));
        double md = 0.0;
        for (size_t i = 0; i < ref.size(); ++i) md = std::max(md, std::fabs(ref[i] - got[i]));
        printf("   stream: G=296 %.1f us  G=444 %.1f us  G=tiles %.1f us  (max |diff| vs product %.2e)\n", t_st[0],
               t_st[1], t_st[2], md);
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
