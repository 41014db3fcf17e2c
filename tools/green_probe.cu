// green_probe.cu -- can a green context (SM partition) confine runtime-API kernels, and does a
// 16-CTA cluster then launch promptly on the SMs left outside it?  Probe, not the product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/green_probe tools/green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>
#include <unistd.h>
#include <cstdlib>
#define CK(x) do { auto e_ = (x); if ((int)e_ != 0) { printf("error %d at line %d\n", (int)e_, __LINE__); return 1; } } while (0)

__global__ void smid_kernel(int *out, long long spin) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0 && blockIdx.x < 4096) out[blockIdx.x] = (int)s;
    long long t0 = clock64();
    while (clock64() - t0 < spin) {}
}
__global__ void __cluster_dims__(16, 1, 1) cluster_kernel(unsigned long long *t) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    if (threadIdx.x == 0) atomicMin(t, g);
}
__global__ void stamp(unsigned long long *t) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    *t = g;
}

int main(int argc, char **argv) {
    const unsigned want = argc > 1 ? atoi(argv[1]) : 128;
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    cudaFree(0);  // primary context via the runtime
    CUdevResource res;
    CK(cuDeviceGetDevResource(dev, &res, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs %u\n", res.sm.smCount);
    CUstream gs;
    if (want > 0) {
        CUdevResource grp[1], rem;
        unsigned nb = 1;
        CK(cuDevSmResourceSplitByCount(grp, &nb, &res, &rem, 0, want));
        printf("split: %u group(s) of %u SMs, remaining %u\n", nb, grp[0].sm.smCount, rem.sm.smCount);
        CUdevResourceDesc desc;
        CK(cuDevResourceGenerateDesc(&desc, grp, 1));
        CUgreenCtx g;
        CK(cuGreenCtxCreate(&g, desc, dev, CU_GREEN_CTX_DEFAULT_STREAM));
        CK(cuGreenCtxStreamCreate(&gs, g, CU_STREAM_NON_BLOCKING, 0));
    } else {
        CK(cuStreamCreate(&gs, CU_STREAM_NON_BLOCKING));  // no partition: the busy kernel may use every SM
    }
    int *d;
    CK(cudaMalloc(&d, 4096 * sizeof(int)));
    const int nblk = 4096;
    // a deep queue of short CTAs (50 KB smem: 4 per SM, ~10 us each) on the green stream, like
    // the far-column GEMM's tiles (runtime launch syntax on a driver stream)
    cudaFuncSetAttribute(smid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
    smid_kernel<<<60000, 128, 50 * 1024, (cudaStream_t)gs>>>(d, 200000LL);  // ~100 us each, ~10 ms in all
    CK(cudaGetLastError());
    unsigned long long *t;
    CK(cudaMalloc(&t, 2 * sizeof(unsigned long long)));
    cudaStream_t ms;
    CK(cudaStreamCreateWithFlags(&ms, cudaStreamNonBlocking));
    CK(cudaMemsetAsync(t, 0xff, 2 * sizeof(unsigned long long), ms));
    // a 16-CTA cluster (512 threads, 150 KB smem: one CTA per SM) on the primary context
    cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    usleep(2000);
    stamp<<<1, 1, 0, ms>>>(t + 1);
    cluster_kernel<<<16, 512, 150 * 1024, ms>>>(t);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ms));
    unsigned long long h[2];
    CK(cudaMemcpy(h, t, sizeof(h), cudaMemcpyDeviceToHost));
    printf("16-CTA cluster started %.1f us after its predecessor (green busy kernel still running)\n", (h[0] - h[1]) / 1e3);
    CK(cudaDeviceSynchronize());
    std::vector<int> hs(nblk);
    CK(cudaMemcpy(hs.data(), d, nblk * sizeof(int), cudaMemcpyDeviceToHost));
    std::set<int> sms(hs.begin(), hs.end());
    printf("green-stream kernel ran on %zu distinct SMs\n", sms.size());
    return 0;
}
