// fp64_peak.cu -- measured FP64 ceilings on this B200: register-resident DMMA
// (mma.sync.m8n8k4.f64) and DFMA loops over all SMs, CUDA-event timed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double *out, int iters) {
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 42.0) out[0] = s;
}

__global__ void dfma_loop(double *out, int iters) {
    double c[8];
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x;
    double a = 1.0 + 1e-12, b = 1e-9;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, b);
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i];
    if (s == 42.0) out[0] = s;
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int sms = p.multiProcessorCount;
    double *d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps : {4, 8, 16}) {
        int blocks = sms * 2, threads = warps * 32 / 2;
        dmma_loop<<<blocks, threads>>>(d, 100);
        cudaEventRecord(e0);
        dmma_loop<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = (double)blocks * (threads / 32) * iters * 8 * 512.0;
        printf("{\"kind\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", warps, flops / ms / 1e9);
    }
    for (int warps : {8, 16, 32}) {
        int blocks = sms * 2, threads = warps * 32 / 2;
        dfma_loop<<<blocks, threads>>>(d, 100);
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(d, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = (double)blocks * threads * iters * 8 * 2.0;
        printf("{\"kind\": \"dfma\", \"warps_per_sm\": %d, \"tflops\": %.3f}\n", warps, flops / ms / 1e9);
    }
    printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, p.clockRate);
    return 0;
}
