// lat_probe.cu -- dependent-chain latency (cycles) of primitives used on the LU critical path.
#include <cstdio>
#include <cuda_runtime.h>
#define N 256
__global__ void k(double *out, long long *cyc, double x0, unsigned u0) {
    double x = x0, y = x0 * 0.5;
    unsigned u = u0 + threadIdx.x;
    long long t0, t1;
    int slot = 0;
#define MEASURE(stmt)                                   \
    __syncwarp(); t0 = clock64();                       \
    _Pragma("unroll 1") for (int i = 0; i < N; i += 8) { stmt; stmt; stmt; stmt; stmt; stmt; stmt; stmt; } \
    __syncwarp(); t1 = clock64();                       \
    if (threadIdx.x == 0) cyc[slot] = (t1 - t0); ++slot;
    MEASURE(x = fma(x, 1.0000001, 1e-300))                              // 0 DFMA
    MEASURE(x = x * 1.0000001)                                          // 1 DMUL
    MEASURE(x = 1.0 / x)                                                // 2 DDIV (IEEE)
    MEASURE(asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x)))       // 3 rcp.approx.f64
    MEASURE(x = __shfl_xor_sync(0xffffffffu, x, 1))                     // 4 SHFL double
    MEASURE(asm volatile("redux.sync.max.u32 %0, %0, 0xffffffff;" : "+r"(u)))  // 5 REDUX
    MEASURE(u = u * 3u + 1u)                                            // 6 IMAD
    MEASURE(y = (x > y) ? x : y * 1.0000001)                            // 7 DSETP+select+DMUL
    MEASURE(u = __shfl_xor_sync(0xffffffffu, u, 1))                     // 8 SHFL u32
    MEASURE(x = fabs(x) + 1e-300)                                       // 9 DADD
    __shared__ double sm[64];
    sm[threadIdx.x] = x;
    __syncthreads();
    MEASURE(x = sm[(int)(x) & 31] + 0.0)                                // 10 LDS + DADD
    MEASURE(__syncthreads())                                            // 11 BAR (1 warp)
    out[threadIdx.x] = x + y + u;
}
int main() {
    double *o; long long *c;
    cudaMalloc(&o, 1024 * 8); cudaMalloc(&c, 64 * 8);
    k<<<1, 32>>>(o, c, 1.5, 3); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.5, 3); cudaDeviceSynchronize();
    long long h[64]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
    const char *names[] = {"DFMA", "DMUL", "DDIV(IEEE 1/x)", "rcp.approx.f64", "SHFL.f64(2x)", "REDUX.u32", "IMAD",
                           "DSETP+sel+DMUL", "SHFL.u32", "DADD", "LDS+DADD", "BAR.SYNC(1 warp)"};
    for (int i = 0; i < 12; ++i) printf("%-18s %6.1f cycles/op\n", names[i], (double)h[i] / N);
    return 0;
}
