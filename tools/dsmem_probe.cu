// dsmem_probe.cu -- latency of the per-column cluster exchange used by lu3 (debug tool).
// Variants: (a) st.async + mbarrier complete_tx, (b) cluster barrier only, (c) __syncthreads only,
// plus REDUX / SHFL chains.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/dsmem_probe tools/dsmem_probe.cu
#include <cstdio>
#include <cooperative_groups.h>
#include "../paper_2208_01239_b200/csrc/common.cuh"
namespace cg = cooperative_groups;
using namespace frob;
unsigned long long &frob::launch_counter() { static unsigned long long c = 0; return c; }

FROB_DEV void st_async16(unsigned raddr, const uint4 v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(rbar)
                 : "memory");
}
FROB_DEV void mbar_arrive_expect(unsigned addr, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(tx) : "memory");
}
FROB_DEV bool mbar_try(unsigned addr, unsigned parity) {
    unsigned ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    return ok;
}
FROB_DEV bool mbar_test(unsigned addr, unsigned parity) {
    unsigned ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    return ok;
}

constexpr int CS = 8, NT = 256, NW = NT / 32, REC = 160, ITERS = 2000;

template <int MODE>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(NT, 1) xchg(long long *out, int nrec_push) {
    __shared__ __align__(16) unsigned char rec[2][CS * NW][REC];
    __shared__ __align__(8) unsigned long long mbar[2];
    cg::cluster_group cl = cg::this_cluster();
    const int crank = cl.block_rank(), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) { mbar_init(smem_u32(&mbar[0]), 1); mbar_init(smem_u32(&mbar[1]), 1); mbar_init_fence(); }
    cl.sync();
    const unsigned my_rec = mapa_u32(smem_u32(&rec[0][0][0]), lane % CS);
    const unsigned my_bar = mapa_u32(smem_u32(&mbar[0]), lane % CS);
    unsigned long long acc = 0;
    long long t0 = clock64();
    for (int j = 0; j < ITERS; ++j) {
        const int s = j & 1;
        if (MODE == 0) {
            if (tid == 0) mbar_arrive_expect(smem_u32(&mbar[s]), CS * NW * nrec_push * 16);
            if (lane < CS) {
                const unsigned off = (unsigned)(((s * CS * NW) + crank * NW + warp) * REC);
                uint4 v = make_uint4(j, acc, 1, 2);
                for (int c = 0; c < nrec_push; ++c) st_async16(my_rec + off + c * 16, v, my_bar + s * 8);
            }
            while (!mbar_try(smem_u32(&mbar[s]), (j >> 1) & 1)) { }
            acc += *reinterpret_cast<unsigned *>(&rec[s][lane][0]);
        } else if (MODE == 1) {
            if (lane < CS) {
                const unsigned off = (unsigned)(((s * CS * NW) + crank * NW + warp) * REC);
                asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(my_rec + off), "r"(j) : "memory");
            }
            asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            acc += *reinterpret_cast<unsigned *>(&rec[s][lane][0]);
        } else if (MODE == 2) {
            if (lane == 0) *reinterpret_cast<unsigned *>(&rec[s][warp][0]) = j;
            __syncthreads();
            acc += *reinterpret_cast<unsigned *>(&rec[s][lane % NW][0]);
        } else if (MODE == 3) {
            // REDUX chain x3
            unsigned v = (unsigned)(acc + tid);
            unsigned r;
            asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
            asm volatile("redux.sync.max.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(r + lane));
            asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(r + lane));
            acc += r;
        } else if (MODE == 4) {
            // 16 double shuffles from a runtime lane
            double x[16];
            for (int c = 0; c < 16; ++c) x[c] = (double)(acc + c);
            const int src = (int)(acc & 31);
            double sum = 0;
#pragma unroll
            for (int c = 0; c < 16; ++c) sum += __shfl_sync(0xffffffffu, x[c], src);
            acc += (unsigned long long)sum;
        } else if (MODE == 5) {
            // LDS -> LDS dependent chain
            unsigned *r = reinterpret_cast<unsigned *>(&rec[0][0][0]);
            acc = r[(acc + tid) & 63];
        }
    }
    long long t1 = clock64();
    if (tid == 0 && crank == 0) out[0] = (t1 - t0) / ITERS;
    if (acc == 0xdeadbeef) out[1] = acc;
    cl.sync();
}

int main() {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    const char *names[] = {"st.async x1 + mbarrier", "cluster barrier", "__syncthreads", "3 x REDUX chain",
                           "16 x SHFL.f64 (runtime lane)", "dependent LDS"};
    for (int m = 0; m < 6; ++m) {
        for (int np : {1, 10}) {
            if (m > 0 && np > 1) continue;
            for (int rep = 0; rep < 2; ++rep) {
                switch (m) {
                    case 0: xchg<0><<<CS, NT>>>(d, np); break;
                    case 1: xchg<1><<<CS, NT>>>(d, np); break;
                    case 2: xchg<2><<<CS, NT>>>(d, np); break;
                    case 3: xchg<3><<<CS, NT>>>(d, np); break;
                    case 4: xchg<4><<<CS, NT>>>(d, np); break;
                    case 5: xchg<5><<<CS, NT>>>(d, np); break;
                }
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            }
            printf("%-32s pushes/lane=%2d : %lld cycles/iter (%s)\n", names[m], np, h[0], cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
