// tma.cuh -- 2D TMA (cp.async.bulk.tensor) helpers for row-major fp64 matrices.
// Host: tensor maps are encoded through the driver entry point cuTensorMapEncodeTiled (no
// link-time libcuda dependency).  Device: one elected thread issues box loads (completion
// via mbarrier transaction bytes) and box stores (bulk groups).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include "common.cuh"

namespace frob {

// Matrix of `rows` x `cols` doubles with row stride `ld_doubles`, box = box_rows x 16 doubles
// (128 bytes, 128-byte swizzle).  Out-of-range box elements load as zero and are not stored.
cudaError_t tma_map_rows128(CUtensorMap *map, const void *base, long long rows, long long cols, long long ld_doubles,
                            int box_rows);

// byte offset of 16-byte chunk c (0..7) of row r inside a 128B-swizzled box (1024-byte aligned)
FROB_DEV unsigned swz128(int r, int c) { return (unsigned)(r * 128 + ((c ^ (r & 7)) << 4)); }

FROB_DEV void tma_load_2d(unsigned smem_dst, const CUtensorMap *map, int c0, int c1, unsigned mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_dst),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(mbar)
        : "memory");
}
FROB_DEV void tma_store_2d(const CUtensorMap *map, int c0, int c1, unsigned smem_src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<unsigned long long>(map)),
                 "r"(c0), "r"(c1), "r"(smem_src)
                 : "memory");
}
FROB_DEV void tma_store_commit_wait() {
    asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group 0;" ::: "memory");
}
FROB_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
FROB_DEV void mbar_arrive_expect_tx(unsigned addr, unsigned tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(addr), "r"(tx) : "memory");
}
FROB_DEV void mbar_wait_cta(unsigned addr, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\n"
        "W_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

}  // namespace frob
