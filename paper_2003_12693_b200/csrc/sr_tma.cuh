// sr_tma.cuh -- TMA tile loads (cp.async.bulk.tensor) completed on an mbarrier, for the stencil
// kernels' halo tiles (sm_100a).  Host side: cuTensorMapEncodeTiled through the runtime's driver
// entry point (no -lcuda).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace srsb {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// Checked build (-DSRSB_CHECKS, tools/checked_lib.py): every staged shared-memory access named with
// SRSB_CHK(ptr, bytes) must lie inside the launch's dynamic shared memory, else the kernel prints the
// site and traps.  Stands in for compute-sanitizer's memcheck on the shared-memory side, which this
// pool does not allow.  Compiles to nothing in the normal build.
#ifdef SRSB_CHECKS
static __device__ __noinline__ void srsb_chk_fail(const char* file, int line, uint32_t off, uint32_t n, uint32_t size) {
    printf("SRSB_CHECKS: %s:%d shared access [%u, %u) outside dynamic shared memory of %u bytes (block %d,%d,%d thread %d,%d)\n",
           file, line, off, off + n, size, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x, threadIdx.y);
    __trap();
}
__device__ __forceinline__ void srsb_chk(const void* p, uint32_t n, const char* file, int line) {
    extern __shared__ unsigned char srsb_chk_base[];
    uint32_t size;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(size));
    const uint32_t off = smem_u32(p) - smem_u32(srsb_chk_base);
    if (off > size || n > size - off) srsb_chk_fail(file, line, off, n, size);
}
#define SRSB_CHK(p, n) ::srsb::srsb_chk((p), (n), __FILE__, __LINE__)
#else
#define SRSB_CHK(p, n) ((void)0)
#endif

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "SRSB_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra SRSB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// box {c0 .. c0 + box0) x {c1 .. c1 + box1) of plane c2 -> dst (dense, box0 fastest); coordinates
// outside the tensor are zero-filled by the TMA unit.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
        "[%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// L2 prefetch of the same box (no shared memory, no completion): the later tma_load_3d of the box hits L2.
__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

// L2 prefetch of contiguous bytes (multiple of 16, 16-byte aligned); no completion mechanism
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// contiguous bytes (multiple of 16, 16-byte aligned) global -> shared, completing on bar
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

}  // namespace srsb
