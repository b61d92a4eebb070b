// Inline-PTX helpers shared by the libsplidar kernels (sm_90+ / sm_100a): mbarriers and 1-D TMA
// bulk copies (cp.async.bulk). Internal; not part of the C ABI and not shared with oracle/.
#pragma once
#include <stdint.h>

namespace spl {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Device clock (ns) and the GEMV launch timer (PowerArgs::ktime): the first CTA to start lowers
// ktime[0], the last to finish raises ktime[1]; k_power_check adds ktime[1] - ktime[0] to ktime[2]
// and counts the launch in ktime[3] (the kernel's own duration, measured on the device).
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void ktime_start(unsigned long long *kt) {
    if (kt) atomicMin(kt, global_ns());
}
__device__ __forceinline__ void ktime_end(unsigned long long *kt) {
    if (kt) atomicMax(kt + 1, global_ns());
}

// Programmatic dependent launch (PDL). pdl_trigger: this CTA lets the next kernel of the stream /
// graph edge be scheduled now (its CTAs may become resident while this grid still runs); pdl_wait:
// blocks until every prerequisite grid has completed and its memory operations are visible. Every
// kernel that may be launched as a PDL secondary calls pdl_wait before its first global access
// (read or write), so completion stays transitive along a chain of PDL edges. Both are no-ops in a
// launch without the PDL attribute / programmatic edge.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
// Address of the same shared-memory variable in CTA `rank` of the cluster (shared::cluster window).
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
// 8-byte store into another CTA's shared memory whose arrival is counted (8 bytes of tx) on that
// CTA's mbarrier: the receiver's wait on the mbarrier both synchronises and makes the data visible.
__device__ __forceinline__ void st_async_f64(uint32_t raddr, double v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 ::"r"(raddr), "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on the mbarrier (bytes % 16 == 0, both
// addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace spl
