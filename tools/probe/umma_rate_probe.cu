// Probe: tcgen05.mma kind::i8 issue/throughput for the shapes of power_i8.cu, descriptors
// precomputed, 8 MMAs per loop iteration, every SM busy. Prints TOPS for
//   (a) M128 N128 K32 into one accumulator, (b) into 4 accumulators (the GEMV's p-slices),
//   (c) M128 N256 K32 into 2 accumulators, (d) M128 N64 K32 into 8 accumulators.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_rate_probe umma_rate_probe.cu
#include <cstdio>
#include "../../paper_2509_20500_b200/csrc/tc05.cuh"
using namespace spl;

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
}

template <int N, int NACC>
__global__ void k_rate(int reps, int *sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 128 * 64 + 64 * N; i += blockDim.x) sm[i] = (uint8_t)i;
    tc05::fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (threadIdx.x / 32 == 0) tc05::alloc<512>(&tbase);
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    if (threadIdx.x == 0) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm), sb = sa + 128 * 64;
        const uint32_t id = tc05::idesc_i8(128, N, true);
        uint64_t ad[2], bd[2];
        for (int s = 0; s < 2; ++s) {
            ad[s] = tc05::smem_desc(sa + s * 256, 128, 512);
            bd[s] = tc05::smem_desc(sb + s * 4 * (N / 16) * 128, (N / 16) * 128, 128);
        }
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                tc05::mma_i8(tbase + (uint32_t)((i % NACC) * N), ad[i & 1], bd[i & 1], id, r | (i >= NACC));
        }
        tc05::commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc05::fence_after();
    if (threadIdx.x == 0 && reps < 0) *sink = 1;
    tc05::fence_before();
    __syncthreads();
    if (threadIdx.x / 32 == 0) tc05::dealloc<512>(tbase);
}

template <int N, int NACC>
void run(const char *name) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 128 * 64 + 64 * N;
    cudaFuncSetAttribute(k_rate<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_rate<N, NACC><<<sms, 128, smem>>>(100, nullptr);
    cudaEvent_t t0, t1;
    cudaEventCreate(&t0); cudaEventCreate(&t1);
    const int reps = 20000;
    cudaEventRecord(t0);
    k_rate<N, NACC><<<sms, 128, smem>>>(reps, nullptr);
    cudaEventRecord(t1);
    cudaEventSynchronize(t1);
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    const double ops = 2.0 * 128 * N * 32 * 8.0 * reps * sms;
    printf("%-34s %8.3f ms  %7.1f TOPS  %6.1f ns per MMA per SM  (%s)\n", name, ms, ops / ms / 1e9,
           ms * 1e6 / (8.0 * reps), cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<128, 1>("M128 N128 K32, 1 accumulator");
    run<128, 4>("M128 N128 K32, 4 accumulators");
    run<256, 2>("M128 N256 K32, 2 accumulators");
    run<64, 8>("M128 N64 K32, 8 accumulators");
    return 0;
}
