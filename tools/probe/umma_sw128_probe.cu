// Probe: tcgen05.mma kind::i8 with B = MN-major u8 in the 128-byte-swizzle layout a tensor-map TMA
// box of [KB rows][128 B] leaves in shared memory (16-byte chunk c of row k at chunk c ^ (k % 8)),
// boxes of consecutive 128-byte column spans KB * 128 bytes apart. Descriptor (CuTe's canonical
// MN-major SW128 layout ((T,8,m),(8,k)):((1,T,LBO),(8T,SBO))): LBO = next 128-byte MN span (a box),
// SBO = next 8 K-rows (1024 B), layout type 2. A = K-major SWIZZLE_NONE as in umma_i8_probe.cu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_sw128_probe umma_sw128_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2509_20500_b200/csrc/tc05.cuh"

using namespace spl;

constexpr int M = 128, N = 256, KB = 64;

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
}
__host__ __device__ inline size_t a_off(int m, int k, int K) {     // K-major: [m/8][k/16][m%8][k%16]
    return (size_t)(m / 8) * (K / 16) * 128 + (size_t)(k / 16) * 128 + (m % 8) * 16 + (k % 16);
}
__host__ __device__ inline size_t b_off(int k, int n) {             // TMA SW128 boxes
    return (size_t)(n / 128) * KB * 128 + (size_t)k * 128 + ((((n % 128) / 16) ^ (k % 8)) * 16) + n % 16;
}
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return tc05::smem_desc(saddr, lbo, sbo) | (2ull << 61);
}

__global__ void k_check(const uint8_t *A, const uint8_t *B, int32_t *D, int variant) {
    extern __shared__ __align__(1024) uint8_t sm_raw[];
    uint8_t *sm = sm_raw + ((1024 - ((uint32_t)__cvta_generic_to_shared(sm_raw) & 1023)) & 1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t *sb = sm, *sa = sm + KB * N;
    for (int i = threadIdx.x; i < M * KB; i += blockDim.x) sa[i] = A[i];
    for (int i = threadIdx.x; i < KB * N; i += blockDim.x) sb[i] = B[i];
    tc05::fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (threadIdx.x / 32 == 0) tc05::alloc<256>(&tbase);
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t sa_u = (uint32_t)__cvta_generic_to_shared(sa), sb_u = (uint32_t)__cvta_generic_to_shared(sb);
        const uint32_t id = tc05::idesc_i8(M, N, true);
        for (int s = 0; s < KB / 32; ++s) {
            const uint64_t ad = tc05::smem_desc(sa_u + s * 256, 128, (KB / 16) * 128);
            const uint32_t lbo = variant == 0 ? KB * 128 : 1024, sbo = variant == 0 ? 1024 : KB * 128;
            const uint64_t bd = desc_sw128(sb_u + s * 32 * 128, lbo, sbo);
            tc05::mma_i8(tm, ad, bd, id, s ? 1u : 0u);
        }
        tc05::commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc05::fence_after();
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int c = 0; c < N; c += 32) {
        uint32_t r[32];
        tc05::ld32x32(tm + ((uint32_t)(32 * w) << 16) + c, r);
        tc05::wait_ld();
        for (int i = 0; i < 32; ++i) D[(size_t)(32 * w + lane) * N + c + i] = (int32_t)r[i];
    }
    tc05::fence_before();
    __syncthreads();
    if (w == 0) tc05::dealloc<256>(tm);
}

int main() {
    std::vector<uint8_t> a((size_t)M * KB), b((size_t)KB * N), ai(a.size()), bi(b.size());
    srand(4321);
    for (auto &x : a) x = rand() & 255;
    for (auto &x : b) x = rand() & 255;
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < KB; ++k) ai[a_off(m, k, KB)] = a[(size_t)m * KB + k];
    for (int k = 0; k < KB; ++k)
        for (int n = 0; n < N; ++n) bi[b_off(k, n)] = b[(size_t)k * N + n];
    uint8_t *dA, *dB;
    int32_t *dD;
    cudaMalloc(&dA, ai.size()); cudaMalloc(&dB, bi.size()); cudaMalloc(&dD, sizeof(int32_t) * M * N);
    cudaMemcpy(dA, ai.data(), ai.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, bi.data(), bi.size(), cudaMemcpyHostToDevice);
    const int smem = M * KB + KB * N + 1024;
    cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int fails = 0;
    for (int variant = 0; variant < 2; ++variant) {
        cudaMemset(dD, 0, sizeof(int32_t) * M * N);
        k_check<<<1, 128, smem>>>(dA, dB, dD, variant);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) { printf("variant %d: CUDA error %s\n", variant, cudaGetErrorString(e)); return 2; }
        std::vector<int32_t> d((size_t)M * N);
        cudaMemcpy(d.data(), dD, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost);
        long bad = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                long s = 0;
                for (int k = 0; k < KB; ++k) s += (long)a[(size_t)m * KB + k] * b[(size_t)k * N + n];
                if (s != d[(size_t)m * N + n]) ++bad;
            }
        printf("variant %d (LBO=%s, SBO=%s): %s (%ld bad of %d)\n", variant, variant ? "1024" : "box", variant ? "box" : "1024",
               bad ? "FAIL" : "ok", bad, M * N);
        fails += bad != 0;
    }
    return fails == 2;
}
