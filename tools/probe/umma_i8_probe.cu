// Probe: tcgen05.mma kind::i8 with the SWIZZLE_NONE layouts of csrc/tc05.cuh.
//   A = K-major u8 [M=128][K] (core matrices: LBO = 128 B along K, SBO = KB bytes * 8 along M)
//   B = MN-major u8 [K][N]     (core matrices: SBO = 128 B along N, LBO = N * 8 bytes along K)
// Checks D = A B (s32) against the host, then times back-to-back MMAs on every SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o umma_i8_probe umma_i8_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../paper_2509_20500_b200/csrc/tc05.cuh"

using namespace spl;

constexpr int M = 128;

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(done) : "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(ph) : "memory");
}

// image offsets
__host__ __device__ inline size_t a_off(int m, int k, int K) {     // K-major: [m/8][k/16][m%8][k%16]
    return (size_t)(m / 8) * (K / 16) * 128 + (size_t)(k / 16) * 128 + (m % 8) * 16 + (k % 16);
}
__host__ __device__ inline size_t b_off(int k, int n, int N) {     // MN-major: [k/8][n/16][k%8][n%16]
    return (size_t)(k / 8) * (N / 16) * 128 + (size_t)(n / 16) * 128 + (k % 8) * 16 + (n % 16);
}

template <int N>
__global__ void k_check(const uint8_t *A, const uint8_t *B, int K, int32_t *D, int reps) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t *sa = sm, *sb = sm + M * K;
    for (int i = threadIdx.x; i < M * K; i += blockDim.x) sa[i] = A[i];
    for (int i = threadIdx.x; i < K * N; i += blockDim.x) sb[i] = B[i];
    tc05::fence_proxy_async_smem();
    if (threadIdx.x == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (threadIdx.x / 32 == 0) tc05::alloc<(N < 32 ? 32 : N)>(&tbase);
    tc05::fence_before();
    __syncthreads();
    tc05::fence_after();
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t sa_u = (uint32_t)__cvta_generic_to_shared(sa), sb_u = (uint32_t)__cvta_generic_to_shared(sb);
        const uint32_t id = tc05::idesc_i8(M, N, true);
        for (int r = 0; r < reps; ++r)
            for (int s = 0; s < K / 32; ++s) {
                const uint64_t ad = tc05::smem_desc(sa_u + s * 256, 128, (K / 16) * 128);
                const uint64_t bd = tc05::smem_desc(sb_u + s * 4 * (N / 16) * 128, (N / 16) * 128, 128);
                tc05::mma_i8(tm, ad, bd, id, (r | s) ? 1u : 0u);
            }
        tc05::commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc05::fence_after();
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (D) {
        for (int c = 0; c < N; c += 32) {
            uint32_t r[32];
            tc05::ld32x32(tm + ((uint32_t)(32 * w) << 16) + c, r);
            tc05::wait_ld();
            for (int i = 0; i < 32; ++i) D[(size_t)(32 * w + lane) * N + c + i] = (int32_t)r[i];
        }
    }
    tc05::fence_before();
    __syncthreads();
    if (w == 0) tc05::dealloc<(N < 32 ? 32 : N)>(tm);
}

template <int N>
int run(int K) {
    std::vector<uint8_t> a((size_t)M * K), b((size_t)K * N), ai(a.size()), bi(b.size());
    srand(1234 + K + N);
    for (auto &x : a) x = rand() & 255;
    for (auto &x : b) x = rand() & 255;
    for (int m = 0; m < M; ++m)
        for (int k = 0; k < K; ++k) ai[a_off(m, k, K)] = a[(size_t)m * K + k];
    for (int k = 0; k < K; ++k)
        for (int n = 0; n < N; ++n) bi[b_off(k, n, N)] = b[(size_t)k * N + n];
    uint8_t *dA, *dB;
    int32_t *dD;
    cudaMalloc(&dA, ai.size()); cudaMalloc(&dB, bi.size()); cudaMalloc(&dD, sizeof(int32_t) * M * N);
    cudaMemcpy(dA, ai.data(), ai.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, bi.data(), bi.size(), cudaMemcpyHostToDevice);
    const int smem = M * K + K * N;
    cudaFuncSetAttribute(k_check<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_check<N><<<1, 128, smem>>>(dA, dB, K, dD, 1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e)); return 1; }
    std::vector<int32_t> d((size_t)M * N);
    cudaMemcpy(d.data(), dD, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            long s = 0;
            for (int k = 0; k < K; ++k) s += (long)a[(size_t)m * K + k] * b[(size_t)k * N + n];
            if (s != d[(size_t)m * N + n]) {
                if (bad < 5) printf("  mismatch m=%d n=%d got %d want %ld\n", m, n, d[(size_t)m * N + n], s);
                ++bad;
            }
        }
    printf("N=%d K=%d: %s (%ld bad)\n", N, K, bad ? "FAIL" : "ok", bad);
    // throughput: every SM, reps x K/32 MMAs
    if (!bad) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        const int reps = 4000;
        cudaEvent_t t0, t1;
        cudaEventCreate(&t0); cudaEventCreate(&t1);
        k_check<N><<<sms, 128, smem>>>(dA, dB, K, nullptr, 10);
        cudaEventRecord(t0);
        k_check<N><<<sms, 128, smem>>>(dA, dB, K, nullptr, reps);
        cudaEventRecord(t1);
        cudaEventSynchronize(t1);
        float ms = 0;
        cudaEventElapsedTime(&ms, t0, t1);
        const double ops = 2.0 * M * N * K * (double)reps * sms;
        printf("  %d SMs x %d x (M%d N%d K%d): %.3f ms = %.1f TOPS\n", sms, reps * K / 32, M, N, 32, ms, ops / ms / 1e9);
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dD);
    return bad != 0;
}

int main() {
    int f = 0;
    f |= run<128>(32);
    f |= run<128>(128);
    f |= run<64>(64);
    f |= run<256>(64);
    return f;
}
