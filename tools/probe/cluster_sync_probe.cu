// Latency of barrier.cluster (cg::this_cluster().sync()) vs cluster size, 512-thread CTAs, and of a
// DSMEM round trip (remote store + barrier). Usage: ./cluster_sync_probe
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, double *out) {
    cg::cluster_group cl = cg::this_cluster();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) cl.sync();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
}

__global__ void k_syncthreads(int iters, double *out) {
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
}

int main() {
    double *d, h;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(k_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int C : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C);
        cfg.blockDim = dim3(512);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, k_sync, 2000, d);
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("cluster %2d x 512: cl.sync %.0f cycles (%s)\n", C, h, cudaGetErrorString(cudaGetLastError()));
    }
    k_syncthreads<<<1, 512>>>(2000, d);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads 512: %.0f cycles\n", h);
    return 0;
}
