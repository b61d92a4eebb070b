// Resident clusters of C CTAs x 512 threads (<= 128 registers) at a given dynamic shared memory size:
// how many structured-solve items fit one wave for each team width. Usage: ./cluster_occ_probe
#include <cstdio>
__global__ void __launch_bounds__(512, 1) k_dummy(double *o) {
    extern __shared__ double s[];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (o) o[blockIdx.x] = s[(threadIdx.x + 1) % 512];
}
int main() {
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    for (int E : {4, 8, 10, 11, 12, 16}) {
        const int chunk = 512 * E;
        const int C = (32768 + chunk - 1) / chunk;
        for (int nbuf : {3, 4}) {
            size_t smem = (size_t)nbuf * (chunk + chunk / E) * 8;
            if (smem > 227 * 1024) { printf("E=%2d C=%2d nbuf=%d smem %zu KB: too big\n", E, C, nbuf, smem / 1024); continue; }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(C);
            cfg.blockDim = dim3(512);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            int n = 0;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
            printf("E=%2d C=%2d nbuf=%d smem %3zu KB: %d resident clusters (%s)\n", E, C, nbuf, smem / 1024, n,
                   cudaGetErrorString(e));
        }
    }
    return 0;
}
