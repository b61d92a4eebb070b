// Per-device host state of the library: kernel attributes and device properties are per
// (device, context), so every cache here is keyed by the current device ordinal. A process that
// drives several GPUs (cudaSetDevice / torch.cuda.set_device between calls) gets each kernel's
// attributes set once on every device it launches on. Never called inside a stream capture.
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"

namespace spl {

int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        (void)cudaGetLastError();
        d = 0;
    }
    return d;
}

// Streaming multiprocessors of the current device (MIG / MPS partitions report fewer than 148).
int device_sm_count() {
    static std::mutex mu;
    static std::map<int, int> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    const auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) {
        (void)cudaGetLastError();
        return kNumSMsDefault;     // not cached: the next call asks again
    }
    cache[dev] = n;
    return n;
}

bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("SPLIDAR_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

cudaError_t func_attrs_once(const void *fn, int max_dyn_smem, bool nonportable_cluster) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void *, int, bool>, cudaError_t> done;
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_tuple(dev, fn, max_dyn_smem, nonportable_cluster);
    const auto it = done.find(key);
    if (it != done.end()) return it->second;
    cudaError_t e = cudaSuccess;
    if (max_dyn_smem > 0) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn_smem);
    if (e == cudaSuccess && nonportable_cluster)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e == cudaSuccess) done[key] = e;
    return e;
}

}  // namespace spl
