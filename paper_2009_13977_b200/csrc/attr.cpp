// Per-device kernel attribute bookkeeping (see fasth_internal.h).
#include <map>
#include <mutex>
#include <utility>

#include "fasth_internal.h"

namespace fasthb {

cudaError_t ensure_smem(const void* kernel, size_t bytes, bool nonportable_cluster) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{dev, kernel}];
    if (have >= bytes && have) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    if (nonportable_cluster) {
        e = cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    have = bytes;
    return cudaSuccess;
}

}  // namespace fasthb
