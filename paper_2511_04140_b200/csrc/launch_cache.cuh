// launch_cache.cuh -- per-device caches of launch configuration state, so a compress or
// decompress call issues no attribute / occupancy queries once warmed up (small inputs
// are launch-bound, and a CUDA graph capture must not see them).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>

namespace fb200 {

namespace launch_cache_detail {
inline std::mutex& lock() {
    static std::mutex m;
    return m;
}
}  // namespace launch_cache_detail

// raise the kernel's dynamic shared memory limit to at least `bytes` (only grows).  The
// 48 KB default bounds static + dynamic smem together, so there is no shortcut below it
// (a 47 KB walker launch beside 1 KB of static smem failed with "invalid argument").
inline cudaError_t ensure_dynamic_smem(const void* kern, uint32_t bytes) {
    if (bytes <= 16u * 1024u) return cudaSuccess;     // + static smem stays below 48 KB
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    std::lock_guard<std::mutex> g(launch_cache_detail::lock());
    static std::map<std::pair<int, const void*>, uint32_t> set;
    uint32_t& have = set[{dev, kern}];
    if (bytes <= have) return cudaSuccess;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes))) return e;
    have = bytes;
    return cudaSuccess;
}

// resident blocks per SM for (kernel, block size, dynamic smem) and the SM count
inline cudaError_t resident_blocks(const void* kern, int threads, uint32_t smem, int* per_sm, int* sms) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e) return e;
    std::lock_guard<std::mutex> g(launch_cache_detail::lock());
    static std::map<std::tuple<int, const void*, int, uint32_t>, std::pair<int, int>> memo;
    const auto key = std::make_tuple(dev, kern, threads, smem);
    auto it = memo.find(key);
    if (it == memo.end()) {
        int b = 0, n = 0;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem))) return e;
        if ((e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev))) return e;
        it = memo.emplace(key, std::make_pair(b, n)).first;
    }
    *per_sm = it->second.first;
    *sms = it->second.second;
    return cudaSuccess;
}

}  // namespace fb200
