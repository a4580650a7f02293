// Error state and device queries for the C-ABI (include/leafi_b200.h).
#include <cuda_runtime.h>

#include <mutex>
#include <set>
#include <string>
#include <tuple>

#include "common.cuh"

namespace lf {

static thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

void keep_pool_warm() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_dev = dev;
}

int sm_count() {
    static thread_local int cached_dev = -1, cached = 0;
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && dev == cached_dev) return cached;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    cached_dev = dev;
    cached = n;
    return n;
}

cudaError_t smem_optin_impl(const void* fn, int bytes) {
    static std::mutex mu;
    static std::set<std::tuple<const void*, int, int>> done;   // (kernel, device, bytes)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const auto key = std::make_tuple(fn, dev, bytes);
    {
        std::lock_guard<std::mutex> g(mu);
        if (done.count(key)) return cudaSuccess;
    }
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    done.insert(key);
    return cudaSuccess;
}

}  // namespace lf

extern "C" {

const char* lf_last_error(void) { return lf::g_last_error.c_str(); }

int lf_version(void) { return 1; }

int lf_device_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return n;
}

}  // extern "C"
