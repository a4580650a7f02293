// Error state and device queries for the C-ABI (include/leafi_b200.h).
#include <cuda_runtime.h>

#include <string>

#include "common.cuh"

namespace lf {

static thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
    return n;
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
