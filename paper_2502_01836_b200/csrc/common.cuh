// Shared helpers for the sm_100a LeaFi kernels.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/leafi_b200.h"

namespace lf {

int fail(int code, const std::string& msg);

#define LF_CUDA(expr)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return ::lf::fail(LF_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define LF_REQUIRE(cond, msg)                                  \
    do {                                                       \
        if (!(cond)) return ::lf::fail(LF_EINVAL, (msg));      \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// Opt a kernel into more than 48 KB of dynamic shared memory.  The attribute
// belongs to the device context, so it is set once per (kernel, device, size),
// not once per process: one process driving several GPUs sets it on each.
cudaError_t smem_optin_impl(const void* fn, int bytes);
template <class F>
inline cudaError_t smem_optin(F* fn, int bytes) { return smem_optin_impl(reinterpret_cast<const void*>(fn), bytes); }

// Keep the stream-ordered allocator's pool warm across calls: by default the
// pool trims to zero at every synchronisation, which turns each search call's
// scratch into fresh cudaMalloc/cudaFree (and implicit syncs).
void keep_pool_warm();

// Stream-ordered scratch allocation that frees itself.
struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    Scratch() = default;
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
    cudaError_t alloc(size_t bytes, cudaStream_t st) {
        keep_pool_warm();
        s = st;
        return cudaMallocAsync(&p, bytes ? bytes : 16, st);
    }
    template <class T>
    T* as() const { return reinterpret_cast<T*>(p); }
};

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum_DOUBLE) over fp32 inputs promoted to fp64.  np.add.reduceat
// seeds each segment with its first element and adds the pairwise sum of the
// rest: summarize.py:49,56 therefore computes a[s] + pairwise(a[s+1 .. s+w)).
__device__ __host__ inline double np_pairwise_f32(const float* a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += (double)a[i];
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = (double)a[j];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += (double)a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += (double)a[i];
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return np_pairwise_f32(a, n2) + np_pairwise_f32(a + n2, n - n2);
}

// Segment mean as the reference computes it (summarize.py:49).
__device__ __host__ inline double segment_mean(const float* row, int start, int width) {
    double s = (double)row[start] + np_pairwise_f32(row + start + 1, width - 1);
    return s / (double)width;
}

// Segment standard deviation of the EAPCA summary (oracle/leafi_oracle.py eapca):
// sqrt(sum (x_t - mean)^2 / w), the squares added left to right, no FMA.
__device__ __host__ inline double segment_sd(const float* row, int start, int width, double mean) {
    double acc = 0.0;
    for (int t = start; t < start + width; ++t) {
        const double d = (double)row[t] - mean;
#ifdef __CUDA_ARCH__
        acc = __dadd_rn(acc, __dmul_rn(d, d));
#else
        acc = acc + d * d;
#endif
    }
    return sqrt(acc / (double)width);
}

__device__ inline double warp_sum_f64(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (distance, id) lexicographic order: tree.py:212 lexsort((ids, dists)).
__device__ inline bool pair_less(double da, long long ia, double db, long long ib) {
    return da < db || (da == db && ia < ib);
}

constexpr double kInf = __builtin_huge_val();

// Lazy filter inference on the tensor cores (filters_tc.cu): predictions for gathered
// query rows bucketed by filter, written as pred - offset into visit-order records.
int filter_pairs_tc(const float* d_rows, int64_t P, int m, const float* d_W1T, const float* d_b1,
                    const float* d_W2, const float* d_b2, int F, const int4* d_tiles, const int* d_ntiles,
                    const int2* d_dst, const double* d_offset, double* d_adj, int Nn, cudaStream_t st);

// In-search filter inference (filters_tc.cu): the fp16 pack over query rows gathered
// with TMA gather4 from d_xh (fp16 [Q][m], power-of-two exponents d_xexp).
int filter_reach_f16(const __half* d_xh, const int* d_xexp, int64_t Q, int m, const uint16_t* d_W1T_h,
                     const int* d_wexp, const float* d_b1, const float* d_W2, const float* d_b2, int F,
                     const int4* d_tiles, const int* d_ntiles, const int2* d_dst, const double* d_offset,
                     double* d_adj, int Nn, cudaStream_t st);
// fp32 rows -> power-of-two-scaled fp16 rows + exponents (filters_tc.cu).
// mo: output row stride (> m: zero-padded columns; 0 = m)
int rows_to_f16(const float* d_X, int64_t rows, int m, __half* d_out, int* d_exps, cudaStream_t st, int mo = 0);

}  // namespace lf
