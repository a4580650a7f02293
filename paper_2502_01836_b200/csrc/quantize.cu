// int8 shadow of the collection for the bounded leaf scan (scan_q8_kernel).
//
// Per row: scale = max|x| / 127, code_i = rint(x_i / scale) in [-127, 127],
// xx = sum code_i^2 and qerr = ||scale * code - x||_2 computed in fp64 and
// rounded up to fp32.  By the triangle inequality, for every query q
//     ||x - q|| - qerr  <=  ||scale * code - q||  <=  ||x - q|| + qerr,
// so the scan can drop a row from 1/4 of its bytes when the bound already
// exceeds the best-so-far, and re-read the exact fp32 row otherwise.
#include "common.cuh"

namespace lf {

__global__ void quantize_kernel(const float* __restrict__ X, int64_t n, int m, int8_t* __restrict__ X8,
                                float4* __restrict__ meta) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= n) return;
    const float* x = X + r * m;
    float mx = 0.f;
    for (int i = lane; i < m; i += 32) mx = fmaxf(mx, fabsf(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float s = mx > 0.f ? mx / 127.f : 1.f;
    int sq = 0;
    double err = 0.0;
    for (int i = lane; i < m; i += 32) {
        float c = rintf(x[i] / s);
        c = fminf(fmaxf(c, -127.f), 127.f);
        const int ci = (int)c;
        X8[r * m + i] = (int8_t)ci;
        sq += ci * ci;
        const double e = (double)s * (double)ci - (double)x[i];
        err = __fma_rn(e, e, err);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        err += __shfl_xor_sync(0xffffffffu, err, o);
    }
    if (lane == 0)    // sq <= 512 * 127^2 < 2^24: exact in fp32
        meta[r] = make_float4(s, (float)sq, __double2float_ru(sqrt(err) * (1.0 + 1e-9) + 1e-30), 0.f);
}

}  // namespace lf

extern "C" int lf_quantize_rows(const float* d_X, int64_t n, int32_t m, int8_t* d_X8, float* d_qmeta,
                                void* stream) {
    LF_REQUIRE(n >= 0 && m >= 1, "bad sizes");
    if (n == 0) return LF_OK;
    lf::quantize_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, lf::as_stream(stream)>>>(
        d_X, n, m, d_X8, reinterpret_cast<float4*>(d_qmeta));
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
