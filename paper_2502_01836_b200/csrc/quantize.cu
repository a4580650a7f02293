// int8 shadow of the collection for the bounded leaf scan (scan_q8_kernel).
//
// Per row: scale = max|x| / 127, code_i = rint(x_i / scale) in [-127, 127],
// xx = sum code_i^2 and qerr = ||scale * code - x||_2 computed in fp64 and
// rounded up to fp32.  By the triangle inequality, for every query q
//     ||x - q|| - qerr  <=  ||scale * code - q||  <=  ||x - q|| + qerr,
// so the scan can drop a row from 1/4 of its bytes when the bound already
// exceeds the best-so-far, and re-read the exact fp32 row otherwise.
#include "common.cuh"
#include "tc.cuh"

namespace lf {

__global__ void quantize_kernel(const float* __restrict__ X, int64_t n, int m, int8_t* __restrict__ X8,
                                float4* __restrict__ meta) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= n) return;
    const float* x = X + r * m;
    const int m8 = (m + 31) / 32 * 32;            // code rows are zero-padded to a multiple of 32
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
        X8[r * m8 + i] = (int8_t)ci;
        sq += ci * ci;
        const double e = (double)s * (double)ci - (double)x[i];
        err = __fma_rn(e, e, err);
    }
    for (int i = m + lane; i < m8; i += 32) X8[r * m8 + i] = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
        err += __shfl_xor_sync(0xffffffffu, err, o);
    }
    if (lane == 0)    // sq <= 512 * 127^2 < 2^24: exact in fp32
        meta[r] = make_float4(s, (float)sq, __double2float_ru(sqrt(err) * (1.0 + 1e-9) + 1e-30), 0.f);
}

// Query codes, quantised once per batch exactly like the rows:
// codes [Q][MP] (zero-padded to MP = 256-multiple), meta [Q] = {scale, qq, err, 0}.
__global__ void quantize_queries_kernel(const float* __restrict__ queries, int64_t Q, int M, int MP,
                                        int8_t* __restrict__ qc, float4* __restrict__ qm) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= Q) return;
    const float* x = queries + q * M;
    float mx = 0.f;
    for (int i = lane; i < M; i += 32) mx = fmaxf(mx, fabsf(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float sq = mx > 0.f ? mx / 127.f : 1.f;
    int qq = 0;
    double err = 0.0;
    for (int i = lane; i < MP; i += 32) {
        int c = 0;
        if (i < M) {
            c = (int)fminf(fmaxf(rintf(x[i] / sq), -127.f), 127.f);
            const double e = (double)sq * (double)c - (double)x[i];
            err = __fma_rn(e, e, err);
        }
        qc[q * MP + i] = (int8_t)c;
        qq += c * c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        qq += __shfl_xor_sync(0xffffffffu, qq, o);
        err += __shfl_xor_sync(0xffffffffu, err, o);
    }
    if (lane == 0) qm[q] = make_float4(sq, (float)qq, __double2float_ru(sqrt(err) * (1.0 + 1e-9) + 1e-30), 0.f);
}

int quantize_queries(const float* d_q, int64_t Q, int m, int mp, int8_t* d_codes, float4* d_meta, cudaStream_t st) {
    if (Q == 0) return LF_OK;
    quantize_queries_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(d_q, Q, m, mp, d_codes, d_meta);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

int encode_map_2d(CUtensorMap* map, CUtensorMapDataType dtype, const void* base, int64_t rows, int64_t cols,
                  int64_t row_stride_bytes, int box_cols, int box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    if (!fn) return fail(LF_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_stride_bytes};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(LF_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return LF_OK;
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

