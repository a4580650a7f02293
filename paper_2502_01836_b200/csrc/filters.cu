// K3: learned-filter inference for every (query, filter) pair.
//
// Reference: MlpModel.forward (mlp.py:90-95), y = b2 + W2 . relu(x W1 + b1) in
// fp32, called lazily per visited filtered leaf (tree.py:278-286).  Here every
// (query, filter) prediction is produced eagerly in one launch; since visit
// order does not depend on filters (tree.py:1-8, F1), eager evaluation yields
// the same prune decisions.
//
// Batch invariance (enhanced.py:283-285): each output's reduction
// order depends only on (m, f) -- never on Q, the tile a query lands in or
// the launch grid -- so calibration-time and search-time predictions are
// bit-identical.
//
// v1: fp32 SIMT register-tiled GEMM (CUDA-core FFMA).  BM=64 queries x BN=128
// hidden units per CTA, BK=16, 4x8 outputs per thread; the hidden activations
// never leave registers: bias, rectifier and the W2 dot product are fused in
// the epilogue.
#include "common.cuh"

namespace lf {

constexpr int FBM = 64, FBN = 128, FBK = 16, FTHREADS = 256;

__global__ void __launch_bounds__(FTHREADS) filter_kernel(
    const float* __restrict__ X, int64_t Q, int m, const float* __restrict__ W1,
    const float* __restrict__ b1, const float* __restrict__ W2, const float* __restrict__ b2,
    int F, float* __restrict__ pred) {
    __shared__ float Xs[FBK][FBM + 4];
    __shared__ float Ws[FBK][FBN];
    const int f = blockIdx.y;
    const int64_t q0 = (int64_t)blockIdx.x * FBM;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const float* W1f = W1 + (int64_t)f * m * m;
    const float* b1f = b1 + (int64_t)f * m;
    const float* W2f = W2 + (int64_t)f * m;

    float part[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j0 = 0; j0 < m; j0 += FBN) {
        float acc[4][8];
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
        for (int k0 = 0; k0 < m; k0 += FBK) {
            // X tile [64 q][16 k] -> Xs[k][q]
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                int li = tid + e * FTHREADS;          // 0..1023
                int qq = li >> 4, kk = li & 15;
                int64_t qg = q0 + qq;
                int kg = k0 + kk;
                Xs[kk][qq] = (qg < Q && kg < m) ? X[qg * m + kg] : 0.f;
            }
            // W1 tile [16 k][128 j]
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                int li = tid + e * FTHREADS;          // 0..2047
                int kk = li >> 7, jj = li & 127;
                int kg = k0 + kk, jg = j0 + jj;
                Ws[kk][jj] = (kg < m && jg < m) ? W1f[(int64_t)kg * m + jg] : 0.f;
            }
            __syncthreads();
#pragma unroll
            for (int kk = 0; kk < FBK; ++kk) {
                float a[4], b[8];
#pragma unroll
                for (int r = 0; r < 4; ++r) a[r] = Xs[kk][ty * 4 + r];
#pragma unroll
                for (int c = 0; c < 8; ++c) b[c] = Ws[kk][tx + 16 * c];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 8; ++c) acc[r][c] = __fmaf_rn(a[r], b[c], acc[r][c]);
            }
            __syncthreads();
        }
        // epilogue: h = relu(acc + b1), part += h * W2  (fixed c order)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            int j = j0 + tx + 16 * c;
            if (j < m) {
                float bj = b1f[j], wj = W2f[j];
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    float h = fmaxf(__fadd_rn(acc[r][c], bj), 0.f);
                    part[r] = __fmaf_rn(h, wj, part[r]);
                }
            }
        }
    }
    // reduce over the 16 tx lanes (fixed butterfly order)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        float v = part[r];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
        part[r] = v;
    }
    if (tx == 0) {
        float bb = b2[f];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            int64_t qg = q0 + ty * 4 + r;
            if (qg < Q) pred[qg * F + f] = __fadd_rn(part[r], bb);
        }
    }
}

}  // namespace lf

extern "C" int lf_filter_predict(const float* d_queries, int64_t Q, int32_t m, const float* d_W1,
                                 const float* d_b1, const float* d_W2, const float* d_b2,
                                 int32_t F, float* d_pred, void* stream) {
    LF_REQUIRE(Q >= 0 && m >= 1 && F >= 0, "bad sizes");
    if (Q == 0 || F == 0) return LF_OK;
    LF_REQUIRE(F <= 65535, "at most 65535 filters per launch");
    dim3 grid((unsigned)((Q + lf::FBM - 1) / lf::FBM), (unsigned)F);
    lf::filter_kernel<<<grid, lf::FTHREADS, 0, lf::as_stream(stream)>>>(d_queries, Q, m, d_W1, d_b1,
                                                                       d_W2, d_b2, F, d_pred);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
