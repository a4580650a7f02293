// K5: exact query x leaf minimum-distance matrix for training-data generation.
//
// Reference: collect_targets (traingen.py:147-220) computes, per selected leaf,
// batch_distances(queries, leaf_block).min(axis=1) (series.py:127-139: direct
// subtract-square-sum form, fp64), and collect_local_targets (:135-144) does
// the same for each leaf's own local queries.
//
// v1: fp64 SIMT register-tiled direct form -- (x - q) is exact in fp64 for
// fp32-exact inputs and every square is exact, so only the summation order
// differs from numpy (|rel err| ~ 1e-16); identical rows give exactly 0.0
// (test_traingen.py:53-57,76-82).  Tile: 64 queries x 64 rows x 32 dims in
// smem, 4x4 (query, row) pairs per thread, per-leaf min folded with a 64-bit
// atomicMin on the bit pattern of the non-negative squared distance.
#include <vector>

#include "common.cuh"

namespace lf {

constexpr int MBM = 64, MBN = 64, MBK = 32, MTHREADS = 256;

struct Tile {
    int64_t q_begin, q_end;     // query rows [q_begin, q_end)
    int64_t r_begin, r_end;     // data rows [r_begin, r_end)
};

// Accumulates acc[4][4] = sum_i (q_i - x_i)^2 for this thread's pairs.
__device__ inline void tile_sq_dists(const float* __restrict__ Qm, const float* __restrict__ X,
                                     int m, const Tile& t, double (&Qs)[MBK][MBM + 1],
                                     double (&Xs)[MBK][MBN + 1], double (&acc)[4][4]) {
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < m; k0 += MBK) {
#pragma unroll
        for (int e = 0; e < (MBM * MBK) / MTHREADS; ++e) {     // 8
            int li = tid + e * MTHREADS;
            int rr = li >> 5, kk = li & 31;
            int kg = k0 + kk;
            int64_t qg = t.q_begin + rr, xg = t.r_begin + rr;
            Qs[kk][rr] = (qg < t.q_end && kg < m) ? (double)Qm[qg * m + kg] : 0.0;
            Xs[kk][rr] = (xg < t.r_end && kg < m) ? (double)X[xg * m + kg] : 0.0;
        }
        __syncthreads();
        const int kmax = min(MBK, m - k0);
        for (int kk = 0; kk < kmax; ++kk) {
            double qa[4], xb[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) qa[a] = Qs[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) xb[b] = Xs[kk][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    double d = xb[b] - qa[a];
                    acc[a][b] = __fma_rn(d, d, acc[a][b]);
                }
        }
        __syncthreads();
    }
}

// min over this tile's rows for each query, folded into out[q * ldo] (bits of d^2).
__device__ inline void fold_min(const Tile& t, const double (&acc)[4][4], double* out, int64_t ldo) {
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double v = kInf;
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if (t.r_begin + tx + 16 * b < t.r_end) v = fmin(v, acc[a][b]);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
        int64_t qg = t.q_begin + ty + 16 * a;
        if (tx == 0 && qg < t.q_end && v != kInf)
            atomicMin(reinterpret_cast<unsigned long long*>(out + qg * ldo),
                      (unsigned long long)__double_as_longlong(v));
    }
}

// grid: x = row chunk within a leaf, y = query tile, z = selected leaf.
__global__ void __launch_bounds__(MTHREADS) leaf_min_kernel(const float* __restrict__ Qm,
                                                            int64_t Q, lf_index idx,
                                                            const int* __restrict__ sel,
                                                            double* __restrict__ dl, int64_t ldd) {
    __shared__ double Qs[MBK][MBM + 1];
    __shared__ double Xs[MBK][MBN + 1];
    const int s = blockIdx.z;
    const int leaf = sel[s];
    const int64_t lb = idx.d_leaf_ptr[leaf], le = idx.d_leaf_ptr[leaf + 1];
    Tile t;
    t.r_begin = lb + (int64_t)blockIdx.x * MBN;
    if (t.r_begin >= le) return;
    t.r_end = min(le, t.r_begin + MBN);
    t.q_begin = (int64_t)blockIdx.y * MBM;
    t.q_end = min(Q, t.q_begin + MBM);
    double acc[4][4];
    tile_sq_dists(Qm, idx.d_X, idx.m, t, Qs, Xs, acc);
    fold_min(t, acc, dl + s, ldd);
}

// grid: x = row chunk, y = query tile within the group, z = group.
__global__ void __launch_bounds__(MTHREADS) local_min_kernel(const float* __restrict__ Qm,
                                                             lf_index idx,
                                                             const long long* __restrict__ qptr,
                                                             const int* __restrict__ gleaf,
                                                             double* __restrict__ dl) {
    __shared__ double Qs[MBK][MBM + 1];
    __shared__ double Xs[MBK][MBN + 1];
    const int g = blockIdx.z;
    const int leaf = gleaf[g];
    const int64_t lb = idx.d_leaf_ptr[leaf], le = idx.d_leaf_ptr[leaf + 1];
    Tile t;
    t.r_begin = lb + (int64_t)blockIdx.x * MBN;
    t.q_begin = qptr[g] + (int64_t)blockIdx.y * MBM;
    if (t.r_begin >= le || t.q_begin >= qptr[g + 1]) return;
    t.r_end = min(le, t.r_begin + MBN);
    t.q_end = min((int64_t)qptr[g + 1], t.q_begin + MBM);
    double acc[4][4];
    tile_sq_dists(Qm, idx.d_X, idx.m, t, Qs, Xs, acc);
    fold_min(t, acc, dl, 1);
}

__global__ void __launch_bounds__(MTHREADS) pair_dist_kernel(const float* __restrict__ Qm, int64_t Q,
                                                             const float* __restrict__ B, int64_t nB,
                                                             int m, double* __restrict__ out) {
    __shared__ double Qs[MBK][MBM + 1];
    __shared__ double Xs[MBK][MBN + 1];
    Tile t;
    t.r_begin = (int64_t)blockIdx.x * MBN;
    t.r_end = min(nB, t.r_begin + MBN);
    t.q_begin = (int64_t)blockIdx.y * MBM;
    t.q_end = min(Q, t.q_begin + MBM);
    double acc[4][4];
    tile_sq_dists(Qm, B, m, t, Qs, Xs, acc);
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            int64_t qg = t.q_begin + ty + 16 * a, xg = t.r_begin + tx + 16 * b;
            if (qg < t.q_end && xg < t.r_end) out[qg * nB + xg] = sqrt(acc[a][b]);
        }
}

__global__ void fill_inf_kernel(double* p, int64_t rows, int64_t cols, int64_t ld) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < rows * cols) p[(t / cols) * ld + (t % cols)] = kInf;
}

__global__ void sqrt_kernel(double* p, int64_t rows, int64_t cols, int64_t ld) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < rows * cols) {
        double* e = p + (t / cols) * ld + (t % cols);
        *e = sqrt(*e);
    }
}

static unsigned blocks_for(int64_t n) { return (unsigned)((n + 255) / 256); }

}  // namespace lf

extern "C" int lf_leaf_min_dist(const float* d_queries, int64_t Q, const lf_index* idx,
                                const int32_t* d_leaf_sel, int32_t S, double* d_dl, int64_t ldd,
                                void* stream) {
    using namespace lf;
    LF_REQUIRE(idx != nullptr && Q >= 0 && S >= 0 && ldd >= S, "bad arguments");
    if (Q == 0 || S == 0) return LF_OK;
    LF_REQUIRE(S <= 65535, "at most 65535 leaves per launch");
    cudaStream_t st = as_stream(stream);
    fill_inf_kernel<<<blocks_for(Q * S), 256, 0, st>>>(d_dl, Q, S, ldd);
    LF_CUDA(cudaGetLastError());
    const int64_t qt = (Q + MBM - 1) / MBM;
    const int64_t rt = (idx->max_leaf_rows + MBN - 1) / MBN;
    LF_REQUIRE(qt <= 65535, "too many queries for one launch (split the batch)");
    dim3 grid((unsigned)rt, (unsigned)qt, (unsigned)S);
    leaf_min_kernel<<<grid, MTHREADS, 0, st>>>(d_queries, Q, *idx, d_leaf_sel, d_dl, ldd);
    LF_CUDA(cudaGetLastError());
    sqrt_kernel<<<blocks_for(Q * S), 256, 0, st>>>(d_dl, Q, S, ldd);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

extern "C" int lf_local_min_dist(const float* d_queries, const lf_index* idx, const int64_t* h_qptr,
                                 const int32_t* h_group_leaf, int32_t n_groups, double* d_dl,
                                 void* stream) {
    using namespace lf;
    LF_REQUIRE(idx != nullptr && n_groups >= 0, "bad arguments");
    if (n_groups == 0) return LF_OK;
    LF_REQUIRE(n_groups <= 65535, "at most 65535 groups per launch");
    cudaStream_t st = as_stream(stream);
    const int64_t Q = h_qptr[n_groups];
    int64_t max_group = 0;
    for (int g = 0; g < n_groups; ++g) max_group = std::max<int64_t>(max_group, h_qptr[g + 1] - h_qptr[g]);
    if (Q == 0) return LF_OK;
    Scratch dq, dg;
    LF_CUDA(dq.alloc(sizeof(long long) * (n_groups + 1), st));
    LF_CUDA(dg.alloc(sizeof(int) * n_groups, st));
    LF_CUDA(cudaMemcpyAsync(dq.p, h_qptr, sizeof(long long) * (n_groups + 1), cudaMemcpyHostToDevice, st));
    LF_CUDA(cudaMemcpyAsync(dg.p, h_group_leaf, sizeof(int) * n_groups, cudaMemcpyHostToDevice, st));
    fill_inf_kernel<<<blocks_for(Q), 256, 0, st>>>(d_dl, Q, 1, 1);
    LF_CUDA(cudaGetLastError());
    const int64_t qt = (max_group + MBM - 1) / MBM;
    const int64_t rt = (idx->max_leaf_rows + MBN - 1) / MBN;
    LF_REQUIRE(qt <= 65535, "group too large");
    dim3 grid((unsigned)rt, (unsigned)qt, (unsigned)n_groups);
    local_min_kernel<<<grid, MTHREADS, 0, st>>>(d_queries, *idx, dq.as<long long>(), dg.as<int>(), d_dl);
    LF_CUDA(cudaGetLastError());
    sqrt_kernel<<<blocks_for(Q), 256, 0, st>>>(d_dl, Q, 1, 1);
    LF_CUDA(cudaGetLastError());
    // the host arrays were copied asynchronously from pageable memory: the copy is
    // staged before cudaMemcpyAsync returns, so no sync is needed here.
    return LF_OK;
}

extern "C" int lf_batch_distances(const float* d_queries, int64_t Q, const float* d_block, int64_t B,
                                  int32_t m, double* d_out, void* stream) {
    using namespace lf;
    LF_REQUIRE(Q >= 0 && B >= 0 && m >= 1, "bad sizes");
    if (Q == 0 || B == 0) return LF_OK;
    const int64_t qt = (Q + MBM - 1) / MBM, bt = (B + MBN - 1) / MBN;
    LF_REQUIRE(qt <= 65535, "too many queries for one launch (split the batch)");
    dim3 grid((unsigned)bt, (unsigned)qt);
    pair_dist_kernel<<<grid, MTHREADS, 0, as_stream(stream)>>>(d_queries, Q, d_block, B, m, d_out);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
