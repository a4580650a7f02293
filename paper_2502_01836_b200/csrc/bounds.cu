// K1: query segment means + node lower bounds over SoA envelopes (HBM-bound).
//
// Reference: summarize.py:44-56 (segment means), summarize.py:97-107 (search
// bound, np.dot -> one fp64 FMA chain over segments), summarize.py:114-122
// (batched bound used by traingen, einsum -> sequential sum of (g*g)*w).
// Both orders are reproduced bit-for-bit so visit orders and counters match.
#include <cub/device/device_segmented_sort.cuh>

#include "bounds.cuh"
#include "common.cuh"

namespace lf {

// One thread per (query, segment).
__global__ void paa_kernel(const float* __restrict__ q, int64_t Q, lf_index idx,
                           double* __restrict__ qsumm) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= Q * idx.n_seg) return;
    int64_t qi = t / idx.n_seg;
    int s = (int)(t - qi * idx.n_seg);
    qsumm[t] = segment_mean(q + qi * idx.m, idx.seg_start[s], idx.seg_width[s]);
}

// lb[q][node] for nodes of one query row; segment means staged in smem.
template <int MODE>
__global__ void lb_kernel(const double* __restrict__ qsumm, int64_t Q, int n_seg, lf_index idx,
                          const double* __restrict__ env_min, const double* __restrict__ env_max,
                          int n_env, double* __restrict__ lb) {
    __shared__ double qs[LF_MAX_SEG];
    __shared__ double ws[LF_MAX_SEG];
    for (int64_t qi = blockIdx.y; qi < Q; qi += gridDim.y) {
        __syncthreads();
        if (threadIdx.x < n_seg) {
            qs[threadIdx.x] = qsumm[qi * n_seg + threadIdx.x];
            ws[threadIdx.x] = (double)idx.seg_width[threadIdx.x];
        }
        __syncthreads();
        for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < n_env;
             node += gridDim.x * blockDim.x) {
            double acc = 0.0;
            for (int s = 0; s < n_seg; ++s) {
                double mn = env_min[(int64_t)s * n_env + node];
                double mx = env_max[(int64_t)s * n_env + node];
                double g = fmax(mn - qs[s], qs[s] - mx);
                g = fmax(g, 0.0);
                if (MODE == 0) {
                    acc = __fma_rn(__dmul_rn(ws[s], g), g, acc);          // np.dot(widths*gap, gap)
                } else {
                    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(g, g), ws[s]));  // einsum qns,qns,s
                }
            }
            lb[qi * n_env + node] = sqrt(acc);
        }
    }
}

int launch_bounds(const float* d_q, int64_t Q, const lf_index& idx, const double* env_min,
                  const double* env_max, int n_env, int mode, double* d_qsumm, double* d_lb,
                  cudaStream_t st) {
    if (Q == 0) return LF_OK;
    {
        int64_t n = Q * idx.n_seg;
        int thr = 256;
        paa_kernel<<<(unsigned)((n + thr - 1) / thr), thr, 0, st>>>(d_q, Q, idx, d_qsumm);
        LF_CUDA(cudaGetLastError());
    }
    if (n_env == 0) return LF_OK;
    dim3 block(256);
    dim3 grid((unsigned)((n_env + 255) / 256), (unsigned)(Q < 65535 ? Q : 65535));
    if (mode == 0)
        lb_kernel<0><<<grid, block, 0, st>>>(d_qsumm, Q, idx.n_seg, idx, env_min, env_max,
                                             n_env, d_lb);
    else
        lb_kernel<1><<<grid, block, 0, st>>>(d_qsumm, Q, idx.n_seg, idx, env_min, env_max,
                                             n_env, d_lb);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

__global__ void iota_rows_kernel(int* __restrict__ v, int64_t Q, int n, int* __restrict__ offs) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < Q * n) v[t] = (int)(t % n);
    if (t <= Q) offs[t] = (int)(t * n);
}

// Per-query stable sort of (lb, node id): the heap pop order of tree.py:256-275
// (child lb >= parent lb and child id > parent id, so the heap is a sort).
int sort_visit_order(const double* d_lb, int64_t Q, int n, double* d_lb_sorted, int* d_order,
                     cudaStream_t st) {
    if (Q == 0 || n == 0) return LF_OK;
    LF_REQUIRE(Q * (int64_t)n < (int64_t)INT32_MAX, "query batch too large for one sort");
    Scratch ids, offs, tmp;
    LF_CUDA(ids.alloc(sizeof(int) * Q * n, st));
    LF_CUDA(offs.alloc(sizeof(int) * (Q + 1), st));
    int64_t cnt = Q * n > Q + 1 ? Q * n : Q + 1;
    iota_rows_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(ids.as<int>(), Q, n, offs.as<int>());
    LF_CUDA(cudaGetLastError());
    size_t bytes = 0;
    LF_CUDA(cub::DeviceSegmentedSort::StableSortPairs(
        nullptr, bytes, d_lb, d_lb_sorted, ids.as<int>(), d_order, (int)(Q * n), (int)Q,
        offs.as<int>(), offs.as<int>() + 1, st));
    LF_CUDA(tmp.alloc(bytes, st));
    LF_CUDA(cub::DeviceSegmentedSort::StableSortPairs(
        tmp.p, bytes, d_lb, d_lb_sorted, ids.as<int>(), d_order, (int)(Q * n), (int)Q,
        offs.as<int>(), offs.as<int>() + 1, st));
    return LF_OK;
}

}  // namespace lf

extern "C" int lf_bounds(const float* d_queries, int64_t Q, const lf_index* idx,
                         const double* d_env_min, const double* d_env_max, int32_t n_env,
                         int32_t lb_mode, double* d_qsumm, double* d_lb, void* stream) {
    LF_REQUIRE(idx != nullptr, "idx is NULL");
    LF_REQUIRE(idx->n_seg >= 1 && idx->n_seg <= LF_MAX_SEG, "bad segment count");
    LF_REQUIRE(lb_mode == 0 || lb_mode == 1, "lb_mode must be 0 or 1");
    return lf::launch_bounds(d_queries, Q, *idx, d_env_min, d_env_max, n_env, lb_mode, d_qsumm,
                             d_lb, lf::as_stream(stream));
}

extern "C" int lf_paa_device(const float* d_values, int64_t n, int32_t m, int32_t n_seg, double* d_out,
                             void* stream) {
    LF_REQUIRE(n_seg >= 1 && n_seg <= m && n_seg <= LF_MAX_SEG, "num_segments must be in [1, length]");
    if (n == 0) return LF_OK;
    lf_index idx{};
    idx.m = m;
    idx.n_seg = n_seg;
    const int base = m / n_seg, rem = m % n_seg;
    for (int i = 0, s = 0; i < n_seg; ++i) {
        idx.seg_width[i] = base + (i < rem ? 1 : 0);
        idx.seg_start[i] = s;
        s += idx.seg_width[i];
    }
    const int64_t total = n * n_seg;
    lf::paa_kernel<<<(unsigned)((total + 255) / 256), 256, 0, lf::as_stream(stream)>>>(d_values, n, idx, d_out);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
