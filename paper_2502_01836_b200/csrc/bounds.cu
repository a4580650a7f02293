// K1: query segment means + node lower bounds over SoA envelopes (HBM-bound).
//
// Reference: summarize.py:44-56 (segment means), summarize.py:97-107 (search
// bound, np.dot -> one fp64 FMA chain over segments), summarize.py:114-122
// (batched bound used by traingen, einsum -> sequential sum of (g*g)*w).
// Both orders are reproduced bit-for-bit so visit orders and counters match.
#include <cub/block/block_radix_sort.cuh>
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

// Fused K1 + K2 for trees of up to 8192 nodes: one CTA per query computes every
// node's search bound (lb_kernel<0> formula) straight into registers and sorts
// the (lb, node id) pairs with a stable block radix sort in shared memory --
// the bound matrix never round-trips through HBM before sorting.
constexpr int FS_THREADS = 512;

template <int ITEMS>
__global__ void __launch_bounds__(FS_THREADS) bounds_sort_kernel(const double* __restrict__ qsumm, lf_index idx,
                                                                 const double* __restrict__ env_min,
                                                                 const double* __restrict__ env_max, int n_env,
                                                                 double* __restrict__ lbs, int* __restrict__ order) {
    using Sort = cub::BlockRadixSort<double, FS_THREADS, ITEMS, int>;
    extern __shared__ __align__(16) uint8_t fs_smem[];
    auto& tmp = *reinterpret_cast<typename Sort::TempStorage*>(fs_smem);
    __shared__ double qs[LF_MAX_SEG];
    __shared__ double ws[LF_MAX_SEG];
    const int64_t q = blockIdx.x;
    const int ns = idx.n_seg;
    if (threadIdx.x < ns) {
        qs[threadIdx.x] = qsumm[q * ns + threadIdx.x];
        ws[threadIdx.x] = (double)idx.seg_width[threadIdx.x];
    }
    __syncthreads();
    double keys[ITEMS];
    int vals[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int node = threadIdx.x * ITEMS + i;          // blocked arrangement: stable sort keeps id order
        if (node < n_env) {
            double acc = 0.0;
            for (int sg = 0; sg < ns; ++sg) {
                const double mn = env_min[(int64_t)sg * n_env + node];
                const double mx = env_max[(int64_t)sg * n_env + node];
                double g = fmax(mn - qs[sg], qs[sg] - mx);
                g = fmax(g, 0.0);
                acc = __fma_rn(__dmul_rn(ws[sg], g), g, acc);
            }
            keys[i] = sqrt(acc);
            vals[i] = node;
        } else {
            keys[i] = kInf;                                // padding sorts last
            vals[i] = INT_MAX;
        }
    }
    Sort(tmp).Sort(keys, vals);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int pos = threadIdx.x * ITEMS + i;
        if (pos < n_env) {
            lbs[q * n_env + pos] = keys[i];
            order[q * n_env + pos] = vals[i];
        }
    }
}

template <int ITEMS>
static int launch_fused(const double* d_qsumm, int64_t Q, const lf_index& idx, int n, double* lbs, int* order,
                        cudaStream_t st) {
    using Sort = cub::BlockRadixSort<double, FS_THREADS, ITEMS, int>;
    const int bytes = (int)sizeof(typename Sort::TempStorage);
    static bool attr = false;
    if (!attr) {
        LF_CUDA(cudaFuncSetAttribute(bounds_sort_kernel<ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        attr = true;
    }
    bounds_sort_kernel<ITEMS><<<(unsigned)Q, FS_THREADS, bytes, st>>>(d_qsumm, idx, idx.d_env_min, idx.d_env_max, n,
                                                                      lbs, order);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

// Segment means + bounds + per-query visit order in as few passes as the tree
// size allows: fused block sort up to 8192 nodes, else bounds kernel + CUB.
int bounds_and_order(const float* d_q, int64_t Q, const lf_index& idx, double* d_qsumm, double* d_lb_scratch,
                     double* d_lbs, int* d_order, cudaStream_t st, int* kernels) {
    const int n = idx.n_nodes;
    if (Q == 0 || n == 0) return LF_OK;
    if (n <= FS_THREADS * 16 && Q <= 0x7fffffff) {
        {
            int64_t tot = Q * idx.n_seg;
            paa_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d_q, Q, idx, d_qsumm);
            LF_CUDA(cudaGetLastError());
        }
        int rc;
        if (n <= FS_THREADS * 4) rc = launch_fused<4>(d_qsumm, Q, idx, n, d_lbs, d_order, st);
        else if (n <= FS_THREADS * 8) rc = launch_fused<8>(d_qsumm, Q, idx, n, d_lbs, d_order, st);
        else rc = launch_fused<16>(d_qsumm, Q, idx, n, d_lbs, d_order, st);
        if (kernels) *kernels += 2;
        return rc;
    }
    int rc = launch_bounds(d_q, Q, idx, idx.d_env_min, idx.d_env_max, n, 0, d_qsumm, d_lb_scratch, st);
    if (rc) return rc;
    if (kernels) *kernels += 4;
    return sort_visit_order(d_lb_scratch, Q, n, d_lbs, d_order, st);
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
