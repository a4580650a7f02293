// K4 (fp32 rows): the full fp64 leaf scan (series.py:142-146) -- traces, and
// indexes without an int8 shadow (the default bounded scans are scan_q8.cu /
// scan_pq.cu; LF_SCAN_VARIANT=full forces this one).
#include <climits>

#include <cuda_fp16.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "round.cuh"
#include "tc.cuh"

namespace lf {

// ---------------------------------------------------------------- scan ----
// Each lane owns VEC float4 slots of the series (slot v = lane + 32*u), so one
// warp reads a row with fully coalesced 128-bit loads.
template <int VEC>
__device__ inline void load_query(const float* qrow, int m4, int lane, double (&qv)[VEC][4]) {
#pragma unroll
    for (int u = 0; u < VEC; ++u) {
        int v = lane + 32 * u;
        float4 x = v < m4 ? reinterpret_cast<const float4*>(qrow)[v] : make_float4(0.f, 0.f, 0.f, 0.f);
        qv[u][0] = x.x; qv[u][1] = x.y; qv[u][2] = x.z; qv[u][3] = x.w;
    }
}

template <int VEC>
__device__ inline double row_partial(const float4 (&x)[VEC], const double (&qv)[VEC][4]) {
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < VEC; ++u) {
        double d0 = (double)x[u].x - qv[u][0];
        double d1 = (double)x[u].y - qv[u][1];
        double d2 = (double)x[u].z - qv[u][2];
        double d3 = (double)x[u].w - qv[u][3];
        acc = __fma_rn(d0, d0, acc);
        acc = __fma_rn(d1, d1, acc);
        acc = __fma_rn(d2, d2, acc);
        acc = __fma_rn(d3, d3, acc);
    }
    return acc;
}

template <int VEC>
__global__ void __launch_bounds__(SCAN_THREADS) scan_kernel(RoundState s, lf_index idx,
                                                            const float* __restrict__ queries) {
    __shared__ double sd[CH];
    __shared__ long long sid[CH];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long total = s.chunk_off[s.Q];
    const int m = idx.m, m4 = m >> 2;
    const bool vec_ok = (m & 3) == 0;
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
        // locate (query, selected leaf, chunk)
        const int4 tk = s.tasks[t];             // (query, leaf slot, chunk) from plan_warp_kernel
        const int64_t q = tk.x;
        const int leaf = tk.y;
        const int c = tk.z;
        const int64_t lbeg = idx.d_leaf_ptr[leaf], lend = idx.d_leaf_ptr[leaf + 1];
        const int64_t r0 = lbeg + (int64_t)c * CH;
        const int nrows = (int)min((int64_t)CH, lend - r0);
        const double bsf = round_bsf(s, q);
        const float* qrow = queries + q * m;

        if (vec_ok) {
            double qv[VEC][4];
            load_query<VEC>(qrow, m4, lane, qv);
            int r = warp;
            for (; r + SCAN_WARPS < nrows; r += 2 * SCAN_WARPS) {
                float4 xa[VEC], xb[VEC];
                const float4* pa = reinterpret_cast<const float4*>(idx.d_X + (r0 + r) * m);
                const float4* pb = reinterpret_cast<const float4*>(idx.d_X + (r0 + r + SCAN_WARPS) * m);
#pragma unroll
                for (int u = 0; u < VEC; ++u) {
                    int v = lane + 32 * u;
                    xa[u] = v < m4 ? __ldcs(pa + v) : make_float4(0.f, 0.f, 0.f, 0.f);
                    xb[u] = v < m4 ? __ldcs(pb + v) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                double a = warp_sum_f64(row_partial<VEC>(xa, qv));
                double b = warp_sum_f64(row_partial<VEC>(xb, qv));
                if (lane == 0) {
                    sd[r] = sqrt(a); sid[r] = idx.d_row_id[r0 + r];
                    sd[r + SCAN_WARPS] = sqrt(b); sid[r + SCAN_WARPS] = idx.d_row_id[r0 + r + SCAN_WARPS];
                }
            }
            for (; r < nrows; r += SCAN_WARPS) {
                float4 xa[VEC];
                const float4* pa = reinterpret_cast<const float4*>(idx.d_X + (r0 + r) * m);
#pragma unroll
                for (int u = 0; u < VEC; ++u) {
                    int v = lane + 32 * u;
                    xa[u] = v < m4 ? __ldcs(pa + v) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                double a = warp_sum_f64(row_partial<VEC>(xa, qv));
                if (lane == 0) { sd[r] = sqrt(a); sid[r] = idx.d_row_id[r0 + r]; }
            }
        } else {
            for (int r = warp; r < nrows; r += SCAN_WARPS) {
                const float* x = idx.d_X + (r0 + r) * m;
                double acc = 0.0;
                for (int i = lane; i < m; i += 32) {
                    double d = (double)x[i] - (double)qrow[i];
                    acc = __fma_rn(d, d, acc);
                }
                acc = warp_sum_f64(acc);
                if (lane == 0) { sd[r] = sqrt(acc); sid[r] = idx.d_row_id[r0 + r]; }
            }
        }
        __syncthreads();
        if (warp == 0) {
            double* cd = s.cand_d + t * s.kc;
            long long* ci = s.cand_i + t * s.kc;
            if (s.want_trace) {
                double mn = kInf;
                for (int i = lane; i < nrows; i += 32) mn = fmin(mn, sd[i]);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                if (lane == 0) s.task_min[t] = mn;
            }
            // drop what cannot enter the top-k (tree.py:207 keeps d <= bsf)
            for (int i = lane; i < nrows; i += 32)
                if (!(sd[i] <= bsf)) sd[i] = kInf;
            __syncwarp();
            if (s.kc >= nrows) {
                for (int i = lane; i < s.kc; i += 32) {
                    cd[i] = i < nrows ? sd[i] : kInf;
                    ci[i] = (i < nrows && sd[i] != kInf) ? sid[i] : -1;
                }
            } else {
                for (int sel = 0; sel < s.kc; ++sel) {
                    double bd = kInf; long long bi = LLONG_MAX; int bp = -1;
                    for (int i = lane; i < nrows; i += 32) {
                        if (pair_less(sd[i], sid[i], bd, bi)) { bd = sd[i]; bi = sid[i]; bp = i; }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        double od = __shfl_xor_sync(0xffffffffu, bd, o);
                        long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
                        int op = __shfl_xor_sync(0xffffffffu, bp, o);
                        if (pair_less(od, oi, bd, bi)) { bd = od; bi = oi; bp = op; }
                    }
                    if (lane == 0) {
                        cd[sel] = bd;
                        ci[sel] = (bd == kInf) ? -1 : bi;
                        if (bp >= 0) { sd[bp] = kInf; sid[bp] = LLONG_MAX; }
                    }
                    __syncwarp();
                }
            }
        }
        __syncthreads();
    }
}

cudaError_t launch_scan_full(const RoundState& s, const lf_index& idx, const float* q, cudaStream_t st) {
    const int grid = sm_count() * 4;
    const int m4 = idx.m / 4;
    if ((idx.m & 3) != 0 || m4 <= 32) scan_kernel<1><<<grid, SCAN_THREADS, 0, st>>>(s, idx, q);
    else if (m4 <= 64) scan_kernel<2><<<grid, SCAN_THREADS, 0, st>>>(s, idx, q);
    else if (m4 <= 128) scan_kernel<4><<<grid, SCAN_THREADS, 0, st>>>(s, idx, q);
    else if (m4 <= 256) scan_kernel<8><<<grid, SCAN_THREADS, 0, st>>>(s, idx, q);
    else return cudaErrorInvalidValue;
    return cudaGetLastError();
}

}  // namespace lf
