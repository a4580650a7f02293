// K4 (fp32 rows): the full fp64 leaf scan and the early-abandoning variants
// (LF_SCAN_VARIANT = full | ea2 | ea3; the default is the int8-bounded scan in scan_q8.cu).
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
        const int4 tk = s.tasks[t];             // (query, leaf slot, chunk) from expand_tasks_kernel
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

// Early-abandoning scan, v2 (m % 64 == 0).  A task's rows are read in three
// phases so that the loads that matter are issued with maximum memory-level
// parallelism:
//   phase 0 (k = 1 and no best-so-far yet): 16 rows are scanned in full to get
//            an upper bound on the task's best distance;
//   phase 1: the FIRST 64 dims (256 B) of every row, 8 rows in flight per
//            half-warp, partial sums kept in smem;
//   phase 2: rows whose partial already exceeds the threshold are dropped --
//            the remaining 768 B of those rows are never fetched from HBM;
//   phase 3: survivors are finished piece by piece, abandoning as they go.
// Threshold = round-start bound (tree.py:207: d <= bsf is kept) and, for k = 1,
// the best full distance seen in the task, both with a 1e-12 relative margin.
template <int NCH>
__global__ void __launch_bounds__(SCAN_THREADS, 3) scan_ea2_kernel(RoundState s, lf_index idx,
                                                                   const float* __restrict__ queries) {
    constexpr int M = NCH * 64;
    constexpr int U = 8;
    constexpr double kMargin = 1.0 + 1e-12;
    __shared__ double qs[M];
    __shared__ double part[CH];
    __shared__ double sd[CH];
    __shared__ long long sid[CH];
    __shared__ int surv[CH];
    __shared__ int n_surv;
    __shared__ unsigned long long best_bits;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int hl = lane & 15;
    const int slot = warp * 2 + (lane >> 4);
    const long long total = s.chunk_off[s.Q];
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
        const int4 tk = s.tasks[t];             // (query, leaf slot, chunk) from expand_tasks_kernel
        const int64_t q = tk.x;
        const int leaf = tk.y;
        const int c = tk.z;
        const int64_t lbeg = idx.d_leaf_ptr[leaf], lend = idx.d_leaf_ptr[leaf + 1];
        const int64_t r0 = lbeg + (int64_t)c * CH;
        const int nrows = (int)min((int64_t)CH, lend - r0);
        const double bsf = round_bsf(s, q);
        const float* qrow = queries + q * M;
        const float* X0 = idx.d_X + r0 * M;
        for (int i = threadIdx.x; i < M; i += SCAN_THREADS) qs[i] = (double)qrow[i];
        if (threadIdx.x == 0) { n_surv = 0; best_bits = 0x7ff0000000000000ULL; }
        __syncthreads();

        // ---- phase 0: full distances of the first 16 rows when nothing bounds the task
        const bool sample = (s.k == 1) && !(bsf < kInf);
        if (sample) {
            const int r = slot;
            double acc = 0.0;
            if (r < nrows) {
                const float4* rp = reinterpret_cast<const float4*>(X0 + (int64_t)r * M);
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const float4 x = __ldcs(rp + ch * 16 + hl);
                    const double* qq = qs + ch * 64 + hl * 4;
                    double d0 = (double)x.x - qq[0], d1 = (double)x.y - qq[1];
                    double d2 = (double)x.z - qq[2], d3 = (double)x.w - qq[3];
                    acc = __fma_rn(d0, d0, acc); acc = __fma_rn(d1, d1, acc);
                    acc = __fma_rn(d2, d2, acc); acc = __fma_rn(d3, d3, acc);
                }
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            if (r < nrows && hl == 0)
                atomicMin(&best_bits, (unsigned long long)__double_as_longlong(acc));
            __syncthreads();
        }
        double thr2 = bsf < kInf ? bsf * bsf * kMargin : kInf;
        if (sample) thr2 = fmin(thr2, __longlong_as_double((long long)best_bits) * kMargin);

        // ---- phase 1: first 64 dims of every row, U rows in flight per half-warp
        for (int b0 = 0; b0 < nrows; b0 += 16 * U) {
            float4 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = b0 + slot + 16 * u;
                x[u] = r < nrows ? __ldcs(reinterpret_cast<const float4*>(X0 + (int64_t)r * M) + hl)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            const double* qq = qs + hl * 4;
            const double q0 = qq[0], q1 = qq[1], q2 = qq[2], q3 = qq[3];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                double d0 = (double)x[u].x - q0, d1 = (double)x[u].y - q1;
                double d2 = (double)x[u].z - q2, d3 = (double)x[u].w - q3;
                double a = d0 * d0;
                a = __fma_rn(d1, d1, a); a = __fma_rn(d2, d2, a); a = __fma_rn(d3, d3, a);
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                const int r = b0 + slot + 16 * u;
                if (r < nrows && hl == 0) part[r] = a;
            }
        }
        __syncthreads();
        // ---- phase 2: survivors
        for (int r = threadIdx.x; r < nrows; r += SCAN_THREADS) {
            sid[r] = idx.d_row_id[r0 + r];
            if (part[r] > thr2) {
                sd[r] = kInf;
            } else if (NCH == 1) {
                sd[r] = sqrt(part[r]);
            } else {
                surv[atomicAdd(&n_surv, 1)] = r;
            }
        }
        __syncthreads();
        if (s.ea_count != nullptr && threadIdx.x == 0) {
            atomicAdd(&s.ea_count[0], (unsigned long long)nrows);
            atomicAdd(&s.ea_count[1], (unsigned long long)n_surv);
            atomicAdd(&s.ea_count[2], (unsigned long long)((long long)nrows * idx.m * 4));
            atomicAdd(&s.ea_count[3], (unsigned long long)(0));
        }
        // ---- phase 3: finish survivors, one half-warp per row, 4 rows in flight
        if (NCH > 1) {
            const int ns = n_surv;
            double best2 = __longlong_as_double((long long)best_bits);
            for (int b0 = 0; b0 < ns; b0 += 16 * 4) {
                double acc[4];
                bool alive[4];
                int rr[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int jj = b0 + slot + 16 * u;
                    alive[u] = jj < ns;
                    rr[u] = alive[u] ? surv[jj] : 0;
                    acc[u] = 0.0;
                }
                double p[4];
#pragma unroll
                for (int ch = 1; ch < NCH; ++ch) {
                    float4 x[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        x[u] = alive[u] ? __ldcs(reinterpret_cast<const float4*>(X0 + (int64_t)rr[u] * M) + ch * 16 + hl)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                    const double* qq = qs + ch * 64 + hl * 4;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        double d0 = (double)x[u].x - qq[0], d1 = (double)x[u].y - qq[1];
                        double d2 = (double)x[u].z - qq[2], d3 = (double)x[u].w - qq[3];
                        acc[u] = __fma_rn(d0, d0, acc[u]); acc[u] = __fma_rn(d1, d1, acc[u]);
                        acc[u] = __fma_rn(d2, d2, acc[u]); acc[u] = __fma_rn(d3, d3, acc[u]);
                        double v = acc[u];
#pragma unroll
                        for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                        p[u] = (alive[u] ? part[rr[u]] : 0.0) + v;
                    }
                    const double th = s.k == 1 ? fmin(thr2, best2 * kMargin) : thr2;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (alive[u] && p[u] > th) {
                            alive[u] = false;
                            if (hl == 0) sd[rr[u]] = kInf;
                        }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (alive[u]) {
                        if (s.k == 1) best2 = fmin(best2, p[u]);
                        if (hl == 0) sd[rr[u]] = sqrt(p[u]);
                    }
            }
        }
        __syncthreads();
        if (warp == 0) {
            double* cd = s.cand_d + t * s.kc;
            long long* ci = s.cand_i + t * s.kc;
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
                    for (int i = lane; i < nrows; i += 32)
                        if (pair_less(sd[i], sid[i], bd, bi)) { bd = sd[i]; bi = sid[i]; bp = i; }
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

// Early-abandoning scan, v3 (m % 64 == 0): the abandon test is cheap fp32 and
// conservative, the kept distances are exact fp64.
//   phase 1: the first 64 dims of every row in fp32 (8 rows in flight per
//            half-warp, the next batch's loads issued before this batch is
//            reduced).  fp32 rounding of a 64-term sum is < 1e-5 relative, so
//            a row is dropped only if partial32 * (1 - 1e-4) > thr^2 -- its
//            exact distance then certainly exceeds thr;
//   phase 2: every survivor is re-read whole (1 KiB, all four 256-byte pieces
//            in flight at once) and summed exactly in fp64.
// thr = the round-start bound (tree.py:207 keeps d <= bsf) and, for k = 1,
// the best exact distance this CTA has found, shared through smem.
template <int NCH>
__global__ void __launch_bounds__(SCAN_THREADS, 4) scan_ea3_kernel(RoundState s, lf_index idx,
                                                                   const float* __restrict__ queries) {
    constexpr int M = NCH * 64;
    constexpr int U = 8;
    constexpr float kSafe = 1.0f - 1e-4f;
    __shared__ float qf[M];
    __shared__ double sd[CH];
    __shared__ long long sid[CH];
    __shared__ int surv[CH];
    __shared__ int n_surv;
    __shared__ unsigned long long best_bits;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int hl = lane & 15;
    const int slot = warp * 2 + (lane >> 4);
    const long long total = s.chunk_off[s.Q];
    for (long long t = blockIdx.x; t < total; t += gridDim.x) {
        const int4 tk = s.tasks[t];
        const int64_t q = tk.x;
        const int leaf = tk.y;
        const int64_t lbeg = idx.d_leaf_ptr[leaf], lend = idx.d_leaf_ptr[leaf + 1];
        const int64_t r0 = lbeg + (int64_t)tk.z * CH;
        const int nrows = (int)min((int64_t)CH, lend - r0);
        const double bsf = round_bsf(s, q);
        const float* X0 = idx.d_X + r0 * M;
        const float* qrow = queries + q * M;
        for (int i = threadIdx.x; i < M; i += SCAN_THREADS) qf[i] = qrow[i];
        if (threadIdx.x == 0) { n_surv = 0; best_bits = 0x7ff0000000000000ULL; }
        __syncthreads();
        const double thr2 = bsf < kInf ? bsf * bsf : kInf;

        // exact fp64 distance of row r (whole row, 16 lanes, all pieces in flight)
        auto exact_row = [&](int r, bool valid) -> double {
            float4 x[NCH];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                x[ch] = valid ? __ldg(reinterpret_cast<const float4*>(X0 + (int64_t)r * M) + ch * 16 + hl)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            double acc = 0.0;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const float* qq = qf + ch * 64 + hl * 4;
                double d0 = (double)x[ch].x - (double)qq[0], d1 = (double)x[ch].y - (double)qq[1];
                double d2 = (double)x[ch].z - (double)qq[2], d3 = (double)x[ch].w - (double)qq[3];
                acc = __fma_rn(d0, d0, acc); acc = __fma_rn(d1, d1, acc);
                acc = __fma_rn(d2, d2, acc); acc = __fma_rn(d3, d3, acc);
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            return acc;
        };

        // ---- phase 0 (k = 1, nothing bounds the task yet): 16 exact rows for a bound
        if (s.k == 1 && !(bsf < kInf)) {
            const bool v = slot < nrows;
            const double e = exact_row(slot, v);
            if (v && hl == 0) atomicMin(&best_bits, (unsigned long long)__double_as_longlong(e));
            __syncthreads();
        }
        // ---- phase 1: first 64 dims in fp32, software-pipelined loads
        {
            const float q0 = qf[hl * 4], q1 = qf[hl * 4 + 1], q2 = qf[hl * 4 + 2], q3 = qf[hl * 4 + 3];
            float4 cur[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = slot + 16 * u;
                cur[u] = r < nrows ? __ldg(reinterpret_cast<const float4*>(X0 + (int64_t)r * M) + hl)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            for (int b0 = 0; b0 < nrows; b0 += 16 * U) {
                float4 nxt[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int r = b0 + 16 * U + slot + 16 * u;
                    nxt[u] = r < nrows ? __ldg(reinterpret_cast<const float4*>(X0 + (int64_t)r * M) + hl)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                }
                double thr_now = thr2;
                if (s.k == 1) thr_now = fmin(thr_now, __longlong_as_double((long long)best_bits));
                const float thr32 = thr_now < 3.0e38 ? (float)thr_now : 3.4e38f;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float d0 = cur[u].x - q0, d1 = cur[u].y - q1, d2 = cur[u].z - q2, d3 = cur[u].w - q3;
                    float a = d0 * d0;
                    a = fmaf(d1, d1, a); a = fmaf(d2, d2, a); a = fmaf(d3, d3, a);
#pragma unroll
                    for (int o = 8; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                    const int r = b0 + slot + 16 * u;
                    if (r < nrows && hl == 0) {
                        if (a * kSafe > thr32) {
                            sd[r] = kInf;
                        } else {
                            surv[atomicAdd(&n_surv, 1)] = r;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) cur[u] = nxt[u];
            }
        }
        __syncthreads();
        if (s.ea_count != nullptr && threadIdx.x == 0) {
            atomicAdd(&s.ea_count[0], (unsigned long long)nrows);
            atomicAdd(&s.ea_count[1], (unsigned long long)n_surv);
            atomicAdd(&s.ea_count[2], (unsigned long long)((long long)nrows * idx.m * 4));
            atomicAdd(&s.ea_count[3], (unsigned long long)(0));
        }
        // ---- phase 2: survivors, exact fp64 over the whole row
        {
            const int ns = n_surv;
            for (int b0 = 0; b0 < ns; b0 += 16) {
                const int jj = b0 + slot;
                const bool v = jj < ns;
                const int r = v ? surv[jj] : 0;
                const double e = exact_row(r, v);
                if (v && hl == 0) {
                    sd[r] = sqrt(e);
                    if (s.k == 1) atomicMin(&best_bits, (unsigned long long)__double_as_longlong(e));
                }
            }
        }
        __syncthreads();
        if (warp == 0) {
            double* cd = s.cand_d + t * s.kc;
            long long* ci = s.cand_i + t * s.kc;
            for (int i = lane; i < nrows; i += 32) {
                sid[i] = idx.d_row_id[r0 + i];
                if (!(sd[i] <= bsf)) sd[i] = kInf;
            }
            __syncwarp();
            if (s.kc >= nrows) {
                for (int i = lane; i < s.kc; i += 32) {
                    cd[i] = i < nrows ? sd[i] : kInf;
                    ci[i] = (i < nrows && sd[i] != kInf) ? sid[i] : -1;
                }
            } else {
                for (int sel = 0; sel < s.kc; ++sel) {
                    double bd = kInf; long long bi = LLONG_MAX; int bp = -1;
                    for (int i = lane; i < nrows; i += 32)
                        if (pair_less(sd[i], sid[i], bd, bi)) { bd = sd[i]; bi = sid[i]; bp = i; }
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

template <int NCH>
static cudaError_t launch_ea_nch(const RoundState& s, const lf_index& idx, const float* q, bool v3, cudaStream_t st) {
    const int sms = sm_count();
    if (v3) scan_ea3_kernel<NCH><<<sms * 4, SCAN_THREADS, 0, st>>>(s, idx, q);
    else scan_ea2_kernel<NCH><<<sms * 3, SCAN_THREADS, 0, st>>>(s, idx, q);
    return cudaGetLastError();
}

cudaError_t launch_scan_ea_fp32(const RoundState& s, const lf_index& idx, const float* q, bool v3, cudaStream_t st) {
    switch (idx.m / 64) {
        case 1: return launch_ea_nch<1>(s, idx, q, v3, st);
        case 2: return launch_ea_nch<2>(s, idx, q, v3, st);
        case 3: return launch_ea_nch<3>(s, idx, q, v3, st);
        case 4: return launch_ea_nch<4>(s, idx, q, v3, st);
        case 5: return launch_ea_nch<5>(s, idx, q, v3, st);
        case 6: return launch_ea_nch<6>(s, idx, q, v3, st);
        case 7: return launch_ea_nch<7>(s, idx, q, v3, st);
        case 8: return launch_ea_nch<8>(s, idx, q, v3, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lf
