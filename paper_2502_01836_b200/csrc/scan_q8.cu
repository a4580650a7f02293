// K4 (default): the TMA-pipelined int8-bounded leaf scan.
#include <climits>

#include <cuda_fp16.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "round.cuh"
#include "tc.cuh"

namespace lf {

// MINB resident CTAs per SM (register and shared-memory budgets follow).  Each CTA
// works one task at a time and its tail (survivor list, exact re-check, per-task top-k)
// is separated by CTA barriers, so more resident CTAs keep the memory pipe busy between
// tasks: m <= 256 runs 4 per SM (C5, 100M x 96, k = 10: 46.3 -> 31.3 ms per batch;
// 25M x 256 k = 10: 10.29 -> 10.11 ms), longer rows keep 2.
template <int M32, int MINB = 2>
struct Q8Cfg {
    static constexpr int M = M32 * 32;                      // code row stride (roundup(m, 32))
    static constexpr int P = (M + 255) / 256;              // 256-code passes per row (16 codes per lane)
    static constexpr int CODE_BYTES = Q8_ROWS * M;
    static constexpr int META_OFF = CODE_BYTES;             // 64 x float4 row metadata
    static constexpr int QC_OFF = META_OFF + Q8_ROWS * 16;  // query codes (first stage of a task)
    static constexpr int QM_OFF = QC_OFF + P * 256;         // query metadata float4
    static constexpr int HDR_OFF = QM_OFF + 16;             // {r0 (i64), q (i32), nrows (i32)}
    static constexpr int STAGE_BYTES = (HDR_OFF + 16 + 127) / 128 * 128;
    static constexpr int BUDGET = MINB == 2 ? 81920 : MINB == 3 ? 45056 : 32768;
    static constexpr int STAGES = (BUDGET / CODE_BYTES) < 2 ? 2 : ((BUDGET / CODE_BYTES) > 8 ? 8 : BUDGET / CODE_BYTES);
    static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
    static constexpr int LO_OFF = BAR_OFF + 2 * STAGES * 8;
    static constexpr int SR_OFF = LO_OFF + CH * 4;
    static constexpr int SD_OFF = SR_OFF + CH * 4;
    static constexpr int HI_OFF = SD_OFF + CH * 8;                   // upper ends (k > 1)
    static constexpr int HIST_OFF = HI_OFF + CH * 4;                 // 256-bin radix-select histogram
    static constexpr int MISC_OFF = HIST_OFF + 256 * 4;
    static constexpr int SMEM = MISC_OFF + 32;
};

template <int M32, int MINB = 2>
__global__ void __launch_bounds__(Q8_THREADS, MINB) scan_q8_kernel(RoundState s, lf_index idx,
                                                                   const float* __restrict__ queries,
                                                                   const int8_t* __restrict__ qcodes,
                                                                   const float4* __restrict__ qmeta) {
    using Cfg = Q8Cfg<M32, MINB>;
    constexpr int NCH = (M32 * 32 + 63) / 64;          // 64-float chunks of the fp32 row (exact re-check)
    constexpr int M = Cfg::M, P = Cfg::P, S = Cfg::STAGES;
    extern __shared__ __align__(128) unsigned char q8_smem[];
    unsigned char* stages = q8_smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(q8_smem + Cfg::BAR_OFF);
    uint64_t* empty = full + S;
    float* lo_s = reinterpret_cast<float*>(q8_smem + Cfg::LO_OFF);
    int* surv_r = reinterpret_cast<int*>(q8_smem + Cfg::SR_OFF);
    double* surv_d = reinterpret_cast<double*>(q8_smem + Cfg::SD_OFF);
    unsigned int* hi_bits = reinterpret_cast<unsigned int*>(q8_smem + Cfg::MISC_OFF);   // [2], by task parity
    int* n_surv = reinterpret_cast<int*>(hi_bits + 2);                                 // [2]
    unsigned int* sel = reinterpret_cast<unsigned int*>(n_surv + 2);                  // [2] radix-select state
    float* hi_s = reinterpret_cast<float*>(q8_smem + Cfg::HI_OFF);
    int* hist = reinterpret_cast<int*>(q8_smem + Cfg::HIST_OFF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            q8_bar_init(&full[i], 1);
            q8_bar_init(&empty[i], Q8_CONS_WARPS * 32);   // every consumer lane releases itself
        }
        hi_bits[0] = hi_bits[1] = 0x7f800000u;
        n_surv[0] = n_surv[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const long long total = s.chunk_off[s.Q];

    if (warp == 0) {   // ---------------------------------------------- producer
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            int slot = 0;
            uint32_t ph = 0;
            long long t = blockIdx.x;
            int4 tk = t < total ? s.tasks[t] : make_int4(0, 0, 0, 0);
            for (; t < total; t += gridDim.x) {
                const long long tn = t + gridDim.x;
                const int4 tk_next = tn < total ? s.tasks[tn] : make_int4(0, 0, 0, 0);   // prefetch
                const int64_t lend = idx.d_leaf_ptr[tk.y + 1];
                const int64_t r0 = idx.d_leaf_ptr[tk.y] + (int64_t)tk.z * CH;
                const int nrows = (int)min((int64_t)CH, lend - r0);
                for (int j = 0; j < nrows; j += Q8_ROWS) {
                    const int rows = min(Q8_ROWS, nrows - j);
                    q8_wait(&empty[slot], ph ^ 1);
                    unsigned char* dst = stages + slot * Cfg::STAGE_BYTES;
                    uint32_t bytes = (uint32_t)(rows * (M + 16));
                    if (j == 0) {
                        *reinterpret_cast<long long*>(dst + Cfg::HDR_OFF) = r0;
                        *reinterpret_cast<int2*>(dst + Cfg::HDR_OFF + 8) = make_int2(tk.x, nrows);
                        bytes += P * 256 + 16;
                    }
                    q8_expect_tx(&full[slot], bytes);    // release: orders the header stores
                    q8_bulk(dst, idx.d_X8 + (r0 + j) * M, (uint32_t)(rows * M), &full[slot], pol);
                    q8_bulk(dst + Cfg::META_OFF, idx.d_qmeta + (r0 + j) * 4, (uint32_t)(rows * 16), &full[slot], pol);
                    if (j == 0) {
                        q8_bulk(dst + Cfg::QC_OFF, qcodes + (int64_t)tk.x * (P * 256), P * 256, &full[slot], pol);
                        q8_bulk(dst + Cfg::QM_OFF, qmeta + tk.x, 16, &full[slot], pol);
                    }
                    if (++slot == S) { slot = 0; ph ^= 1; }
                }
                tk = tk_next;
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const int cw = warp - 1;
    const int ctid = threadIdx.x - 32;
    // Rows of <= 128 codes (SHORT): 8 lanes per row, 16 codes each, the warp's 8 rows of a
    // stage in two passes of 4; longer rows: 16 lanes per row and 256-code passes, a
    // half-warp's 4 rows summed by a transposing butterfly.
    constexpr bool SHORT = M <= 128;
    const int hl = SHORT ? (lane & 7) : (lane & 15);
    const int rbase = cw * 8 + (lane >> 4) * 4;        // this half-warp's 4 rows of a stage
    const bool b8 = (hl & 8) != 0, b4 = (hl & 4) != 0;
    // row whose total this lane ends with
    const int myrow = SHORT ? cw * 8 + (hl & 1) * 4 + (lane >> 3) : rbase + (b8 ? 2 : 0) + (b4 ? 1 : 0);
    const bool writer = SHORT ? hl < 2 : (hl & 3) == 0;
    int slot = 0;
    uint32_t ph = 0;
    int par = 0;
    for (long long t = blockIdx.x; t < total; t += gridDim.x, par ^= 1) {
        // first stage of the task: header + query codes
        q8_wait(&full[slot], ph);
        const unsigned char* st0 = stages + slot * Cfg::STAGE_BYTES;
        const int64_t r0 = *reinterpret_cast<const long long*>(st0 + Cfg::HDR_OFF);
        const int2 hq = *reinterpret_cast<const int2*>(st0 + Cfg::HDR_OFF + 8);
        const int64_t q = hq.x;
        const int nrows = hq.y;
        const double bsf = round_bsf(s, q);                  // consumed in the tail only
        int qw[P][4];
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int4 v = *reinterpret_cast<const int4*>(st0 + Cfg::QC_OFF + p * 256 + hl * 16);
            qw[p][0] = v.x; qw[p][1] = v.y; qw[p][2] = v.z; qw[p][3] = v.w;
        }
        const float4 qmv = *reinterpret_cast<const float4*>(st0 + Cfg::QM_OFF);
        const float sq = qmv.x, eq = qmv.z;
        const float sq2qq = sq * sq * qmv.y;
        float hmin = __int_as_float(0x7f800000);
        // ---- bounds from the int8 codes, stage by stage
        for (int j = 0; j < nrows; j += Q8_ROWS) {
            if (j > 0) q8_wait(&full[slot], ph);
            const int rows = min(Q8_ROWS, nrows - j);
            const unsigned char* stg = stages + slot * Cfg::STAGE_BYTES;
            int d[4];
            if constexpr (SHORT) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int r = cw * 8 + u * 4 + (lane >> 3);
                    int dot = 0;
                    if (r < rows && hl * 16 < M) {
                        const int4 w = *reinterpret_cast<const int4*>(stg + r * M + hl * 16);
                        dot = __dp4a(w.x, qw[0][0], dot);
                        dot = __dp4a(w.y, qw[0][1], dot);
                        dot = __dp4a(w.z, qw[0][2], dot);
                        dot = __dp4a(w.w, qw[0][3], dot);
                    }
                    dot += __shfl_xor_sync(0xffffffffu, dot, 4);
                    dot += __shfl_xor_sync(0xffffffffu, dot, 2);
                    dot += __shfl_xor_sync(0xffffffffu, dot, 1);
                    d[u] = dot;
                }
                d[0] = (hl & 1) ? d[1] : d[0];
            } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int r = rbase + u;
                int dot = 0;
#pragma unroll
                for (int p = 0; p < P; ++p) {
                    if (r < rows && p * 256 + hl * 16 < M) {
                        const int4 w = *reinterpret_cast<const int4*>(stg + r * M + p * 256 + hl * 16);
                        dot = __dp4a(w.x, qw[p][0], dot);
                        dot = __dp4a(w.y, qw[p][1], dot);
                        dot = __dp4a(w.z, qw[p][2], dot);
                        dot = __dp4a(w.w, qw[p][3], dot);
                    }
                }
                d[u] = dot;
            }
            // transposing butterfly over the 16 lanes of the half: 4 row partials -> 1 row total
            {
                const int s0 = b8 ? d[0] : d[2], s1 = b8 ? d[1] : d[3];
                const int k0 = b8 ? d[2] : d[0], k1 = b8 ? d[3] : d[1];
                const int e0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 8);
                const int e1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 8);
                int v = (b4 ? e1 : e0) + __shfl_xor_sync(0xffffffffu, b4 ? e0 : e1, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                d[0] = v;
            }
            }
            if (myrow < rows) {
                const float4 mr = *reinterpret_cast<const float4*>(stg + Cfg::META_OFF + myrow * 16);
                const float sx2xx = mr.x * mr.x * mr.y;
                const float e = mr.z + eq;
                const float d2 = sx2xx + sq2qq - 2.f * (mr.x * sq) * (float)d[0];
                const float tol = 1e-5f * (sx2xx + sq2qq);
                const float lo = (sqrtf(fmaxf(d2 - tol, 0.f)) - e) * (1.f - 1e-6f);
                const float hi = (sqrtf(fmaxf(d2 + tol, 0.f)) + e) * (1.f + 1e-6f);
                hmin = fminf(hmin, hi);
                if (writer) {
                    lo_s[j + myrow] = lo;
                    if (s.k > 1) hi_s[j + myrow] = hi;
                }
            }
            q8_arrive(&empty[slot]);
            if (++slot == S) { slot = 0; ph ^= 1; }
        }
        if (s.k == 1) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) hmin = fminf(hmin, __shfl_xor_sync(0xffffffffu, hmin, o));
            if (lane == 0) atomicMin(&hi_bits[par], __float_as_uint(hmin));
        }
        q8_cons_sync();
        float kth_hi = __int_as_float(0x7f800000);
        if (s.k > 1 && s.kc <= nrows && !(bsf < kInf)) {
            // no k-th best yet: the task's kc-th smallest upper end bounds its kc-th best distance
            // (radix select over the upper ends' bits, which order like the non-negative floats)
            unsigned prefix = 0, mask = 0;
            int rem = s.kc;
            for (int shift = 24; shift >= 0; shift -= 8) {
                hist[ctid] = 0;
                q8_cons_sync();
                for (int r = ctid; r < nrows; r += Q8_CONS) {
                    const unsigned key = __float_as_uint(hi_s[r]);
                    if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
                }
                q8_cons_sync();
                if (cw == 0) {
                    int c[8], sum = 0;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) { c[jj] = hist[lane * 8 + jj]; sum += c[jj]; }
                    int incl = sum;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const int v = __shfl_up_sync(0xffffffffu, incl, d);
                        if (lane >= d) incl += v;
                    }
                    const int excl = incl - sum;
                    if (excl < rem && rem <= incl) {
                        int acc = excl, b = 7;
                        for (int jj = 0; jj < 8; ++jj) {
                            if (acc + c[jj] >= rem) { b = jj; break; }
                            acc += c[jj];
                        }
                        sel[0] = prefix | ((unsigned)(lane * 8 + b) << shift);
                        sel[1] = (unsigned)(rem - acc);
                    }
                }
                q8_cons_sync();
                prefix = sel[0];
                rem = (int)sel[1];
                mask |= 255u << shift;
            }
            kth_hi = __uint_as_float(prefix);
        }
        // ---- survivors
        {
            double thr = bsf;
            if (s.k == 1) thr = fmin(thr, (double)__uint_as_float(hi_bits[par]));
            else thr = fmin(thr, (double)kth_hi);
            const float thr_f = thr < kInf ? __double2float_ru(thr) : __int_as_float(0x7f800000);
            for (int r = ctid; r < nrows; r += Q8_CONS)
                if (lo_s[r] <= thr_f) surv_r[atomicAdd(&n_surv[par], 1)] = r;
        }
        q8_cons_sync();
        const int ns = n_surv[par];
        {   // exact fp64 direct-form distances of the survivors (series.py:142-146); fp32 rows
            // have stride m (the int8 codes are zero-padded to M)
            const int mr = idx.m;
            const float* X0 = idx.d_X + r0 * mr;
            const float* qrow = queries + q * mr;
            const int hslot = cw * 2 + (lane >> 4);
            const int hx = lane & 15;                    // 16 lanes per survivor row
            for (int b0 = 0; b0 < ns; b0 += 16) {
                const int jj = b0 + hslot;
                const bool v = jj < ns;
                const int r = v ? surv_r[jj] : 0;
                float4 x[NCH];
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
                    x[ch] = (v && ch * 64 + hx * 4 < mr)
                                ? __ldg(reinterpret_cast<const float4*>(X0 + (int64_t)r * mr) + ch * 16 + hx)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
                double acc = 0.0;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const float4 qv = ch * 64 + hx * 4 < mr
                                          ? __ldg(reinterpret_cast<const float4*>(qrow) + ch * 16 + hx)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                    const double d0 = (double)x[ch].x - (double)qv.x, d1 = (double)x[ch].y - (double)qv.y;
                    const double d2 = (double)x[ch].z - (double)qv.z, d3 = (double)x[ch].w - (double)qv.w;
                    acc = __fma_rn(d0, d0, acc); acc = __fma_rn(d1, d1, acc);
                    acc = __fma_rn(d2, d2, acc); acc = __fma_rn(d3, d3, acc);
                }
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (v && hx == 0) surv_d[jj] = sqrt(acc);
            }
        }
        q8_cons_sync();
        if (ctid == 0) {
            if (s.ea_count != nullptr) {
                atomicAdd(&s.ea_count[0], (unsigned long long)nrows);
                atomicAdd(&s.ea_count[1], (unsigned long long)ns);
                atomicAdd(&s.ea_count[2], (unsigned long long)((long long)nrows * (M + 16)));
                atomicAdd(&s.ea_count[3], (unsigned long long)((long long)ns * idx.m * 4));
            }
            hi_bits[par] = 0x7f800000u;          // reused by the task after next
            n_surv[par] = 0;
        }
        if (cw == 0) {   // per-task candidates from the survivors only
            double* cd = s.cand_d + t * s.kc;
            long long* ci = s.cand_i + t * s.kc;
            double last_d = -1.0;
            long long last_i = -1;
            for (int sel = 0; sel < s.kc; ++sel) {
                double bd = kInf;
                long long bi = LLONG_MAX;
                for (int i = lane; i < ns; i += 32) {
                    const double dd = surv_d[i];
                    if (!(dd <= bsf)) continue;
                    const long long id = idx.d_row_id[r0 + surv_r[i]];
                    if (pair_less(last_d, last_i, dd, id) && pair_less(dd, id, bd, bi)) { bd = dd; bi = id; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
                    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (pair_less(od, oi, bd, bi)) { bd = od; bi = oi; }
                }
                if (lane == 0) {
                    cd[sel] = bd;
                    ci[sel] = (bi == LLONG_MAX) ? -1 : bi;
                }
                last_d = bd;
                last_i = bi;
            }
        }
    }
}
template <int M32, int MINB = (M32 <= 8 ? 4 : 2)>
static cudaError_t launch_q8_m(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc8,
                               const float4* qm8, cudaStream_t st) {
    using Cfg = Q8Cfg<M32, MINB>;
    if (cudaError_t e = smem_optin(scan_q8_kernel<M32, MINB>, Cfg::SMEM); e != cudaSuccess) return e;
    scan_q8_kernel<M32, MINB><<<sm_count() * MINB, Q8_THREADS, Cfg::SMEM, st>>>(s, idx, q, qc8, qm8);
    return cudaGetLastError();
}

cudaError_t launch_scan_q8(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc8,
                           const float4* qm8, cudaStream_t st) {
    switch ((idx.m + 31) / 32) {                     // the shadow's row stride, in 32-byte units
        case 1: return launch_q8_m<1>(s, idx, q, qc8, qm8, st);
        case 2: return launch_q8_m<2>(s, idx, q, qc8, qm8, st);
        case 3: return launch_q8_m<3>(s, idx, q, qc8, qm8, st);
        case 4: return launch_q8_m<4>(s, idx, q, qc8, qm8, st);
        case 5: return launch_q8_m<5>(s, idx, q, qc8, qm8, st);
        case 6: return launch_q8_m<6>(s, idx, q, qc8, qm8, st);
        case 7: return launch_q8_m<7>(s, idx, q, qc8, qm8, st);
        case 8: return launch_q8_m<8>(s, idx, q, qc8, qm8, st);
        case 9: return launch_q8_m<9>(s, idx, q, qc8, qm8, st);
        case 10: return launch_q8_m<10>(s, idx, q, qc8, qm8, st);
        case 11: return launch_q8_m<11>(s, idx, q, qc8, qm8, st);
        case 12: return launch_q8_m<12>(s, idx, q, qc8, qm8, st);
        case 13: return launch_q8_m<13>(s, idx, q, qc8, qm8, st);
        case 14: return launch_q8_m<14>(s, idx, q, qc8, qm8, st);
        case 15: return launch_q8_m<15>(s, idx, q, qc8, qm8, st);
        case 16: return launch_q8_m<16>(s, idx, q, qc8, qm8, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lf
