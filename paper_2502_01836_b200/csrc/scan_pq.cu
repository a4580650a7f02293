// K4 variant (LF_SCAN_VARIANT=pq): the projected two-stage scan.
#include <climits>

#include "common.cuh"
#include "round.cuh"
#include "tc.cuh"

namespace lf {

// ----------------------------------------------------------- projected scan ----
// Two-stage bounded scan over a PROJECTED int8 shadow (lf_index.d_Xp): per row the
// int8 codes of y = P (x - mu) for an orthonormal basis P of pca_k directions (the
// collection's leading principal directions) plus {scale, sum code^2, code error e,
// residual norm r = ||(x - mu) - P^T y||}.  Because P has orthonormal rows,
//     ||x - q||^2 = ||y - y_q||^2 + ||r_vec - r_vec_q||^2,
// the int8 codes give ||y - y_q|| within e + e_q (triangle inequality, fp32
// rounding covered by tol) and | r - r_q | <= ||r_vec - r_vec_q|| <= r + r_q, so
//     lo = sqrt(A_lo^2 + (r - r_q)^2),  hi = sqrt(A_hi^2 + (r + r_q)^2).
// A row costs pca_k + 16 bytes instead of m + 16 (random walks keep ~98% of their
// energy in 32 directions); rows whose lo reaches min(bsf, min hi) are re-read
// whole and summed EXACTLY in fp64, so results equal the full scan.
// Same TMA bulk-copy pipeline as scan_q8_kernel: 1 producer warp, 8 consumer warps.
constexpr int PQ_ROWS = 256;                  // rows per stage

template <int KP>
struct PQCfg {
    static constexpr int L = KP / 16;         // lanes per row (16 codes each)
    static constexpr int RPW = 32 / L;        // rows per warp instruction
    static constexpr int CODE_BYTES = PQ_ROWS * KP;
    static constexpr int STAGE_BYTES = (CODE_BYTES + PQ_ROWS * 16 + 127) / 128 * 128;
    static constexpr int STAGES = KP == 32 ? 6 : 4;
    static constexpr int QC_OFF = CODE_BYTES + PQ_ROWS * 16;         // query codes (first stage of a task)
    static constexpr int QM_OFF = QC_OFF + KP;                       // query meta float4
    static constexpr int HDR_OFF = QM_OFF + 16;                       // r0 i64, q, nrows
    static constexpr int STAGE_TOTAL = (HDR_OFF + 16 + 127) / 128 * 128;
    static constexpr int BAR_OFF = STAGES * STAGE_TOTAL;
    static constexpr int LO_OFF = BAR_OFF + 2 * STAGES * 8;
    static constexpr int SR_OFF = LO_OFF + CH * 4;
    static constexpr int SD_OFF = SR_OFF + CH * 4;
    static constexpr int MISC_OFF = SD_OFF + CH * 8;
    static constexpr int SMEM = MISC_OFF + 16;
};

// Query projection: y_q = P (q - mu) in fp64, residual norm, int8 codes (same
// scheme as the rows).  Warp per query.  codes [Q][KP], meta [Q] = {s, qq, e, r}.
__global__ void project_queries_kernel(const float* __restrict__ queries, int64_t Q, int m, int k, int KP,
                                       const double* __restrict__ P, const double* __restrict__ mu,
                                       int8_t* __restrict__ qc, float4* __restrict__ qm) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= Q) return;
    const float* x = queries + q * m;
    double y[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) y[j] = 0.0;
    for (int j = 0; j < k; ++j) {
        double acc = 0.0;
        for (int i = lane; i < m; i += 32) acc = __fma_rn(P[(int64_t)j * m + i], (double)x[i] - mu[i], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        y[j < 64 ? j : 63] = acc;
    }
    double rr = 0.0;
    for (int i = lane; i < m; i += 32) {
        double v = (double)x[i] - mu[i];
        for (int j = 0; j < k; ++j) v -= P[(int64_t)j * m + i] * y[j];
        rr = __fma_rn(v, v, rr);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rr += __shfl_xor_sync(0xffffffffu, rr, o);
    float mx = 0.f;
    for (int j = 0; j < k; ++j) mx = fmaxf(mx, (float)fabs(y[j]));
    const float s = mx > 0.f ? mx / 127.f : 1.f;
    double err = 0.0;
    int qq = 0;
    for (int j = 0; j < KP; ++j) {
        int c = 0;
        if (j < k) {
            c = (int)fmin(fmax(rint(y[j] / (double)s), -127.0), 127.0);
            const double e = (double)s * c - y[j];
            err = __fma_rn(e, e, err);
        }
        if (lane == 0) qc[q * KP + j] = (int8_t)c;
        qq += c * c;
    }
    if (lane == 0)
        qm[q] = make_float4(s, (float)qq, __double2float_ru(sqrt(err) * (1.0 + 1e-9) + 1e-30), (float)sqrt(rr));
}


template <int KP>
__global__ void __launch_bounds__(Q8_THREADS, 2) scan_pq_kernel(RoundState s, lf_index idx,
                                                                const float* __restrict__ queries,
                                                                const int8_t* __restrict__ qcodes,
                                                                const float4* __restrict__ qmeta,
                                                                int* __restrict__ surv_cnt,
                                                                unsigned short* __restrict__ surv_rows) {
    using Cfg = PQCfg<KP>;
    constexpr int S = Cfg::STAGES, L = Cfg::L, RPW = Cfg::RPW;
    extern __shared__ __align__(128) unsigned char pq_smem[];
    unsigned char* stages = pq_smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(pq_smem + Cfg::BAR_OFF);
    uint64_t* empty = full + S;
    float* lo_s = reinterpret_cast<float*>(pq_smem + Cfg::LO_OFF);
    int* surv_r = reinterpret_cast<int*>(pq_smem + Cfg::SR_OFF);
    double* surv_d = reinterpret_cast<double*>(pq_smem + Cfg::SD_OFF);
    unsigned int* hi_bits = reinterpret_cast<unsigned int*>(pq_smem + Cfg::MISC_OFF);   // [2]
    int* n_surv = reinterpret_cast<int*>(hi_bits + 2);                                 // [2]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            q8_bar_init(&full[i], 1);
            q8_bar_init(&empty[i], Q8_CONS_WARPS);
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
            constexpr int PF = 4;                        // task records in flight ahead
            int4 ring[PF];
#pragma unroll
            for (int i = 0; i < PF; ++i) {
                const long long ti = blockIdx.x + (long long)i * gridDim.x;
                ring[i] = ti < total ? s.task_rows[ti] : make_int4(0, 0, 0, 0);
            }
            int head = 0;
            for (long long t = blockIdx.x; t < total; t += gridDim.x) {
                int4 tr = ring[0];
#pragma unroll
                for (int i = 0; i < PF; ++i)
                    if (i == head) tr = ring[i];
                const long long tf = t + (long long)PF * gridDim.x;
                const int4 nx = tf < total ? s.task_rows[tf] : make_int4(0, 0, 0, 0);
#pragma unroll
                for (int i = 0; i < PF; ++i)
                    if (i == head) ring[i] = nx;
                head = head + 1 == PF ? 0 : head + 1;
                const int4 tk = make_int4(tr.w, 0, 0, 0);
                const int64_t r0 = (int64_t)(unsigned)tr.x | ((int64_t)tr.y << 32);
                const int nrows = tr.z;
                for (int j = 0; j < nrows; j += PQ_ROWS) {
                    const int rows = min(PQ_ROWS, nrows - j);
                    q8_wait(&empty[slot], ph ^ 1);
                    unsigned char* dst = stages + slot * Cfg::STAGE_TOTAL;
                    uint32_t bytes = (uint32_t)(rows * (KP + 16));
                    if (j == 0) {
                        *reinterpret_cast<long long*>(dst + Cfg::HDR_OFF) = r0;
                        *reinterpret_cast<int2*>(dst + Cfg::HDR_OFF + 8) = make_int2(tk.x, nrows);
                        bytes += KP + 16;
                    }
                    q8_expect_tx(&full[slot], bytes);
                    q8_bulk(dst, idx.d_Xp + (r0 + j) * KP, (uint32_t)(rows * KP), &full[slot], pol);
                    q8_bulk(dst + Cfg::CODE_BYTES, idx.d_pmeta + (r0 + j) * 4, (uint32_t)(rows * 16), &full[slot], pol);
                    if (j == 0) {
                        q8_bulk(dst + Cfg::QC_OFF, qcodes + (int64_t)tk.x * KP, KP, &full[slot], pol);
                        q8_bulk(dst + Cfg::QM_OFF, qmeta + tk.x, 16, &full[slot], pol);
                    }
                    if (++slot == S) { slot = 0; ph ^= 1; }
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------ consumers
    const int cw = warp - 1;
    const int ctid = threadIdx.x - 32;
    const int sub = lane % L;                       // this lane's 16-code slice of its row
    const int rw = lane / L;                        // row within the warp instruction
    const int m = idx.m;
    int slot = 0;
    uint32_t ph = 0;
    int par = 0;
    for (long long t = blockIdx.x; t < total; t += gridDim.x, par ^= 1) {
        q8_wait(&full[slot], ph);
        const unsigned char* st0 = stages + slot * Cfg::STAGE_TOTAL;
        const int64_t r0 = *reinterpret_cast<const long long*>(st0 + Cfg::HDR_OFF);
        const int2 hq = *reinterpret_cast<const int2*>(st0 + Cfg::HDR_OFF + 8);
        const int64_t q = hq.x;
        const int nrows = hq.y;
        const double bsf = round_bsf(s, q);
        const int4 qw = *reinterpret_cast<const int4*>(st0 + Cfg::QC_OFF + sub * 16);
        const float4 qmv = *reinterpret_cast<const float4*>(st0 + Cfg::QM_OFF);
        const float sq = qmv.x, eq = qmv.z, rq = qmv.w;
        const float sq2qq = sq * sq * qmv.y;
        float hmin = __int_as_float(0x7f800000);
        for (int j = 0; j < nrows; j += PQ_ROWS) {
            if (j > 0) q8_wait(&full[slot], ph);
            const int rows = min(PQ_ROWS, nrows - j);
            const unsigned char* stg = stages + slot * Cfg::STAGE_TOTAL;
#pragma unroll
            for (int it = 0; it < PQ_ROWS / (Q8_CONS_WARPS * RPW); ++it) {
                const int r = (it * Q8_CONS_WARPS + cw) * RPW + rw;
                const bool v = r < rows;
                const int4 w = v ? *reinterpret_cast<const int4*>(stg + r * KP + sub * 16) : make_int4(0, 0, 0, 0);
                int dot = __dp4a(w.x, qw.x, 0);
                dot = __dp4a(w.y, qw.y, dot);
                dot = __dp4a(w.z, qw.z, dot);
                dot = __dp4a(w.w, qw.w, dot);
#pragma unroll
                for (int o = L / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
                if (v) {
                    const float4 mr = *reinterpret_cast<const float4*>(stg + Cfg::CODE_BYTES + r * 16);
                    const float sx2xx = mr.x * mr.x * mr.y;
                    const float e = mr.z + eq;
                    const float a2 = sx2xx + sq2qq - 2.f * (mr.x * sq) * (float)dot;
                    const float tol = 1e-5f * (sx2xx + sq2qq);
                    const float alo = fmaxf(sqrtf(fmaxf(a2 - tol, 0.f)) - e, 0.f);
                    const float ahi = sqrtf(fmaxf(a2 + tol, 0.f)) + e;
                    const float blo = fmaxf(fabsf(mr.w - rq) - 1e-6f * (mr.w + rq), 0.f);
                    const float bhi = (mr.w + rq) * (1.f + 1e-6f);
                    const float lo = sqrtf(fmaf(alo, alo, blo * blo)) * (1.f - 1e-5f);
                    const float hi = sqrtf(fmaf(ahi, ahi, bhi * bhi)) * (1.f + 1e-5f);
                    hmin = fminf(hmin, hi);
                    if (sub == 0) lo_s[j + r] = lo;
                }
            }
            __syncwarp();
            if (lane == 0) q8_arrive(&empty[slot]);
            if (++slot == S) { slot = 0; ph ^= 1; }
        }
        if (s.k == 1) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) hmin = fminf(hmin, __shfl_xor_sync(0xffffffffu, hmin, o));
            if (lane == 0) atomicMin(&hi_bits[par], __float_as_uint(hmin));
        }
        q8_cons_sync();
        {
            double thr = bsf;
            if (s.k == 1) thr = fmin(thr, (double)__uint_as_float(hi_bits[par]));
            const float thr_f = thr < kInf ? __double2float_ru(thr) : __int_as_float(0x7f800000);
            for (int r = ctid; r < nrows; r += Q8_CONS)
                if (lo_s[r] <= thr_f) surv_r[atomicAdd(&n_surv[par], 1)] = r;
        }
        q8_cons_sync();
        const int ns = n_surv[par];
        if (ns <= PQ_SQ) {
            // the common case: hand the few survivors to survivor_exact_kernel (no global
            // loads on this CTA's critical path); the candidates are written there
            for (int i = ctid; i < ns; i += Q8_CONS) surv_rows[t * PQ_SQ + i] = (unsigned short)surv_r[i];
            if (ctid == 0) {
                surv_cnt[t] = ns;
                if (s.ea_count != nullptr) {
                    atomicAdd(&s.ea_count[0], (unsigned long long)nrows);
                    atomicAdd(&s.ea_count[1], (unsigned long long)ns);
                    atomicAdd(&s.ea_count[2], (unsigned long long)((long long)nrows * (KP + 16)));
                    atomicAdd(&s.ea_count[3], (unsigned long long)((long long)ns * m * 4));
                }
            }
            q8_cons_sync();
            if (ctid == 0) {
                hi_bits[par] = 0x7f800000u;
                n_surv[par] = 0;
            }
            continue;
        }
        if (ctid == 0) surv_cnt[t] = -1;                 // candidates written below
        {   // exact fp64 direct-form distances of the survivors (series.py:142-146), half a warp each
            const float* X0 = idx.d_X + r0 * m;
            const float* qrow = queries + q * m;
            const int hl = lane & 15;
            const int hslot = cw * 2 + (lane >> 4);
            for (int b0 = 0; b0 < ns; b0 += 16) {
                const int jj = b0 + hslot;
                const bool v = jj < ns;
                const int r = v ? surv_r[jj] : 0;
                double acc = 0.0;
                for (int c = hl * 4; c < m; c += 64) {
                    float4 xv = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (v) xv = __ldg(reinterpret_cast<const float4*>(X0 + (int64_t)r * m + c));
                    const float4 qv = __ldg(reinterpret_cast<const float4*>(qrow + c));
                    const double d0 = (double)xv.x - (double)qv.x, d1 = (double)xv.y - (double)qv.y;
                    const double d2 = (double)xv.z - (double)qv.z, d3 = (double)xv.w - (double)qv.w;
                    acc = __fma_rn(d0, d0, acc); acc = __fma_rn(d1, d1, acc);
                    acc = __fma_rn(d2, d2, acc); acc = __fma_rn(d3, d3, acc);
                }
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (v && hl == 0) surv_d[jj] = sqrt(acc);
            }
        }
        q8_cons_sync();
        if (ctid == 0) {
            if (s.ea_count != nullptr) {
                atomicAdd(&s.ea_count[0], (unsigned long long)nrows);
                atomicAdd(&s.ea_count[1], (unsigned long long)ns);
                atomicAdd(&s.ea_count[2], (unsigned long long)((long long)nrows * (KP + 16)));
                atomicAdd(&s.ea_count[3], (unsigned long long)((long long)ns * m * 4));
            }
            hi_bits[par] = 0x7f800000u;
            n_surv[par] = 0;
        }
        if (cw == 0) {
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

// Exact fp64 re-read of the projected scan's survivors (series.py:142-146), one warp
// per task, 4 rows in flight per iteration; then the task's kc best (d, id) with
// d <= bsf (tree.py:207) as its candidates.  Tasks the scan finished itself have
// surv_cnt = -1.
__global__ void survivor_exact_kernel(RoundState s, lf_index idx, const float* __restrict__ queries,
                                      const int* __restrict__ surv_cnt,
                                      const unsigned short* __restrict__ surv_rows) {
    const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= s.chunk_off[s.Q]) return;
    const int ns = surv_cnt[t];
    if (ns < 0) return;
    const int4 tk = s.tasks[t];
    const int64_t q = tk.x;
    const int64_t r0 = idx.d_leaf_ptr[tk.y] + (int64_t)tk.z * CH;
    const int m = idx.m;
    const double bsf = round_bsf(s, q);
    const float* qrow = queries + q * m;
    const unsigned short* rl = surv_rows + t * PQ_SQ;
    double dist_mine = kInf;                          // lane i keeps row i's distance (ns <= 64: two slots)
    double dist_mine2 = kInf;
    constexpr int RF = 8;                             // rows in flight per warp
    for (int b = 0; b < ns; b += RF) {
        double acc[RF];
#pragma unroll
        for (int u = 0; u < RF; ++u) acc[u] = 0.0;
        for (int c = lane * 4; c < m; c += 128) {
            const float4 qv = __ldg(reinterpret_cast<const float4*>(qrow + c));
            float4 xv[RF];
#pragma unroll
            for (int u = 0; u < RF; ++u)
                xv[u] = b + u < ns ? __ldg(reinterpret_cast<const float4*>(idx.d_X + (r0 + rl[b + u]) * m + c))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < RF; ++u) {
                const double d0 = (double)xv[u].x - (double)qv.x, d1 = (double)xv[u].y - (double)qv.y;
                const double d2 = (double)xv[u].z - (double)qv.z, d3 = (double)xv[u].w - (double)qv.w;
                acc[u] = __fma_rn(d0, d0, acc[u]); acc[u] = __fma_rn(d1, d1, acc[u]);
                acc[u] = __fma_rn(d2, d2, acc[u]); acc[u] = __fma_rn(d3, d3, acc[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < RF; ++u) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
            const int i = b + u;
            if (i < ns) {
                if (lane == (i & 31)) {
                    if (i < 32) dist_mine = sqrt(acc[u]);
                    else dist_mine2 = sqrt(acc[u]);
                }
            }
        }
    }
    long long id_mine = lane < ns ? idx.d_row_id[r0 + rl[lane]] : LLONG_MAX;
    long long id_mine2 = lane + 32 < ns ? idx.d_row_id[r0 + rl[lane + 32]] : LLONG_MAX;
    if (!(dist_mine <= bsf)) { dist_mine = kInf; id_mine = LLONG_MAX; }
    if (!(dist_mine2 <= bsf)) { dist_mine2 = kInf; id_mine2 = LLONG_MAX; }
    double* cd = s.cand_d + t * s.kc;
    long long* ci = s.cand_i + t * s.kc;
    double last_d = -1.0;
    long long last_i = -1;
    for (int sel = 0; sel < s.kc; ++sel) {
        double bd = kInf;
        long long bi = LLONG_MAX;
        if (pair_less(last_d, last_i, dist_mine, id_mine) && pair_less(dist_mine, id_mine, bd, bi)) {
            bd = dist_mine; bi = id_mine;
        }
        if (pair_less(last_d, last_i, dist_mine2, id_mine2) && pair_less(dist_mine2, id_mine2, bd, bi)) {
            bd = dist_mine2; bi = id_mine2;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, o);
            const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (pair_less(od, oi, bd, bi)) { bd = od; bi = oi; }
        }
        if (lane == 0) {
            cd[sel] = bd;
            ci[sel] = (bi == LLONG_MAX || bd == kInf) ? -1 : bi;
        }
        last_d = bd;
        last_i = bi;
    }
}

cudaError_t launch_project_queries(const float* q, int64_t Q, const lf_index& idx, int8_t* qc, float4* qm,
                                   cudaStream_t st) {
    project_queries_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(q, Q, idx.m, idx.pca_k, idx.pca_k,
                                                                             idx.d_P, idx.d_mu, qc, qm);
    return cudaGetLastError();
}

template <int KP>
static cudaError_t launch_pq_kp(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc,
                                const float4* qm, int* surv_cnt, unsigned short* surv_rows, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(scan_pq_kernel<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             PQCfg<KP>::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    scan_pq_kernel<KP><<<sm_count() * 2, Q8_THREADS, PQCfg<KP>::SMEM, st>>>(s, idx, q, qc, qm, surv_cnt, surv_rows);
    return cudaGetLastError();
}

cudaError_t launch_scan_pq(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc,
                           const float4* qm, int* surv_cnt, unsigned short* surv_rows, int64_t max_tasks,
                           cudaStream_t st) {
    cudaError_t e = idx.pca_k == 32 ? launch_pq_kp<32>(s, idx, q, qc, qm, surv_cnt, surv_rows, st)
                                    : launch_pq_kp<64>(s, idx, q, qc, qm, surv_cnt, surv_rows, st);
    if (e != cudaSuccess) return e;
    survivor_exact_kernel<<<(unsigned)((max_tasks * 32 + 255) / 256), 256, 0, st>>>(s, idx, q, surv_cnt, surv_rows);
    return cudaGetLastError();
}

}  // namespace lf
