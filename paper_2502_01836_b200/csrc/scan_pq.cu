// K4b-d (default from round 1 on; LF_SCAN_VARIANT=q8 disables): the projected scan
// cascade.
#include <algorithm>
#include <climits>

#include "common.cuh"
#include "round.cuh"
#include "tc.cuh"

namespace lf {

// ----------------------------------------------------------- projected scan ----
// Bounded scan over a PROJECTED int8 shadow (lf_index.d_Xp): per row the int8 codes
// of y = P (x - mu) for an orthonormal basis P of pca_k directions (the collection's
// leading principal directions) plus {scale, ||scale * code||^2, code error e,
// residual norm r = ||(x - mu) - P^T y||}.  Because P has orthonormal rows,
//     ||x - q||^2 = ||y - y_q||^2 + ||r_vec - r_vec_q||^2,
// the int8 codes give ||y - y_q|| within e + e_q (triangle inequality, fp32
// rounding covered by tol) and | r - r_q | <= ||r_vec - r_vec_q|| <= r + r_q, so
//     lo = sqrt(A_lo^2 + (r - r_q)^2),  hi = sqrt(A_hi^2 + (r + r_q)^2).
// A row costs pca_k + 16 bytes instead of m + 16 (random walks keep ~97% of their
// energy in 32 directions).  Rows whose lo reaches min(bsf, min hi) -- 2% on the
// bench workload -- get the full-length int8 interval (pq_q8_bound_kernel), and the
// ones that survive that are re-read whole and summed EXACTLY in fp64
// (pq_tail_kernel), so results equal the full scan.
// One WARP per task (no CTA barriers): at pca_k + 16 = 48 bytes a 512-row chunk is
// only 24 KB, so the per-task barriers of the CTA-pipelined q8 scan would dominate.
// Each warp streams its own tasks through a private ring of PQW_NS shared-memory
// slots of PQW_STG rows, filled by cp.async.bulk (lane 0 issues, an mbarrier per
// slot completes on the bytes): the refill of a slot is issued as soon as the warp
// has read it, so PQW_NS - 1 pieces per warp are always in flight.  Lane i owns rows
// i, i + 32, ... of a piece; lo / hi live in registers, min hi is a warp reduction
// and survivors are compacted by ballot.
// ring geometry (tools/pq_sweep.sh: 64 rows x 4 slots x 16 warps, 64 x 3 x 20 and a
// next-task prefetch all within 1%; 32-row slots are slower)
#ifndef LF_PQW_STG
#define LF_PQW_STG 64
#endif
#ifndef LF_PQW_NS
#define LF_PQW_NS 4
#endif
#ifndef LF_PQW_WARPS32
#define LF_PQW_WARPS32 16
#endif
constexpr int PQW_STG = LF_PQW_STG;           // rows per ring slot
constexpr int PQW_NS = LF_PQW_NS;             // ring slots per warp
constexpr int PQ_PIECES = CH / PQW_STG;       // slots per task (max)
constexpr int PQ_SLOTS = CH / 32;             // rows per lane per task

template <int KP>
struct PQW {
    static constexpr int WARPS = KP == 32 ? LF_PQW_WARPS32 : 8;
    static constexpr int CODE = PQW_STG * KP;
    // codes + 8 B fp16 metadata per row; the metadata copy starts at an even row (16-byte
    // aligned source), so a slot holds up to two more metadata rows
    static constexpr int STAGE = CODE + (PQW_STG + 2) * 8;
    static constexpr int RING = WARPS * PQW_NS * STAGE;
    static constexpr int BAR_OFF = RING;
    static constexpr int SMEM = BAR_OFF + WARPS * PQW_NS * 8;
};

__device__ __forceinline__ float sqrt_approx(float x) {   // MUFU.SQRT, denormals kept
    float r;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Query projection: y_q = P (q - mu) in fp64, residual norm, int8 codes (same
// scheme as the rows).  One CTA of 8 warps per query, each warp k / 8 directions;
// the residual norm is sqrt(max(||q - mu||^2 - ||y_q||^2, 0)) (P has orthonormal
// rows; fp64 keeps the cancellation far below the bound's 1e-6 slack).
// codes [Q][KP], meta [Q] = {s, qq, e, r}.
constexpr int PJ_WARPS = 8;
__global__ void __launch_bounds__(PJ_WARPS * 32) project_queries_kernel(const float* __restrict__ queries, int64_t Q,
                                                                       int m, int k, int KP,
                                                                       const double* __restrict__ P,
                                                                       const double* __restrict__ mu,
                                                                       int8_t* __restrict__ qc,
                                                                       float4* __restrict__ qm) {
    __shared__ double y[64];
    __shared__ double part[PJ_WARPS];
    const int64_t q = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float* x = queries + q * m;
    for (int j = warp; j < k; j += PJ_WARPS) {
        double acc = 0.0;
        for (int i = lane; i < m; i += 32) acc = __fma_rn(P[(int64_t)j * m + i], (double)x[i] - mu[i], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) y[j] = acc;
    }
    double xx = 0.0;
    for (int i = threadIdx.x; i < m; i += PJ_WARPS * 32) {
        const double v = (double)x[i] - mu[i];
        xx = __fma_rn(v, v, xx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xx += __shfl_xor_sync(0xffffffffu, xx, o);
    if (lane == 0) part[warp] = xx;
    __syncthreads();
    if (warp != 0) return;
    xx = lane < PJ_WARPS ? part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xx += __shfl_xor_sync(0xffffffffu, xx, o);
    double yy = 0.0;
    float mx = 0.f;
    for (int j = lane; j < k; j += 32) {
        yy = __fma_rn(y[j], y[j], yy);
        mx = fmaxf(mx, (float)fabs(y[j]));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        yy += __shfl_xor_sync(0xffffffffu, yy, o);
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const float s = mx > 0.f ? mx / 127.f : 1.f;
    double err = 0.0;
    int qq = 0;
    for (int j = lane; j < KP; j += 32) {
        int c = 0;
        if (j < k) {
            c = (int)fmin(fmax(rint(y[j] / (double)s), -127.0), 127.0);
            const double e = (double)s * c - y[j];
            err = __fma_rn(e, e, err);
        }
        qc[q * KP + j] = (int8_t)c;
        qq += c * c;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        qq += __shfl_xor_sync(0xffffffffu, qq, o);
        err += __shfl_xor_sync(0xffffffffu, err, o);
    }
    if (lane == 0)
        qm[q] = make_float4(s, (float)qq, __double2float_ru(sqrt(err) * (1.0 + 1e-9) + 1e-30),
                            (float)sqrt(fmax(xx - yy, 0.0)));
}


// Exact fp64 distances of rows rl[0 .. ns) of a task, one warp, RF rows in flight;
// dist[i] (shared memory) = sqrt(sum (x - q)^2) in the direct form of series.py:142-146.
__device__ __forceinline__ void pq_exact_rows(const float* __restrict__ X0, const float* __restrict__ qrow, int m,
                                              const unsigned short* rl, int ns, double* dist, int lane) {
    constexpr int RF = 8;
    for (int b = 0; b < ns; b += RF) {
        double acc[RF];
#pragma unroll
        for (int u = 0; u < RF; ++u) acc[u] = 0.0;
        for (int c0 = lane * 4; c0 < m; c0 += 256) {      // two 512-byte column blocks in flight
            float4 qv[2], xv[2][RF];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = c0 + h * 128;
                qv[h] = c < m ? __ldg(reinterpret_cast<const float4*>(qrow + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int u = 0; u < RF; ++u)
                    xv[h][u] = (b + u < ns && c < m)
                                   ? __ldg(reinterpret_cast<const float4*>(X0 + (int64_t)rl[b + u] * m + c))
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < RF; ++u) {
                    const double d0 = (double)xv[h][u].x - (double)qv[h].x, d1 = (double)xv[h][u].y - (double)qv[h].y;
                    const double d2 = (double)xv[h][u].z - (double)qv[h].z, d3 = (double)xv[h][u].w - (double)qv[h].w;
                    acc[u] = __fma_rn(d0, d0, acc[u]); acc[u] = __fma_rn(d1, d1, acc[u]);
                    acc[u] = __fma_rn(d2, d2, acc[u]); acc[u] = __fma_rn(d3, d3, acc[u]);
                }
        }
#pragma unroll
        for (int u = 0; u < RF; ++u) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
            if (lane == 0 && b + u < ns) dist[b + u] = sqrt(acc[u]);
        }
    }
    __syncwarp();
}

// The task's kc best (d, id) with d <= bsf (tree.py:207) over ns survivors, as its
// candidates; dist(i) / id(i) give survivor i's exact distance and row id (NaN: pruned).
template <class DistF, class IdF>
__device__ __forceinline__ void pq_select(const RoundState& s, long long t, int lane, int ns, double bsf, DistF dist,
                                          IdF id_of) {
    double* cd = s.cand_d + t * s.kc;
    long long* ci = s.cand_i + t * s.kc;
    double last_d = -1.0;
    long long last_i = -1;
    for (int sel = 0; sel < s.kc; ++sel) {
        double bd = kInf;
        long long bi = LLONG_MAX;
        for (int i = lane; i < ns; i += 32) {
            const double dd = dist(i);
            if (!(dd <= bsf)) continue;
            const long long id = id_of(i);
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

// SEED (round 0, k = 1; ov.qbest): with no best-so-far the projected upper bound
// (residual term r + r_q) is loose and most rows would survive.  Each task tracks the
// row with the smallest projected ESTIMATE ||y - y_q||^2 + r^2 + r_q^2 (residuals taken
// as orthogonal), reads that one row exactly (fp64, the warp's 1 KiB load) and prunes
// with its distance -- a real row's exact distance bounds the task's (and query's)
// nearest from above, so the cascade stays exact.  Tasks of one query share the best
// seed through ov.qbest.
template <int KP, bool SEED>
__global__ void __launch_bounds__(PQW<KP>::WARPS * 32) scan_pq_kernel(RoundState s, lf_index idx,
                                                                      const float* __restrict__ queries,
                                                                      const int8_t* __restrict__ qcodes,
                                                                      const float4* __restrict__ qmeta,
                                                                      int* __restrict__ surv_cnt,
                                                                      PQOverflow ov) {
    using C = PQW<KP>;
    constexpr int V = KP / 16;                        // int4 code vectors per row
    constexpr int RPL = PQW_STG / 32;                 // rows per lane per slot
    extern __shared__ __align__(128) unsigned char pqw_smem[];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long gw = (long long)blockIdx.x * C::WARPS + wib;
    const long long nw = (long long)gridDim.x * C::WARPS;
    const long long total = s.chunk_off[s.Q];
    const int m = idx.m;
    unsigned char* ring = pqw_smem + wib * PQW_NS * C::STAGE;
    uint64_t* bars = reinterpret_cast<uint64_t*>(pqw_smem + C::BAR_OFF) + wib * PQW_NS;
    unsigned short* rows_w = ov.wrows + gw * CH;      // fallback scratch (entry list full), global
    double* dist_w = ov.wdist + gw * CH;
    if (lane == 0) {
        for (int i = 0; i < PQW_NS; ++i) q8_bar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));

    // issue cursor: (task, piece) NS pieces ahead of the consumer (lane 0 issues)
    long long it = gw;
    int ip = 0, inrows = 0;
    int64_t ir0 = 0;
    if (it < total) {
        const int4 tr = s.task_rows[it];
        ir0 = (int64_t)(unsigned)tr.x | ((int64_t)tr.y << 32);
        inrows = tr.z;
    }
    auto issue = [&](int slot) {
        if (it >= total) return;
        const int rows = min(PQW_STG, inrows - ip * PQW_STG);
        if (lane == 0) {
            unsigned char* dst = ring + slot * C::STAGE;
            const int64_t rr = ir0 + (int64_t)ip * PQW_STG;
            const int64_t ra = rr & ~1ll;                              // even: 16-byte aligned source
            const uint32_t mb = (uint32_t)(((rr + rows - ra) * 8 + 15) & ~15);   // padded array
            q8_expect_tx(&bars[slot], (uint32_t)(rows > 0 ? rows * KP + mb : 0));
            if (rows > 0) {
                q8_bulk(dst, idx.d_Xp + rr * KP, (uint32_t)(rows * KP), &bars[slot], pol);
                q8_bulk(dst + C::CODE, idx.d_pmeta + ra * 4, mb, &bars[slot], pol);
            }
        }
        if (++ip * PQW_STG >= inrows) {
            ip = 0;
            it += nw;
            if (it < total) {
                const int4 tr = s.task_rows[it];
                ir0 = (int64_t)(unsigned)tr.x | ((int64_t)tr.y << 32);
                inrows = tr.z;
            }
        }
    };
#pragma unroll
    for (int i = 0; i < PQW_NS; ++i) issue(i);
    int cslot = 0;
    uint32_t cph = 0;
    unsigned long long c_rows = 0, c_surv = 0, c_fall = 0;
    for (long long t = gw; t < total; t += nw) {
        const int4 tr = s.task_rows[t];
        const double bsf = round_bsf(s, tr.w);
        int4 qw[V];
#pragma unroll
        for (int v = 0; v < V; ++v) qw[v] = __ldg(reinterpret_cast<const int4*>(qcodes + (int64_t)tr.w * KP) + v);
        const float4 qmv = __ldg(qmeta + tr.w);
        const int64_t r0 = (int64_t)(unsigned)tr.x | ((int64_t)tr.y << 32);
        const int nrows = tr.z;
        const int64_t q = tr.w;
        const int mo = (int)(r0 & 1);                 // metadata rows start one early when r0 is odd
        const int pieces = nrows > 0 ? (nrows + PQW_STG - 1) / PQW_STG : 1;
        const float sq = qmv.x, eq = qmv.z, rq = qmv.w;
        const float sq2qq = sq * sq * qmv.y;
        const float sq2 = 2.f * sq;
        // lo2 / hi2: squares of the interval ends before their (1 -+ 1e-5) factors; the
        // comparisons below run in the squared domain (one sqrt per task, not two per row)
        float lo2[PQ_SLOTS];
        float hmin2 = __int_as_float(0x7f800000);
        float best_est = __int_as_float(0x7f800000);      // SEED: smallest estimate, its row
        int best_ri = 0;
        const float rq2 = rq * rq;
#pragma unroll
        for (int p = 0; p < PQ_PIECES; ++p) {
            if (p < pieces) {
                q8_wait(&bars[cslot], cph);
                const unsigned char* stg = ring + cslot * C::STAGE;
#pragma unroll
                for (int u = 0; u < RPL; ++u) {
                    const int ri = u * 32 + lane;
                    const bool v = p * PQW_STG + ri < nrows;
                    // rows past the chunk's end read stale slot bytes; their result is masked
                    int4 w[V];
#pragma unroll
                    for (int c = 0; c < V; ++c) w[c] = *reinterpret_cast<const int4*>(stg + ri * KP + c * 16);
                    const uint2 mp = *reinterpret_cast<const uint2*>(stg + C::CODE + (ri + mo) * 8);
                    const float msc = __half2float(__ushort_as_half((unsigned short)(mp.x & 0xffffu)));
                    const float mer = __half2float(__ushort_as_half((unsigned short)(mp.x >> 16)));
                    const float mrn = __half2float(__ushort_as_half((unsigned short)(mp.y & 0xffffu)));
                    int dot = 0, cc = 0;
#pragma unroll
                    for (int c = 0; c < V; ++c) {
                        dot = __dp4a(w[c].x, qw[c].x, dot);
                        dot = __dp4a(w[c].y, qw[c].y, dot);
                        dot = __dp4a(w[c].z, qw[c].z, dot);
                        dot = __dp4a(w[c].w, qw[c].w, dot);
                        cc = __dp4a(w[c].x, w[c].x, cc);
                        cc = __dp4a(w[c].y, w[c].y, cc);
                        cc = __dp4a(w[c].z, w[c].z, cc);
                        cc = __dp4a(w[c].w, w[c].w, cc);
                    }
                    const float nn = fmaf(msc * msc, (float)cc, sq2qq);  // ||x_c||^2 + ||q_c||^2
                    const float a2 = fmaf(-(msc * sq2), (float)dot, nn);
                    const float tol = 1e-5f * nn;
                    const float e = mer + eq;
                    // sqrt.approx (rel err < 2^-22): the tol slack (>= 2.5e-6 sqrt(a2)) and the
                    // final 1 -+ 1e-5 factors cover it, so both ends stay rigorous
                    const float alo = fmaxf(sqrt_approx(fmaxf(a2 - tol, 0.f)) - e, 0.f);
                    const float ahi = sqrt_approx(fmaxf(a2 + tol, 0.f)) + e;
                    // the residual norm is fp16 (nearest): |r - r16| <= 2^-11 r16, widened to 2^-10
                    const float rs = mrn + rq;
                    const float blo = fmaxf(fabsf(mrn - rq) - fmaf(1e-6f, rs, 9.765625e-4f * mrn), 0.f);
                    const float bhi = fmaf(9.765625e-4f, mrn, rs) * (1.f + 1e-6f);
                    lo2[p * RPL + u] = v ? fmaf(alo, alo, blo * blo) : __int_as_float(0x7f800000);
                    hmin2 = fminf(hmin2, v ? fmaf(ahi, ahi, bhi * bhi) : __int_as_float(0x7f800000));
                    if (SEED) {
                        const float est = fmaf(mrn, mrn, a2 + rq2);
                        if (v && est < best_est) { best_est = est; best_ri = p * PQW_STG + ri; }
                    }
                }
                __syncwarp();                            // every lane has read the slot
                issue(cslot);                            // refill it NS pieces ahead
                if (++cslot == PQW_NS) { cslot = 0; cph ^= 1; }
            } else {
#pragma unroll
                for (int u = 0; u < RPL; ++u) lo2[p * RPL + u] = __int_as_float(0x7f800000);
            }
        }
        double thr = bsf;
        if (s.k == 1) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) hmin2 = fminf(hmin2, __shfl_xor_sync(0xffffffffu, hmin2, o));
            thr = fmin(thr, (double)(sqrtf(hmin2) * (1.f + 1e-5f)));
        }
        if (SEED && nrows > 0) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float oe = __shfl_xor_sync(0xffffffffu, best_est, o);
                const int oi = __shfl_xor_sync(0xffffffffu, best_ri, o);
                if (oe < best_est || (oe == best_est && oi < best_ri)) { best_est = oe; best_ri = oi; }
            }
            // the seed row, exactly (series.py:142-146 direct form in fp64)
            const float* xr = idx.d_X + (r0 + best_ri) * m;
            const float* qr = queries + q * m;
            double acc = 0.0;
            for (int c = lane * 4; c < m; c += 128) {
                const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + c));
                const float4 qv = __ldg(reinterpret_cast<const float4*>(qr + c));
                const double d0 = (double)xv.x - qv.x, d1 = (double)xv.y - qv.y;
                const double d2 = (double)xv.z - qv.z, d3 = (double)xv.w - qv.w;
                acc = __fma_rn(d0, d0, acc); acc = __fma_rn(d1, d1, acc);
                acc = __fma_rn(d2, d2, acc); acc = __fma_rn(d3, d3, acc);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const float dseed = __double2float_ru(sqrt(acc));
            unsigned prev = 0;
            if (lane == 0) prev = atomicMin(ov.qbest + q, __float_as_uint(dseed));
            prev = __shfl_sync(0xffffffffu, prev, 0);
            thr = fmin(thr, (double)fminf(dseed, __uint_as_float(prev)));
        }
        const float thr_f = thr < kInf ? __double2float_ru(thr) : __int_as_float(0x7f800000);
        // keep iff sqrt(lo2) (1 - 1e-5) <= thr  <=>  lo2 <= (thr / (1 - 1e-5))^2, rounded up
        const float thr2 = thr < kInf ? __double2float_ru((thr / (1.0 - 1e-5)) * (thr / (1.0 - 1e-5)))
                                      : __int_as_float(0x7f800000);
        unsigned bal[PQ_SLOTS];
        int ns = 0;
#pragma unroll
        for (int g = 0; g < PQ_SLOTS; ++g) {
            bal[g] = __ballot_sync(0xffffffffu, lo2[g] <= thr2);
            ns += __popc(bal[g]);
        }
        c_rows += (unsigned long long)nrows;
        c_surv += (unsigned long long)ns;
        if (ns == 0) {
            if (lane == 0) {
                surv_cnt[t] = 0;
                if (s.cand16 != nullptr) {                       // k = 1 entry tail
                    s.cand16[2 * t] = (unsigned long long)__double_as_longlong(kInf);
                    s.cand16[2 * t + 1] = (unsigned long long)LLONG_MAX;
                }
            }
            continue;
        }
        // survivors -> (task, query, row) entries for the int8 stage (pq_q8_bound_kernel)
        int base = 0;
        if (lane == 0) base = atomicAdd(ov.n, ns);
        base = __shfl_sync(0xffffffffu, base, 0);
        const bool fits = (long long)base + ns <= (long long)ov.cap;
        const unsigned below = (1u << lane) - 1u;
        int off = 0;
#pragma unroll
        for (int g = 0; g < PQ_SLOTS; ++g) {
            if ((bal[g] >> lane) & 1u) {
                const int pos = off + __popc(bal[g] & below);
                if (fits) {
                    const int64_t ar = r0 + g * 32 + lane;      // absolute row
                    ov.ent[base + pos] = make_int4((int)t, (int)q, (int)(unsigned)ar, (int)(ar >> 32));
                } else {
                    if ((long long)base + pos < (long long)ov.cap) ov.ent[base + pos] = make_int4(-1, 0, 0, 0);
                    rows_w[pos] = (unsigned short)(g * 32 + lane);
                }
            }
            off += __popc(bal[g]);
        }
        if (fits) {
            if (lane == 0) {
                surv_cnt[t] = ns;
                ov.base[t] = base;
                ov.thr[t] = __float_as_uint(thr_f);
                if (s.cand16 != nullptr) {                       // k = 1 entry tail
                    s.cand16[2 * t] = (unsigned long long)__double_as_longlong(kInf);
                    s.cand16[2 * t + 1] = (unsigned long long)LLONG_MAX;
                }
            }
            continue;
        }
        __syncwarp();
        if (lane == 0) surv_cnt[t] = -1;                 // entry list full: re-read and select here
        pq_exact_rows(idx.d_X + r0 * m, queries + q * m, m, rows_w, ns, dist_w, lane);
        if (ov.qc8 != nullptr) c_fall += (unsigned long long)ns;
        pq_select(s, t, lane, ns, bsf, [&](int i) { return dist_w[i]; },
                  [&](int i) { return idx.d_row_id[r0 + rows_w[i]]; });
        if (s.cand16 != nullptr && lane == 0) {          // (lane 0 wrote the selection)
            const long long ci = s.cand_i[t];
            s.cand16[2 * t] = (unsigned long long)__double_as_longlong(ci < 0 ? kInf : s.cand_d[t]);
            s.cand16[2 * t + 1] = (unsigned long long)(ci < 0 ? LLONG_MAX : ci);
        }
        __syncwarp();
    }
    if (s.ea_count != nullptr && lane == 0 && c_rows > 0) {
        atomicAdd(&s.ea_count[0], c_rows);
        atomicAdd(&s.ea_count[2], c_rows * (unsigned long long)(KP + 8));
        if (ov.qc8 == nullptr) {                      // else the int8 stage / re-read count theirs
            atomicAdd(&s.ea_count[1], c_surv);
            atomicAdd(&s.ea_count[3], c_surv * (unsigned long long)m * 4ull);
        } else if (c_fall > 0) {
            atomicAdd(&s.ea_count[1], c_fall);
            atomicAdd(&s.ea_count[3], c_fall * (unsigned long long)m * 4ull);
        }
    }
}

// int8 stage of the projected scan's survivor entries, row-parallel: the full-length
// int8 interval of each entry (the bound of scan_q8_kernel; 8 lanes per row, 16 code
// bytes per lane per load, 2 rows per 8-lane group, row metadata loaded up front).
// lo is kept per entry; for k = 1 the task threshold is min'ed with every entry's
// upper bound -- the task's best row survives both stages, so no row whose lower
// bound exceeds it can be the nearest.
#ifndef LF_PQB_MINB
// resident CTAs per SM the register budget targets (bench sweep 2 / 3 / 4 / 6: scan phase
// 1.55 / 1.46 / 1.48 / 1.60 ms per batch)
#define LF_PQB_MINB 3
#endif
template <bool FIX256, int R = 2, int MINB = LF_PQB_MINB>
__global__ void __launch_bounds__(256, MINB) pq_q8_bound_kernel(RoundState s, lf_index idx, PQOverflow ov) {
    // R: entries per 8-lane group in flight (3 and 4 at 2 CTAs / SM: 1.81 / 1.82 vs 1.75 ms per batch)
    const int lane = threadIdx.x & 31, sl = lane & 7, grp = lane >> 3;
    if (blockIdx.x == 0 && threadIdx.x == 0 && ov.xn != nullptr) *ov.xn = 0;   // the exact tail's list
    const long long n = min((long long)*ov.n, (long long)ov.cap);
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const int M8 = FIX256 ? 256 : (idx.m + 31) / 32 * 32;   // the shadow's row stride
    unsigned long long cnt = 0;
    // FIX256 (m <= 256): a lane's 32 query-code bytes stay in registers while its
    // group's entries keep the same query (entries of a task are contiguous), and the
    // next iteration's entries are loaded while this one's rows are in flight
    int64_t cq[R];
    int4 cqv[R][2];
    long long w0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * (4 * R);
    int4 en[R];
#pragma unroll
    for (int u = 0; u < R; ++u) {
        cq[u] = -1;
        cqv[u][0] = cqv[u][1] = make_int4(0, 0, 0, 0);
        const long long i = w0 + u * 4 + grp;
        en[u] = i < n ? ov.ent[i] : make_int4(-1, 0, 0, 0);
    }
    for (; w0 < n; w0 += nw * 4 * R) {
        long long ii[R];
        int4 e[R];
        int64_t row[R];
        int64_t qq[R];
        float4 mr[R], qmv[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            ii[u] = w0 + u * 4 + grp;
            e[u] = en[u];
            row[u] = (int64_t)(unsigned)e[u].z | ((int64_t)e[u].w << 32);
            qq[u] = e[u].y;
        }
        int dot[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
            dot[u] = 0;
            const bool v = e[u].x >= 0 && sl == 0;          // metadata with the first code loads
            mr[u] = v ? __ldcs(reinterpret_cast<const float4*>(idx.d_qmeta) + row[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
            qmv[u] = v ? __ldg(ov.qm8 + qq[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if constexpr (FIX256) {
            int4 w[R][2];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < R; ++u)
                    w[u][h] = e[u].x >= 0 ? __ldcs(reinterpret_cast<const int4*>(idx.d_X8 + row[u] * 256 + sl * 16 + h * 128))
                                          : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < R; ++u)
                if (e[u].x >= 0 && qq[u] != cq[u]) {
                    cq[u] = qq[u];
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        cqv[u][h] = __ldg(reinterpret_cast<const int4*>(ov.qc8 + qq[u] * ov.mp + sl * 16 + h * 128));
                }
#pragma unroll
            for (int u = 0; u < R; ++u) {          // next iteration's entries
                const long long i = w0 + nw * 4 * R + u * 4 + grp;
                en[u] = i < n ? ov.ent[i] : make_int4(-1, 0, 0, 0);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int u = 0; u < R; ++u) {
                    dot[u] = __dp4a(w[u][h].x, cqv[u][h].x, dot[u]);
                    dot[u] = __dp4a(w[u][h].y, cqv[u][h].y, dot[u]);
                    dot[u] = __dp4a(w[u][h].z, cqv[u][h].z, dot[u]);
                    dot[u] = __dp4a(w[u][h].w, cqv[u][h].w, dot[u]);
                }
        } else {
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const long long i = w0 + nw * 4 * R + u * 4 + grp;
                en[u] = i < n ? ov.ent[i] : make_int4(-1, 0, 0, 0);
            }
            // both 128-byte halves of a 256-byte row in flight together (longer rows loop)
            for (int c0 = sl * 16; c0 < M8; c0 += 256) {
                int4 w[R][2], qv[R][2];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const int c = c0 + h * 128;
                        const bool v = e[u].x >= 0 && c < M8;
                        w[u][h] = v ? __ldcs(reinterpret_cast<const int4*>(idx.d_X8 + row[u] * M8 + c))
                                    : make_int4(0, 0, 0, 0);
                        qv[u][h] = v ? __ldg(reinterpret_cast<const int4*>(ov.qc8 + qq[u] * ov.mp + c))
                                     : make_int4(0, 0, 0, 0);
                    }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        dot[u] = __dp4a(w[u][h].x, qv[u][h].x, dot[u]);
                        dot[u] = __dp4a(w[u][h].y, qv[u][h].y, dot[u]);
                        dot[u] = __dp4a(w[u][h].z, qv[u][h].z, dot[u]);
                        dot[u] = __dp4a(w[u][h].w, qv[u][h].w, dot[u]);
                    }
            }
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
            dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], 4);
            dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], 2);
            dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], 1);
            if (e[u].x >= 0 && sl == 0) {
                const float sq = qmv[u].x, eq = qmv[u].z;
                const float sq2qq = sq * sq * qmv[u].y;
                const float sx2xx = mr[u].x * mr[u].x * mr[u].y;
                const float ee = mr[u].z + eq;
                const float d2 = sx2xx + sq2qq - 2.f * (mr[u].x * sq) * (float)dot[u];
                const float tol = 1e-5f * (sx2xx + sq2qq);
                ov.lo8[ii[u]] = (sqrtf(fmaxf(d2 - tol, 0.f)) - ee) * (1.f - 1e-6f);
                ++cnt;
                if (s.k == 1)
                    atomicMin(&ov.thr[e[u].x], __float_as_uint((sqrtf(fmaxf(d2 + tol, 0.f)) + ee) * (1.f + 1e-6f)));
            }
        }
    }
    if (s.ea_count != nullptr) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        if (lane == 0 && cnt > 0) atomicAdd(&s.ea_count[2], cnt * (unsigned long long)(M8 + 16));
    }
}

__device__ __forceinline__ int64_t ent_row(int4 e) { return (int64_t)(unsigned)e.z | ((int64_t)e.w << 32); }

// Tail of the projected scan, one warp per task with survivors (entries
// [base, base + ns) of the entry list, contiguous per task): the rows whose int8
// lower bound (pq_q8_bound_kernel) reaches the task threshold are re-read exactly in
// fp64 (series.py:142-146), RF rows in flight, and the task's kc candidates written.
// Without the int8 shadow (qc8 == nullptr) every entry is re-read.
constexpr int PQT_WARPS = 8;
__global__ void __launch_bounds__(PQT_WARPS * 32) pq_tail_kernel(RoundState s, lf_index idx,
                                                                 const float* __restrict__ queries,
                                                                 const int* __restrict__ surv_cnt, PQOverflow ov) {
    __shared__ unsigned short s_rows[PQT_WARPS][CH];
    __shared__ double s_dist[PQT_WARPS][CH];
    const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long total = s.chunk_off[s.Q];
    const long long nw = (long long)gridDim.x * PQT_WARPS;
    const int m = idx.m;
    unsigned short* rows_w = s_rows[wib];
    double* dist_w = s_dist[wib];
    unsigned long long c_exact = 0;
    for (long long t = (long long)blockIdx.x * PQT_WARPS + wib; t < total; t += nw) {
        const int ns = surv_cnt[t];
        if (ns < 0) continue;                          // the scan warp finished this task
        if (ns == 0) {
            for (int i = lane; i < s.kc; i += 32) {
                s.cand_d[t * s.kc + i] = kInf;
                s.cand_i[t * s.kc + i] = -1;
            }
            continue;
        }
        const int4 tk = s.tasks[t];
        const int64_t q = tk.x;
        const int64_t r0 = idx.d_leaf_ptr[tk.y] + (int64_t)tk.z * CH;
        const double bsf = round_bsf(s, q);
        const int base = ov.base[t];
        const int4* ent = ov.ent + base;
        int nx = 0;                                    // rows for the exact re-read
        if (ov.qc8 != nullptr) {                       // int8 stage done by pq_q8_bound_kernel
            const float thr8 = __uint_as_float(ov.thr[t]);
            for (int b = 0; b < ns; b += 32) {
                const int i = b + lane;
                const bool sv = i < ns && ov.lo8[base + i] <= thr8;
                const unsigned bal = __ballot_sync(0xffffffffu, sv);
                if (sv) rows_w[nx + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)(ent_row(ent[i]) - r0);
                nx += __popc(bal);
            }
        } else {
            for (int i = lane; i < ns; i += 32) rows_w[i] = (unsigned short)(ent_row(ent[i]) - r0);
            nx = ns;
        }
        __syncwarp();
        c_exact += (unsigned long long)nx;
        pq_exact_rows(idx.d_X + r0 * m, queries + q * m, m, rows_w, nx, dist_w, lane);
        pq_select(s, t, lane, nx, bsf, [&](int i) { return dist_w[i]; },
                  [&](int i) { return idx.d_row_id[r0 + rows_w[i]]; });
        __syncwarp();
    }
    if (s.ea_count != nullptr) {                         // c_exact is warp-uniform
        if (lane == 0) {
            if (c_exact) {
                atomicAdd(&s.ea_count[1], c_exact);
                atomicAdd(&s.ea_count[3], c_exact * (unsigned long long)m * 4ull);
            }
        }
    }
}

// k = 1 tail, ENTRY-parallel (no per-task chain of dependent loads):
//   e0: thread per entry -- the entries whose int8 lower bound reaches their task's
//       final threshold (~3% of them) are compacted into a list;
//   e1: 8 lanes per listed entry re-read the row exactly (all loads in flight) and
//       fold (distance, row id) into the task's pair by a 128-bit compare-and-swap
//       loop -- the lexicographic minimum, i.e. the smallest id among equal distances
//       (tree.py:207-214 tie rule), in the same pass.  (A separate tie-break pass
//       after a 64-bit atomicMin of the distance cost one more launch per round.)
__global__ void pq_tail_e0_kernel(PQOverflow ov) {
    const long long n = min((long long)*ov.n, (long long)ov.cap);
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const int t = ov.ent[e].x;
        const bool go = t >= 0 && ov.lo8[e] <= __uint_as_float(ov.thr[t]);
        const unsigned bal = __ballot_sync(__activemask(), go);
        if (bal == 0) continue;
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(bal) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(ov.xn, __popc(bal));
        base = __shfl_sync(__activemask(), base, leader);
        if (go) ov.xlist[base + __popc(bal & ((1u << lane) - 1u))] = (int)e;
    }
}

__global__ void __launch_bounds__(256) pq_tail_e1_kernel(RoundState s, lf_index idx, const float* __restrict__ queries,
                                                        PQOverflow ov) {
    const int lane = threadIdx.x & 31, sl = lane & 7;
    const int n = *ov.xn;
    const long long ng = ((long long)gridDim.x * blockDim.x) >> 3;
    const int m = idx.m;
    const long long bound = ((long long)n + 3) & ~3ll;      // warp-uniform trip count (4 entries per warp)
    for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3; i < bound; i += ng) {
        const bool go = i < n;
        const int e = go ? ov.xlist[i] : 0;
        const int4 en = go ? ov.ent[e] : make_int4(0, 0, 0, 0);
        double acc = 0.0;
        if (go) {
            const float4* xr = reinterpret_cast<const float4*>(idx.d_X + ent_row(en) * m);
            const float4* qr = reinterpret_cast<const float4*>(queries + (int64_t)en.y * m);
            for (int c0 = 0; c0 < m / 4; c0 += 64) {               // 8 float4 per lane in flight
                float4 xv[8], qv[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int c = c0 + sl + 8 * u;
                    const bool v = c < m / 4;
                    xv[u] = v ? __ldcs(xr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                    qv[u] = v ? __ldg(qr + c) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double d0 = (double)xv[u].x - qv[u].x, d1 = (double)xv[u].y - qv[u].y;
                    const double d2 = (double)xv[u].z - qv[u].z, d3 = (double)xv[u].w - qv[u].w;
                    acc = __fma_rn(d0, d0, acc); acc = __fma_rn(d1, d1, acc);
                    acc = __fma_rn(d2, d2, acc); acc = __fma_rn(d3, d3, acc);
                }
            }
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 4);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        if (go && sl == 0) {
            const double d = sqrt(acc);
            {
                // (d, id) lexicographic minimum per task in one 128-bit CAS loop: the id
                // tie-break (tree.py:207-214) without a second pass
                const long long id = idx.d_row_id[ent_row(en)];
                unsigned long long* c = s.cand16 + 2 * (long long)en.x;
                // (starts from the initial value: the CAS returns the current pair atomically)
                unsigned long long cx = (unsigned long long)__double_as_longlong(kInf), cy = (unsigned long long)LLONG_MAX;
                while (pair_less(d, id, __longlong_as_double((long long)cx), (long long)cy)) {
                    unsigned long long ox, oy;
                    asm volatile(
                        "{\n\t.reg .b128 cmp, val, old;\n\t"
                        "mov.b128 cmp, {%2, %3};\n\t"
                        "mov.b128 val, {%4, %5};\n\t"
                        "atom.cas.relaxed.gpu.b128 old, [%6], cmp, val;\n\t"
                        "mov.b128 {%0, %1}, old;\n\t}"
                        : "=l"(ox), "=l"(oy)
                        : "l"(cx), "l"(cy), "l"((unsigned long long)__double_as_longlong(d)), "l"((unsigned long long)id),
                          "l"(c)
                        : "memory");
                    if (ox == cx && oy == cy) break;
                    cx = ox;
                    cy = oy;
                }
            }
        }
    }
    if (s.ea_count != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && n > 0) {
        atomicAdd(&s.ea_count[1], (unsigned long long)n);
        atomicAdd(&s.ea_count[3], (unsigned long long)n * (unsigned long long)m * 4ull);
    }
}


cudaError_t launch_project_queries(const float* q, int64_t Q, const lf_index& idx, int8_t* qc, float4* qm,
                                   cudaStream_t st) {
    project_queries_kernel<<<(unsigned)Q, PJ_WARPS * 32, 0, st>>>(q, Q, idx.m, idx.pca_k, idx.pca_k, idx.d_P,
                                                                  idx.d_mu, qc, qm);
    return cudaGetLastError();
}

template <int KP>
static cudaError_t launch_pq_kp(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc,
                                const float4* qm, int* surv_cnt, const PQOverflow& ov, cudaStream_t st) {
    if (ov.qbest != nullptr) {
        if (cudaError_t e = smem_optin(scan_pq_kernel<KP, true>, PQW<KP>::SMEM); e != cudaSuccess) return e;
        scan_pq_kernel<KP, true><<<sm_count(), PQW<KP>::WARPS * 32, PQW<KP>::SMEM, st>>>(s, idx, q, qc, qm, surv_cnt,
                                                                                          ov);
        return cudaGetLastError();
    }
    if (cudaError_t e = smem_optin(scan_pq_kernel<KP, false>, PQW<KP>::SMEM); e != cudaSuccess) return e;
    scan_pq_kernel<KP, false><<<sm_count(), PQW<KP>::WARPS * 32, PQW<KP>::SMEM, st>>>(s, idx, q, qc, qm, surv_cnt, ov);
    return cudaGetLastError();
}

int pq_scan_warps() { return sm_count() * PQW<32>::WARPS; }   // >= PQW<64>: 16 vs 8 per SM

cudaError_t launch_scan_pq(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc,
                           const float4* qm, int* surv_cnt, const PQOverflow& ov, int64_t max_tasks,
                           cudaStream_t st, cudaEvent_t after_scan) {
    // (ov.n: zeroed by the round's plan kernel; ov.xn: by the int8 stage)
    cudaError_t e = idx.pca_k == 32 ? launch_pq_kp<32>(s, idx, q, qc, qm, surv_cnt, ov, st)
                        : launch_pq_kp<64>(s, idx, q, qc, qm, surv_cnt, ov, st);
    if (e != cudaSuccess) return e;
    if (after_scan != nullptr && (e = cudaEventRecord(after_scan, st)) != cudaSuccess) return e;
    if (ov.qc8 != nullptr) {
        // (R = 3 / 4 at 2 CTAs per SM, 1 at 6 and 2 at 4: 1.54-1.60 vs 1.53 ms per batch; a
        // warp-level min before the per-entry threshold atomics: 1.93 ms; the gathers through
        // a per-warp shared-memory ring of 8-entry pieces -- cp.async.bulk per row and
        // mbarrier: 1.54, 16-byte cp.async with 4 / 6 / 8 pieces in flight: 1.68 / 1.62 /
        // 1.82, vs 1.48 ms for this kernel)
        if ((idx.m + 31) / 32 * 32 == 256)
            pq_q8_bound_kernel<true><<<sm_count() * 8, 256, 0, st>>>(s, idx, ov);
        else
            pq_q8_bound_kernel<false><<<sm_count() * 8, 256, 0, st>>>(s, idx, ov);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (s.cand16 != nullptr) {                       // k = 1: entry-parallel tail
        pq_tail_e0_kernel<<<sm_count() * 8, 256, 0, st>>>(ov);
        pq_tail_e1_kernel<<<sm_count() * 4, 256, 0, st>>>(s, idx, q, ov);
        return cudaGetLastError();
    }
    const long long warps = std::min<long long>(max_tasks, (long long)sm_count() * 64);
    pq_tail_kernel<<<(unsigned)((warps + PQT_WARPS - 1) / PQT_WARPS), PQT_WARPS * 32, 0, st>>>(s, idx, q, surv_cnt, ov);
    return cudaGetLastError();
}

}  // namespace lf
