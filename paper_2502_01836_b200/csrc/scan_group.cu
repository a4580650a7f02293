// K4 variant (LF_SCAN_GROUP=1): the round's tasks grouped by (leaf, chunk) so one pass
// over a chunk serves every query scanning it.
#include <climits>

#include <cuda_fp16.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "round.cuh"
#include "tc.cuh"

namespace lf {

// ------------------------------------------------------ grouped q8 scan ----
// The same bounded int8 scan, with the round's tasks grouped by (leaf, chunk):
// every query that scans a chunk in this round is served by ONE pass over the
// chunk's codes (on the bench workload a round's (query, leaf) pairs touch 1.2-1.9x
// fewer distinct leaves than pairs: ~1/3 of the int8 bytes disappear;
// tools/share_probe.py).  Warp-specialised so the per-query tail never stalls the
// stream:
//   warp 0      producer: a group's query codes + header into a 2-slot ring, then
//               the chunk's rows (codes + metadata) into a 4-stage ring (128 rows
//               per stage), cp.async.bulk + mbarriers, running ahead across groups;
//   warps 1-16  bound warps: each keeps its 8 rows' codes in registers and
//               evaluates the interval of every query of the group (DP4A +
//               transposing butterfly); lower ends (fp16, rounded down) and the
//               per-query min upper end go to a double-buffered group area;
//   warps 17-20 tail warps: thresholds, survivor compaction, exact fp64 re-read of
//               the survivors and, one warp per query, the task's candidates --
//               while the bound warps already stream the next group.
// Candidates are written per original task, so results and counters are
// identical to scan_q8_kernel (tests: test_grouped_scan_identical).
constexpr int QG = 8;                       // queries per group (larger groups are split)
constexpr int SCAP = 1024;                  // survivors of a group handled in one pass
constexpr int GB_WARPS = 16;                // bound warps
constexpr int GT_WARPS = 4;                 // tail warps
constexpr int G_ROWS = 8 * GB_WARPS;        // rows per stage
constexpr int G_THREADS = 32 * (1 + GB_WARPS + GT_WARPS);

// Per group, precomputed by group_info_kernel so the producer's only dependent
// global load per group is this record (prefetched one group ahead).
struct __align__(16) GroupInfo {
    long long r0;
    int nrows, ng, start, pad;
    int q[QG];
};
constexpr int GT_THREADS = 32 * GT_WARPS;

template <int NCH>
struct Q8GCfg {
    static constexpr int M = NCH * 64;
    static constexpr int P = (M + 255) / 256;
    static constexpr int CODE_BYTES = G_ROWS * M;
    static constexpr int STAGE_BYTES = (CODE_BYTES + G_ROWS * 16 + 127) / 128 * 128;
    static constexpr int STAGES = (147456 / STAGE_BYTES) < 2 ? 2 : ((147456 / STAGE_BYTES) > 8 ? 8 : 147456 / STAGE_BYTES);
    static constexpr int GS_CODES = 0;                               // [QG][P*256]
    static constexpr int GS_META = GS_CODES + QG * P * 256;           // [QG] float4
    static constexpr int GS_HDR = GS_META + QG * 16;                 // GroupInfo
    static constexpr int GS_BYTES = (GS_HDR + (int)sizeof(GroupInfo) + 127) / 128 * 128;
    static constexpr int GS_OFF = STAGES * STAGE_BYTES;
    static constexpr int BAR_OFF = GS_OFF + 2 * GS_BYTES;            // full[S] empty[S] gfull[2] gempty[2] bdone[2] tdone[2]
    static constexpr int LO_OFF = BAR_OFF + (2 * STAGES + 8) * 8;    // [2][QG][CH] half
    static constexpr int SR_OFF = LO_OFF + 2 * QG * CH * 2;
    static constexpr int SD_OFF = SR_OFF + SCAP * 4;
    static constexpr int TH_OFF = SD_OFF + SCAP * 8;                 // [QG] float thresholds
    static constexpr int HB_OFF = TH_OFF + QG * 4;                   // [2][QG] min upper end bits
    static constexpr int MISC_OFF = HB_OFF + 2 * QG * 4;
    static constexpr int SMEM = MISC_OFF + 16;
};

__device__ __forceinline__ void q8_tail_sync() { asm volatile("bar.sync 2, %0;" ::"n"(GT_THREADS) : "memory"); }

// exact fp64 direct-form distances of a group's survivors (series.py:142-146),
// half a warp per survivor, over the tail warps; entries are (g << 16 | row)
template <int NCH>
__device__ __forceinline__ void q8g_exact(const lf_index& idx, const float* __restrict__ queries, const int* gq,
                                          int64_t r0, const int* surv_r, double* surv_d, int ns, int tw, int lane) {
    const int mr = idx.m;                      // fp32 row stride (codes are padded to NCH * 64)
    const int hl = lane & 15;
    const float* X0 = idx.d_X + r0 * mr;
    const int hslot = tw * 2 + (lane >> 4);
    for (int b0 = 0; b0 < ns; b0 += 2 * GT_WARPS) {
        const int jj = b0 + hslot;
        const bool v = jj < ns;
        const int ent = v ? surv_r[jj] : 0;
        const int r = ent & 0xffff;
        const float* qrow = queries + (int64_t)gq[ent >> 16] * mr;
        float4 x[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
            x[ch] = (v && ch * 64 + hl * 4 < mr)
                        ? __ldg(reinterpret_cast<const float4*>(X0 + (int64_t)r * mr) + ch * 16 + hl)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        double acc = 0.0;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const float4 qv = ch * 64 + hl * 4 < mr ? __ldg(reinterpret_cast<const float4*>(qrow) + ch * 16 + hl)
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            const double d0 = (double)x[ch].x - (double)qv.x, d1 = (double)x[ch].y - (double)qv.y;
            const double d2 = (double)x[ch].z - (double)qv.z, d3 = (double)x[ch].w - (double)qv.w;
            acc = __fma_rn(d0, d0, acc); acc = __fma_rn(d1, d1, acc);
            acc = __fma_rn(d2, d2, acc); acc = __fma_rn(d3, d3, acc);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (v && hl == 0) surv_d[jj] = sqrt(acc);
    }
}

// one warp: the kc best (d, id) among the survivors of query g, written as the
// candidates of g's task (tree.py:207 keeps d <= bsf)
__device__ __forceinline__ void q8g_pick(const RoundState& s, const lf_index& idx, const int* __restrict__ sorted,
                                         int gstart, int64_t r0, const int* surv_r, const double* surv_d, int ns,
                                         int g, double bsf, int lane) {
    const int t = sorted[gstart + g];
    double* cd = s.cand_d + (int64_t)t * s.kc;
    long long* ci = s.cand_i + (int64_t)t * s.kc;
    double last_d = -1.0;
    long long last_i = -1;
    for (int sel = 0; sel < s.kc; ++sel) {
        double bd = kInf;
        long long bi = LLONG_MAX;
        for (int i = lane; i < ns; i += 32) {
            const int ent = surv_r[i];
            if ((ent >> 16) != g) continue;
            const double dd = surv_d[i];
            if (!(dd <= bsf)) continue;
            const long long id = idx.d_row_id[r0 + (ent & 0xffff)];
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

template <int NCH>
__global__ void __launch_bounds__(G_THREADS, 1) scan_q8g_kernel(RoundState s, lf_index idx,
                                                                const float* __restrict__ queries,
                                                                const int8_t* __restrict__ qcodes,
                                                                const float4* __restrict__ qmeta,
                                                                const int* __restrict__ sorted,
                                                                const GroupInfo* __restrict__ ginfo,
                                                                const int* __restrict__ n_groups_p) {
    using Cfg = Q8GCfg<NCH>;
    constexpr int M = Cfg::M, P = Cfg::P, S = Cfg::STAGES;
    extern __shared__ __align__(128) unsigned char g8_smem[];
    unsigned char* stages = g8_smem;
    unsigned char* gslots = g8_smem + Cfg::GS_OFF;
    uint64_t* full = reinterpret_cast<uint64_t*>(g8_smem + Cfg::BAR_OFF);
    uint64_t* empty = full + S;
    uint64_t* gfull = empty + S;
    uint64_t* gempty = gfull + 2;
    uint64_t* bdone = gempty + 2;
    uint64_t* tdone = bdone + 2;
    __half* lo_all = reinterpret_cast<__half*>(g8_smem + Cfg::LO_OFF);       // [2][QG][CH]
    int* surv_r = reinterpret_cast<int*>(g8_smem + Cfg::SR_OFF);
    double* surv_d = reinterpret_cast<double*>(g8_smem + Cfg::SD_OFF);
    float* thr_s = reinterpret_cast<float*>(g8_smem + Cfg::TH_OFF);
    unsigned int* hb_all = reinterpret_cast<unsigned int*>(g8_smem + Cfg::HB_OFF);   // [2][QG]
    int* n_surv = reinterpret_cast<int*>(g8_smem + Cfg::MISC_OFF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            q8_bar_init(&full[i], 1);
            q8_bar_init(&empty[i], GB_WARPS);
        }
        for (int i = 0; i < 2; ++i) {
            q8_bar_init(&gfull[i], 1);
            q8_bar_init(&gempty[i], GB_WARPS + GT_WARPS);
            q8_bar_init(&bdone[i], GB_WARPS);
            q8_bar_init(&tdone[i], GT_WARPS);
        }
        for (int g = 0; g < 2 * QG; ++g) hb_all[g] = 0x7f800000u;
        *n_surv = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int n_groups = *n_groups_p;

    if (warp == 0) {   // ---------------------------------------------- producer
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            int slot = 0;
            uint32_t ph = 0;
            int gc = 0;
            GroupInfo gn;
            if (blockIdx.x < n_groups) gn = ginfo[blockIdx.x];
            for (int gi = blockIdx.x; gi < n_groups; gi += gridDim.x, ++gc) {
                const GroupInfo gi_ = gn;
                if (gi + (int)gridDim.x < n_groups) gn = ginfo[gi + gridDim.x];      // prefetch
                const int64_t r0 = gi_.r0;
                const int nrows = gi_.nrows;
                const int gs = gc & 1;
                q8_wait(&gempty[gs], (uint32_t)((gc >> 1) & 1) ^ 1u);
                unsigned char* gsl = gslots + gs * Cfg::GS_BYTES;
                *reinterpret_cast<GroupInfo*>(gsl + Cfg::GS_HDR) = gi_;
                q8_expect_tx(&gfull[gs], (uint32_t)(gi_.ng * (P * 256 + 16)));
                for (int g = 0; g < gi_.ng; ++g) {
                    q8_bulk(gsl + Cfg::GS_CODES + g * P * 256, qcodes + (int64_t)gi_.q[g] * (P * 256), P * 256,
                            &gfull[gs], pol);
                    q8_bulk(gsl + Cfg::GS_META + g * 16, qmeta + gi_.q[g], 16, &gfull[gs], pol);
                }
                for (int j = 0; j < nrows; j += G_ROWS) {
                    const int rows = min(G_ROWS, nrows - j);
                    q8_wait(&empty[slot], ph ^ 1);
                    unsigned char* dst = stages + slot * Cfg::STAGE_BYTES;
                    q8_expect_tx(&full[slot], (uint32_t)(rows * (M + 16)));
                    q8_bulk(dst, idx.d_X8 + (r0 + j) * M, (uint32_t)(rows * M), &full[slot], pol);
                    q8_bulk(dst + Cfg::CODE_BYTES, idx.d_qmeta + (r0 + j) * 4, (uint32_t)(rows * 16), &full[slot], pol);
                    if (++slot == S) { slot = 0; ph ^= 1; }
                }
            }
        }
        return;
    }

    if (warp <= GB_WARPS) {   // ------------------------------------------ bound warps
        const int bw = warp - 1;
        const int hl = lane & 15;
        const int rbase = bw * 8 + (lane >> 4) * 4;
        const bool b8 = (hl & 8) != 0, b4 = (hl & 4) != 0;
        const int myrow = rbase + (b8 ? 2 : 0) + (b4 ? 1 : 0);
        int slot = 0;
        uint32_t ph = 0;
        int gc = 0;
        for (int gi = blockIdx.x; gi < n_groups; gi += gridDim.x, ++gc) {
            const int gs = gc & 1, gb = gc & 1;
            q8_wait(&tdone[gb], (uint32_t)((gc >> 1) & 1) ^ 1u);    // the tail of group gc-2 released its area
            q8_wait(&gfull[gs], (uint32_t)((gc >> 1) & 1));
            const unsigned char* gsl = gslots + gs * Cfg::GS_BYTES;
            const GroupInfo* hdr = reinterpret_cast<const GroupInfo*>(gsl + Cfg::GS_HDR);
            const int nrows = hdr->nrows, ng = hdr->ng;
            __half* lo_s = lo_all + gb * QG * CH;
            float hmin[QG];
#pragma unroll
            for (int g = 0; g < QG; ++g) hmin[g] = __int_as_float(0x7f800000);
            for (int j = 0; j < nrows; j += G_ROWS) {
                q8_wait(&full[slot], ph);
                const int rows = min(G_ROWS, nrows - j);
                const unsigned char* stg = stages + slot * Cfg::STAGE_BYTES;
                int4 w[4][P];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int r = rbase + u;
#pragma unroll
                    for (int p = 0; p < P; ++p)
                        w[u][p] = (r < rows && p * 256 + hl * 16 < M)
                                      ? *reinterpret_cast<const int4*>(stg + r * M + p * 256 + hl * 16)
                                      : make_int4(0, 0, 0, 0);
                }
                const float4 mr = myrow < rows
                                      ? *reinterpret_cast<const float4*>(stg + Cfg::CODE_BYTES + myrow * 16)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                const float sx2xx = mr.x * mr.x * mr.y;
#pragma unroll
                for (int g = 0; g < QG; ++g) {
                    if (g < ng) {
                        int d[4] = {0, 0, 0, 0};
#pragma unroll
                        for (int p = 0; p < P; ++p) {
                            const int4 qv = (p * 256 + hl * 16 < M)
                                                ? *reinterpret_cast<const int4*>(gsl + Cfg::GS_CODES + g * P * 256 +
                                                                                 p * 256 + hl * 16)
                                                : make_int4(0, 0, 0, 0);
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                d[u] = __dp4a(w[u][p].x, qv.x, d[u]);
                                d[u] = __dp4a(w[u][p].y, qv.y, d[u]);
                                d[u] = __dp4a(w[u][p].z, qv.z, d[u]);
                                d[u] = __dp4a(w[u][p].w, qv.w, d[u]);
                            }
                        }
                        const int s0 = b8 ? d[0] : d[2], s1 = b8 ? d[1] : d[3];
                        const int k0 = b8 ? d[2] : d[0], k1 = b8 ? d[3] : d[1];
                        const int e0 = k0 + __shfl_xor_sync(0xffffffffu, s0, 8);
                        const int e1 = k1 + __shfl_xor_sync(0xffffffffu, s1, 8);
                        int v = (b4 ? e1 : e0) + __shfl_xor_sync(0xffffffffu, b4 ? e0 : e1, 4);
                        v += __shfl_xor_sync(0xffffffffu, v, 2);
                        v += __shfl_xor_sync(0xffffffffu, v, 1);
                        if (myrow < rows) {
                            const float4 qm = *reinterpret_cast<const float4*>(gsl + Cfg::GS_META + g * 16);
                            const float sq = qm.x, sq2qq = sq * sq * qm.y;
                            const float e = mr.z + qm.z;
                            const float d2 = sx2xx + sq2qq - 2.f * (mr.x * sq) * (float)v;
                            const float tol = 1e-5f * (sx2xx + sq2qq);
                            const float lo = (sqrtf(fmaxf(d2 - tol, 0.f)) - e) * (1.f - 1e-6f);
                            const float hi = (sqrtf(fmaxf(d2 + tol, 0.f)) + e) * (1.f + 1e-6f);
                            hmin[g] = fminf(hmin[g], hi);
                            if ((hl & 3) == 0) lo_s[g * CH + j + myrow] = __float2half_rd(lo);   // stays a lower bound
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) q8_arrive(&empty[slot]);
                if (++slot == S) { slot = 0; ph ^= 1; }
            }
            if (s.k == 1) {
#pragma unroll
                for (int g = 0; g < QG; ++g) {
                    if (g < ng) {
                        float h = hmin[g];
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) h = fminf(h, __shfl_xor_sync(0xffffffffu, h, o));
                        if (lane == 0) atomicMin(&hb_all[gb * QG + g], __float_as_uint(h));
                    }
                }
            }
            __syncwarp();
            if (lane == 0) {
                q8_arrive(&bdone[gb]);            // release: lower ends + upper-end minima of group gc
                q8_arrive(&gempty[gs]);
            }
        }
        return;
    }

    // ------------------------------------------------------------------ tail warps
    const int tw = warp - 1 - GB_WARPS;
    const int ttid = threadIdx.x - 32 * (1 + GB_WARPS);
    int gc = 0;
    for (int gi = blockIdx.x; gi < n_groups; gi += gridDim.x, ++gc) {
        const int gs = gc & 1, gb = gc & 1;
        q8_wait(&gfull[gs], (uint32_t)((gc >> 1) & 1));
        const unsigned char* gsl = gslots + gs * Cfg::GS_BYTES;
        const GroupInfo* hdr = reinterpret_cast<const GroupInfo*>(gsl + Cfg::GS_HDR);
        const int64_t r0 = hdr->r0;
        const int nrows = hdr->nrows, ng = hdr->ng, gstart = hdr->start;
        const int* gq = hdr->q;
        // the group's best-so-far, fetched while the bound warps stream it
        double bsf_mine = lane < ng ? round_bsf(s, gq[lane]) : kInf;
        q8_wait(&bdone[gb], (uint32_t)((gc >> 1) & 1));
        const __half* lo_s = lo_all + gb * QG * CH;
        unsigned int* hb = hb_all + gb * QG;
        if (ttid < ng) {
            double thr = bsf_mine;
            if (s.k == 1) thr = fmin(thr, (double)__uint_as_float(hb[ttid]));
            thr_s[ttid] = thr < kInf ? __double2float_ru(thr) : __int_as_float(0x7f800000);
        }
        q8_tail_sync();
        for (int e = ttid; e < ng * nrows; e += GT_THREADS) {
            const int g = e / nrows, r = e - g * nrows;
            if (__half2float(lo_s[g * CH + r]) <= thr_s[g]) {
                const int at = atomicAdd(n_surv, 1);
                if (at < SCAP) surv_r[at] = (g << 16) | r;
            }
        }
        q8_tail_sync();
        const int ns_all = *n_surv;
        if (ns_all > SCAP) {
            // rare (k > 1 before k rows were found): recount and finish per query
            for (int g = 0; g < ng; ++g) {
                q8_tail_sync();
                if (ttid == 0) *n_surv = 0;
                q8_tail_sync();
                for (int r = ttid; r < nrows; r += GT_THREADS)
                    if (__half2float(lo_s[g * CH + r]) <= thr_s[g]) surv_r[atomicAdd(n_surv, 1)] = (g << 16) | r;
                q8_tail_sync();
                const int ns = *n_surv;
                q8g_exact<NCH>(idx, queries, gq, r0, surv_r, surv_d, ns, tw, lane);
                q8_tail_sync();
                const double bsf_g = __shfl_sync(0xffffffffu, bsf_mine, g);
                if (tw == 0) q8g_pick(s, idx, sorted, gstart, r0, surv_r, surv_d, ns, g, bsf_g, lane);
                if (ttid == 0 && s.ea_count != nullptr) {
                    atomicAdd(&s.ea_count[0], (unsigned long long)nrows);
                    atomicAdd(&s.ea_count[1], (unsigned long long)ns);
                    atomicAdd(&s.ea_count[2], (unsigned long long)(0));
                    atomicAdd(&s.ea_count[3], (unsigned long long)((long long)ns * idx.m * 4));
                }
            }
        } else {
            q8g_exact<NCH>(idx, queries, gq, r0, surv_r, surv_d, ns_all, tw, lane);
            q8_tail_sync();
            for (int g = tw; g < ng; g += GT_WARPS) {
                const double bsf_g = __shfl_sync(0xffffffffu, bsf_mine, g);
                q8g_pick(s, idx, sorted, gstart, r0, surv_r, surv_d, ns_all, g, bsf_g, lane);
            }
            if (ttid == 0 && s.ea_count != nullptr) {
                atomicAdd(&s.ea_count[0], (unsigned long long)nrows * ng);
                atomicAdd(&s.ea_count[1], (unsigned long long)ns_all);
                atomicAdd(&s.ea_count[2], (unsigned long long)((long long)nrows * (NCH * 64 + 16)));
                atomicAdd(&s.ea_count[3], (unsigned long long)((long long)ns_all * idx.m * 4));
            }
        }
        q8_tail_sync();                                    // survivors consumed
        if (ttid == 0) *n_surv = 0;
        if (ttid < QG) hb[ttid] = 0x7f800000u;
        q8_tail_sync();
        __syncwarp();
        if (lane == 0) {
            q8_arrive(&tdone[gb]);                         // group area free for group gc+2
            q8_arrive(&gempty[gs]);
        }
    }
}

// ---- grouping of a round's tasks by (leaf, chunk) (counting sort, stable keys)
__global__ void chunk_base_kernel(const int64_t* __restrict__ leaf_ptr, int n_leaves, int* __restrict__ base) {
    // single CTA: base[l] = sum over leaves < l of ceil(rows / CH)
    __shared__ int part[1024];
    const int per = (n_leaves + blockDim.x - 1) / blockDim.x;
    const int l0 = threadIdx.x * per, l1 = min(n_leaves, l0 + per);
    int sum = 0;
    for (int l = l0; l < l1; ++l) sum += (int)((leaf_ptr[l + 1] - leaf_ptr[l] + CH - 1) / CH);
    part[threadIdx.x] = sum;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
        const int a = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0;
        __syncthreads();
        part[threadIdx.x] += a;
        __syncthreads();
    }
    int run = part[threadIdx.x] - sum;
    for (int l = l0; l < l1; ++l) {
        base[l] = run;
        run += (int)((leaf_ptr[l + 1] - leaf_ptr[l] + CH - 1) / CH);
    }
    if (threadIdx.x == blockDim.x - 1) base[n_leaves] = part[threadIdx.x];
}

__global__ void group_hist_kernel(RoundState s, const int* __restrict__ cbase, int* __restrict__ hist) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.chunk_off[s.Q]) return;
    const int4 tk = s.tasks[t];
    atomicAdd(&hist[cbase[tk.y] + tk.z], 1);
}

// key offsets (cursor) and the group list (<= QG tasks per group): per-block sums,
// a scan of the block sums, then per-block scans (CUB) -- all keys in parallel
constexpr int GL_THREADS = 512;
__global__ void group_blocksum_kernel(const int* __restrict__ hist, int K, int2* __restrict__ bsum) {
    using BR = cub::BlockReduce<int2, GL_THREADS>;
    __shared__ typename BR::TempStorage tmp;
    const int k = blockIdx.x * GL_THREADS + threadIdx.x;
    const int h = k < K ? hist[k] : 0;
    const int2 v = make_int2(h, (h + QG - 1) / QG);
    const int2 tot = BR(tmp).Reduce(v, [](int2 a, int2 b) { return make_int2(a.x + b.x, a.y + b.y); });
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) group_blockscan_kernel(int2* __restrict__ bsum, int nb,
                                                              int* __restrict__ n_groups) {
    __shared__ int2 carry;
    using BS = cub::BlockScan<int2, 1024>;
    __shared__ typename BS::TempStorage tmp;
    if (threadIdx.x == 0) carry = make_int2(0, 0);
    __syncthreads();
    for (int base = 0; base < nb; base += 1024) {
        const int i = base + threadIdx.x;
        const int2 v = i < nb ? bsum[i] : make_int2(0, 0);
        int2 ex, agg;
        BS(tmp).ExclusiveScan(v, ex, make_int2(0, 0), [](int2 a, int2 b) { return make_int2(a.x + b.x, a.y + b.y); },
                              agg);
        if (i < nb) bsum[i] = make_int2(carry.x + ex.x, carry.y + ex.y);
        __syncthreads();
        if (threadIdx.x == 0) carry = make_int2(carry.x + agg.x, carry.y + agg.y);
        __syncthreads();
    }
    if (threadIdx.x == 0) *n_groups = carry.y;
}

__global__ void group_write_kernel(const int* __restrict__ hist, int K, const int2* __restrict__ boff,
                                   int* __restrict__ cur, int2* __restrict__ groups) {
    using BS = cub::BlockScan<int2, GL_THREADS>;
    __shared__ typename BS::TempStorage tmp;
    const int k = blockIdx.x * GL_THREADS + threadIdx.x;
    const int h = k < K ? hist[k] : 0;
    int2 ex;
    BS(tmp).ExclusiveScan(make_int2(h, (h + QG - 1) / QG), ex, make_int2(0, 0),
                          [](int2 a, int2 b) { return make_int2(a.x + b.x, a.y + b.y); });
    if (k >= K) return;
    const int2 o = boff[blockIdx.x];
    const int t0 = o.x + ex.x;
    int g = o.y + ex.y;
    cur[k] = t0;
    for (int i = 0; i < h; i += QG) groups[g++] = make_int2(t0 + i, min(QG, h - i));
}

__global__ void group_scatter_kernel(RoundState s, const int* __restrict__ cbase, int* __restrict__ cur,
                                     int* __restrict__ sorted) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.chunk_off[s.Q]) return;
    const int4 tk = s.tasks[t];
    sorted[atomicAdd(&cur[cbase[tk.y] + tk.z], 1)] = (int)t;
}

__global__ void group_info_kernel(RoundState s, lf_index idx, const int* __restrict__ sorted,
                                  const int2* __restrict__ groups, const int* __restrict__ n_groups,
                                  GroupInfo* __restrict__ info) {
    const int gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= *n_groups) return;
    const int2 gr = groups[gi];
    const int4 tk0 = s.tasks[sorted[gr.x]];
    GroupInfo o;
    o.r0 = idx.d_leaf_ptr[tk0.y] + (int64_t)tk0.z * CH;
    o.nrows = (int)min((long long)CH, (long long)(idx.d_leaf_ptr[tk0.y + 1] - o.r0));
    o.ng = gr.y;
    o.start = gr.x;
    o.pad = 0;
#pragma unroll
    for (int g = 0; g < QG; ++g) o.q[g] = g < gr.y ? s.tasks[sorted[gr.x + g]].x : 0;
    info[gi] = o;
}

size_t group_info_bytes() { return sizeof(GroupInfo); }
int group_blocks(int n_keys) { return (n_keys + GL_THREADS - 1) / GL_THREADS; }

cudaError_t launch_chunk_base(const lf_index& idx, int* cbase, cudaStream_t st) {
    chunk_base_kernel<<<1, 1024, 0, st>>>(idx.d_leaf_ptr, idx.n_leaves, cbase);
    return cudaGetLastError();
}

template <int N>
static cudaError_t launch_q8g_nch(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc8,
                                  const float4* qm8, const GroupScratch& g, cudaStream_t st) {
    if (cudaError_t e = smem_optin(scan_q8g_kernel<N>, Q8GCfg<N>::SMEM); e != cudaSuccess) return e;
    scan_q8g_kernel<N><<<sm_count(), G_THREADS, Q8GCfg<N>::SMEM, st>>>(
        s, idx, q, qc8, qm8, g.sorted, static_cast<const GroupInfo*>(g.info), g.count);
    return cudaGetLastError();
}

cudaError_t launch_grouped_scan(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc8,
                                const float4* qm8, const GroupScratch& g, int64_t max_tasks, cudaStream_t st) {
    const unsigned tgrid = (unsigned)((max_tasks + 255) / 256);
    cudaError_t e = cudaMemsetAsync(g.hist, 0, sizeof(int) * (g.n_keys > 0 ? g.n_keys : 1), st);
    if (e != cudaSuccess) return e;
    group_hist_kernel<<<tgrid, 256, 0, st>>>(s, g.cbase, g.hist);
    const int nb = group_blocks(g.n_keys);
    group_blocksum_kernel<<<nb, GL_THREADS, 0, st>>>(g.hist, g.n_keys, g.bsum);
    group_blockscan_kernel<<<1, 1024, 0, st>>>(g.bsum, nb, g.count);
    group_write_kernel<<<nb, GL_THREADS, 0, st>>>(g.hist, g.n_keys, g.bsum, g.cur, g.list);
    group_scatter_kernel<<<tgrid, 256, 0, st>>>(s, g.cbase, g.cur, g.sorted);
    group_info_kernel<<<tgrid, 256, 0, st>>>(s, idx, g.sorted, g.list, g.count, static_cast<GroupInfo*>(g.info));
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    switch ((idx.m + 63) / 64) {
        case 1: return launch_q8g_nch<1>(s, idx, q, qc8, qm8, g, st);
        case 2: return launch_q8g_nch<2>(s, idx, q, qc8, qm8, g, st);
        case 3: return launch_q8g_nch<3>(s, idx, q, qc8, qm8, g, st);
        case 4: return launch_q8g_nch<4>(s, idx, q, qc8, qm8, g, st);
        case 5: return launch_q8g_nch<5>(s, idx, q, qc8, qm8, g, st);
        case 6: return launch_q8g_nch<6>(s, idx, q, qc8, qm8, g, st);
        case 7: return launch_q8g_nch<7>(s, idx, q, qc8, qm8, g, st);
        case 8: return launch_q8g_nch<8>(s, idx, q, qc8, qm8, g, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lf
