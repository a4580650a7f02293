// K2-K4: the batched best-first search (tree.py:220-297) as rounds over a
// per-query visit order.
//
//   bounds (K1)  ->  stable (lb, node id) sort per query (K2; the heap of
//   tree.py:256-275 pops in exactly this order)  ->  rounds:
//     plan   : one thread per query walks its order from a cursor, applying the
//              break rule lb > bsf*f (tree.py:261-269) and the filter rule
//              pred - offset > bsf*f (tree.py:277-286) with the round-start
//              bsf, and selects up to R leaves to scan;
//     scan   : leaf chunks of CH rows; each warp computes fp64 direct-form
//              distances (series.py:142-146) from 128-bit loads and a
//              warp-shuffle reduction; per-chunk top-k candidates;
//     merge  : one warp per query folds candidates into the running top-k by
//              (distance, id) (tree.py:192-217) and refreshes bsf.
// With sequential=1 every round scans one leaf per query, which reproduces
// the reference's traversal, counters and trace exactly.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_fp16.h>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "bounds.cuh"
#include "common.cuh"
#include "tc.cuh"

namespace lf {

constexpr int CH = 512;          // rows per scan task (512 KiB at m = 256)
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_WARPS = SCAN_THREADS / 32;

struct RoundState {
    int64_t Q;
    int k, kc;                   // kc = candidates kept per task = min(k, CH)
    int R, Rcap;                 // leaves per query this round, and the buffer stride
    double f;                    // bsf_factor
    const int* order;            // [Q][Nn] visit-order records (bounds.cuh OrderArgs)
    const double* lbs;           // [Q][Nn]
    const int* leafo;            // [Q][Nn] leaf slot | LF_REC_HASF, -1 internal
    const double* adj;           // [Q][Nn] pred - offset of the leaf's filter
    const int* olen;             // [Q] valid (sorted) entries of the order
    int* refill;                 // [Q] set when the walk reached olen < Nn
    int* n_refill;               // queries flagged this round (= n_active + 1)
    int lazy;                    // lazy filter inference: adj valid for positions < pcount[q]
    const int* pcount;           // [Q]
    int* preq;                   // [Q] set when the walk stopped at pcount (more predictions needed)
    int* pwin;                   // [Q] positions the next prediction pass covers (doubles per pass)
    int* n_predict;              // walks that reached pcount with a finite bsf (= n_active + 2)
    int* cursor;                 // [Q]
    int* done;                   // [Q]
    double* top_d;               // [Q][k]   running top-k (round-start state)
    long long* top_i;            // [Q][k]
    int* top_n;                  // [Q]
    double* top_d_out;           // merge writes here; host swaps after each round
    long long* top_i_out;
    int* top_n_out;
    int n_leaves;
    const double* bound;         // [Q] external best-so-far bound (other shards), or NULL
    long long* stats;            // [Q][6]
    int* sel_leaf;               // [Q][Rcap]
    int* sel_trace;              // [Q][Rcap]
    int* sel_pre;                // [Q][Rcap+1] chunk prefix within the query
    int* n_sel;                  // [Q]
    long long* chunk_off;        // [Q+1]
    int4* tasks;                 // [max_tasks] (query, leaf slot, chunk, selection index)
    int4* task_rows;             // [max_tasks] (r0 lo, r0 hi, rows, query) or NULL
    unsigned long long* ea_count;  // [2] rows tested / survivors (profiling only, may be NULL)
    double* cand_d;              // [max_tasks][kc]
    long long* cand_i;
    double* task_min;            // [max_tasks] (trace only)
    int* n_active;
    const float* pred;           // [Q][F]
    const double* pred64;        // [Q][F] (alternative to pred)
    const double* offset;        // [F]
    int F;
    int want_trace;
    lf_trace tr;
};

__device__ inline double query_bsf(const RoundState& s, int64_t q) {
    return s.top_n[q] == s.k ? s.top_d[q * s.k + s.k - 1] : kInf;
}

// The bound a round prunes with: the local k-th best, tightened by the bound
// exchanged with the other leaf shards (min over ranks of their k-th best is
// >= the global k-th best, so pruning with it stays exact).
__device__ inline double round_bsf(const RoundState& s, int64_t q) {
    const double b = query_bsf(s, q);
    return s.bound != nullptr ? fmin(b, s.bound[q]) : b;
}

// ---------------------------------------------------------------- plan ----
// Warp-parallel plan: one warp per query evaluates 32 consecutive visit-order
// entries at a time.  Within a round every decision uses the round-start bsf,
// so the entries are independent; ballots locate the first break (lb > bsf*f)
// and the R-th selected leaf, and prefix counts place selections and trace
// entries in visit order.  Counters, selections and traces are identical to a
// serial walk of the same entries (tree.py:256-297 with the round-start bsf).
__global__ void plan_warp_kernel(RoundState s, lf_index idx) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= s.Q) return;
    const unsigned below = (1u << lane) - 1u;
    const int Nn = idx.n_nodes;
    int* pre = s.sel_pre + q * (s.Rcap + 1);
    int ns = 0, nch = 0;
    if (!s.done[q]) {
        const double bsf = round_bsf(s, q);
        const double thr = bsf * s.f;
        const int* ord = s.order + q * Nn;
        const double* lbs = s.lbs + q * Nn;
        const int* lrec = s.leafo + q * Nn;
        const double* adj = s.adj + q * Nn;
        const int olen = s.olen[q];
        // lazy inference: with a finite bsf the filter rule needs adj, valid below pcount
        const int len = (s.lazy && thr < kInf) ? min(olen, s.pcount[q]) : olen;
        long long* st = s.stats + q * LF_N_STATS;
        int cur = s.cursor[q];
        bool fin = false, quota_hit = false;
        int tl = s.want_trace ? s.tr.d_len[q] : 0;
        const int64_t tbase = q * (int64_t)idx.n_leaves;
        long long c_vis = 0, c_srch = 0, c_lbp = 0, c_fp = 0, c_inf = 0, c_rows = 0;
        // records of the current 32 entries, and the next 32 prefetched while these are
        // decided (a walk that neither breaks nor fills its quota moves on by exactly 32)
        auto load = [&](int at, double& l_, int& r_, double& a_) {
            const int k = at + lane;
            l_ = k < len ? lbs[k] : kInf;
            r_ = k < len ? lrec[k] : -1;
            a_ = k < len ? adj[k] : 0.0;
        };
        double lb_c, ad_c;
        int rec_c;
        load(cur, lb_c, rec_c, ad_c);
        while (!fin && cur < len) {
            double lb_n, ad_n;
            int rec_n;
            load(cur + 32, lb_n, rec_n, ad_n);
            const int i = cur + lane;
            const bool valid = i < len;
            const int node = (valid && s.want_trace) ? ord[i] : -1;
            const double lb = lb_c;
            const int rec = rec_c;
            const int leaf = rec >= 0 ? (rec & LF_REC_LEAF) : -1;
            const bool brk = valid && lb > thr;
            const unsigned bmask = __ballot_sync(0xffffffffu, brk);
            const int first_brk = bmask ? __ffs(bmask) - 1 : 32;
            const bool visit = valid && leaf >= 0 && lane < first_brk;
            const int fs = (visit && (rec & LF_REC_HASF)) ? 0 : -1;
            const bool fpr = fs >= 0 && ad_c > thr;        // (pred - offset) > bsf * f, tree.py:282
            const bool scan = visit && !fpr;
            const unsigned smask = __ballot_sync(0xffffffffu, scan);
            const int need = s.R - ns;
            int end;                       // lanes [0, end) are consumed this iteration
            bool quota = false;
            if (__popc(smask) >= need) {
                unsigned mm = smask;
                for (int t = 1; t < need; ++t) mm &= mm - 1;      // clear the lowest need-1 bits
                end = __ffs(mm);                                   // include the need-th selected lane
                quota = true;
            } else {
                end = min(first_brk, len - cur);
            }
            const bool in = lane < end;
            const bool v_in = visit && in;
            const bool s_in = scan && in;
            const bool f_in = v_in && fs >= 0;
            const bool p_in = f_in && fpr;
            long long rows = 0;
            int chunks = 0;
            if (s_in) {
                rows = idx.d_leaf_ptr[leaf + 1] - idx.d_leaf_ptr[leaf];
                chunks = (int)((rows + CH - 1) / CH);
            }
            // inclusive warp scan of chunk counts over selected lanes
            int incl = chunks;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const unsigned sm_in = __ballot_sync(0xffffffffu, s_in);
            const unsigned vm_in = __ballot_sync(0xffffffffu, v_in);
            if (s_in) {
                const int slot = ns + __popc(sm_in & below);
                s.sel_leaf[q * s.Rcap + slot] = leaf;
                pre[slot] = nch + incl - chunks;
            }
            if (s.want_trace && v_in) {
                const int te = tl + __popc(vm_in & below);
                s.tr.d_leaf[tbase + te] = node;
                s.tr.d_lb[tbase + te] = lb;
                s.tr.d_searched[tbase + te] = s_in ? 1 : 0;
                s.tr.d_bsf_before[tbase + te] = bsf;
                if (!s_in) s.tr.d_leaf_nn[tbase + te] = __longlong_as_double(0x7ff8000000000000LL);
                else s.sel_trace[q * s.Rcap + ns + __popc(sm_in & below)] = te;
            }
            long long rsum = rows;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
            c_vis += __popc(vm_in);
            c_srch += __popc(sm_in);
            c_inf += __popc(__ballot_sync(0xffffffffu, f_in));
            c_fp += __popc(__ballot_sync(0xffffffffu, p_in));
            c_rows += rsum;
            tl += __popc(vm_in);
            ns += __popc(sm_in);
            nch += __shfl_sync(0xffffffffu, incl, 31);
            if (quota) {
                cur += end;
                quota_hit = true;
            } else if (first_brk < 32 && first_brk < len - cur) {
                // the break entry: a leaf counts as visited + lb-pruned (tree.py:261-269)
                const int bnode = __shfl_sync(0xffffffffu, node, first_brk);
                const int bleaf = __shfl_sync(0xffffffffu, leaf, first_brk);
                const double blb = __shfl_sync(0xffffffffu, lb, first_brk);
                if (bleaf >= 0) {
                    c_vis += 1;
                    c_lbp += 1;
                    if (s.want_trace && lane == 0) {
                        s.tr.d_leaf[tbase + tl] = bnode;
                        s.tr.d_lb[tbase + tl] = blb;
                        s.tr.d_searched[tbase + tl] = 0;
                        s.tr.d_leaf_nn[tbase + tl] = __longlong_as_double(0x7ff8000000000000LL);
                        s.tr.d_bsf_before[tbase + tl] = bsf;
                    }
                    tl += 1;
                }
                cur += first_brk;
                fin = true;
            } else {
                cur += end;
            }
            if (quota) break;
            if (end == 32) {
                lb_c = lb_n; rec_c = rec_n; ad_c = ad_n;
            } else {
                load(cur, lb_c, rec_c, ad_c);
            }
        }
        if (cur >= Nn) fin = true;
        if (lane == 0) {
            st[0] += c_vis; st[1] += c_srch; st[2] += c_lbp; st[3] += c_fp; st[4] += c_inf; st[5] += c_rows;
            s.cursor[q] = cur;
            if (s.want_trace) s.tr.d_len[q] = tl;
            if (fin) s.done[q] = 1;
            else atomicAdd(s.n_active, 1);
            if (!fin && !quota_hit && cur >= len) {
                if (len < olen) {                          // needs predictions further down
                    s.preq[q] = 1;
                    atomicAdd(s.n_predict, 1);
                } else {                                   // walked off the sorted prefix
                    s.refill[q] = 1;
                    atomicAdd(s.n_refill, 1);
                }
            }
        }
    }
    if (lane == 0) {
        pre[ns] = nch;
        s.n_sel[q] = ns;
        s.chunk_off[q + 1] = nch;
    }
}

// Exclusive scan of per-query chunk counts (single CTA; Q is small).
__global__ void offsets_kernel(long long* off, int64_t Q) {
    __shared__ long long part[1024];
    __shared__ long long carry;
    if (threadIdx.x == 0) { carry = 0; off[0] = 0; }
    __syncthreads();
    for (int64_t base = 0; base < Q; base += blockDim.x) {
        int64_t i = base + threadIdx.x;
        long long v = i < Q ? off[i + 1] : 0;
        part[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < (int)blockDim.x; o <<= 1) {
            long long add = threadIdx.x >= (unsigned)o ? part[threadIdx.x - o] : 0;
            __syncthreads();
            part[threadIdx.x] += add;
            __syncthreads();
        }
        if (i < Q) off[i + 1] = carry + part[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += part[threadIdx.x];
        __syncthreads();
    }
}

// Materialise this round's scan tasks: one warp per query writes
// (query, leaf, chunk) for each chunk of each selected leaf at chunk_off[q] + ...
__global__ void expand_tasks_kernel(RoundState s, const int64_t* __restrict__ leaf_ptr) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= s.Q) return;
    const int ns = s.n_sel[q];
    const long long base = s.chunk_off[q];
    const int* pre = s.sel_pre + q * (s.Rcap + 1);
    for (int j = 0; j < ns; ++j) {
        const int leaf = s.sel_leaf[q * s.Rcap + j];
        const int c0 = pre[j], n = pre[j + 1] - c0;
        const long long lb = leaf_ptr[leaf], le = leaf_ptr[leaf + 1];
        for (int c = lane; c < n; c += 32) {
            s.tasks[base + c0 + c] = make_int4((int)q, leaf, c, j);
            if (s.task_rows != nullptr) {   // row range of the task, so a producer needs no dependent loads
                const long long r0 = lb + (long long)c * CH;
                s.task_rows[base + c0 + c] = make_int4((int)(r0 & 0xffffffffLL), (int)(r0 >> 32),
                                                       (int)min((long long)CH, le - r0), (int)q);
            }
        }
    }
}

// ------------------------------------------------------- lazy inference ----
// After a round, a query with a finite bsf can only ever reach the visit-order
// positions [pcount, pend), pend = the first position whose bound exceeds bsf * f
// (bsf only decreases).  The leaves with a filter in that range are the (query,
// leaf) pairs whose prediction the cascade may need (tree.py:277-286 evaluates a
// subset of exactly these).  pass 1 counts them per filter, a single-CTA scan
// turns the counts into filter buckets and a 128-row tile list, pass 2 fills the
// buckets and gathers the query rows, and filter_pairs_tc (tcgen05, the same
// arithmetic as the dense filter kernel) writes pred - offset into the records.
constexpr int PRED_WINDOW = 1024;   // visit-order positions of a query's first prediction pass

__global__ void fill_int_kernel(int* p, int64_t n, int v) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void pairs_count_kernel(RoundState s, int* pend, int* fhist, unsigned long long* total, lf_index idx,
                                   int all) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= s.Q) return;
    const int start = s.pcount[q];
    const double thr = round_bsf(s, q) * s.f;
    const bool want = all || s.preq[q];
    __syncwarp();
    if (lane == 0) s.preq[q] = 0;
    if (s.done[q] || !(thr < kInf) || !want) {
        if (lane == 0) pend[q] = start;
        return;
    }
    const int Nn = idx.n_nodes;
    // a window of the order at a time (doubling per pass): LeaFi's filters stop most
    // walks long before the bound does (281 of 4,096 leaves visited per query on the
    // bench workload), so predicting every leaf under the bound would be ~15x the work
    const int win = s.pwin[q];
    const int len = min(s.olen[q], start + win);
    const double* lbs = s.lbs + q * Nn;
    const int* lrec = s.leafo + q * Nn;
    int i = start, cnt = 0;
    bool broke = false;
    while (i < len) {                                  // 128 positions per pass, loads in flight together
        double lbv[4];
        int recv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int k = i + 32 * u + lane;
            lbv[u] = k < len ? lbs[k] : kInf;
            recv[u] = k < len ? lrec[k] : -1;
        }
        bool stop = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (stop) break;
            const int k = i + 32 * u + lane;
            const bool valid = k < len;
            const bool brk = valid && lbv[u] > thr;
            const unsigned bmask = __ballot_sync(0xffffffffu, brk);
            const int first = bmask ? __ffs(bmask) - 1 : 32;
            const int rec = (valid && lane < first) ? recv[u] : -1;
            const bool has = rec >= 0 && (rec & LF_REC_HASF);
            if (has) atomicAdd(&fhist[idx.d_leaf_filter[rec & LF_REC_LEAF]], 1);
            cnt += __popc(__ballot_sync(0xffffffffu, has));
            if (bmask) { i += 32 * u + first; broke = true; stop = true; }
        }
        if (stop) break;
        i += 128;
    }
    if (lane == 0) s.pwin[q] = win * 2;
    if (lane == 0) {
        // the break entry itself stays walkable (its bound alone decides), so the walk
        // can finish there instead of asking for predictions again
        pend[q] = broke ? i + 1 : min(i, len);
        if (cnt) atomicAdd(total, (unsigned long long)cnt);
    }
}

// Filter buckets (exclusive scan of the per-filter counts) and the tile list
// (filter, first row, rows <= 128) in one CTA.
__global__ void pair_tiles_kernel(const int* __restrict__ fhist, int F, int* __restrict__ fcur, int4* __restrict__ tiles,
                                  int* __restrict__ ntiles) {
    __shared__ int sp[1024], st[1024];
    __shared__ int carry_p, carry_t;
    if (threadIdx.x == 0) { carry_p = 0; carry_t = 0; }
    __syncthreads();
    for (int base = 0; base < F; base += blockDim.x) {
        const int f = base + threadIdx.x;
        const int h = f < F ? fhist[f] : 0;
        sp[threadIdx.x] = h;
        st[threadIdx.x] = (h + 127) / 128;
        __syncthreads();
        for (int o = 1; o < (int)blockDim.x; o <<= 1) {
            const int ap = threadIdx.x >= (unsigned)o ? sp[threadIdx.x - o] : 0;
            const int at = threadIdx.x >= (unsigned)o ? st[threadIdx.x - o] : 0;
            __syncthreads();
            sp[threadIdx.x] += ap;
            st[threadIdx.x] += at;
            __syncthreads();
        }
        if (f < F) {
            const int p0 = carry_p + sp[threadIdx.x] - h;
            const int nt = (h + 127) / 128;
            const int t0 = carry_t + st[threadIdx.x] - nt;
            fcur[f] = p0;
            for (int t = 0; t < nt; ++t) tiles[t0 + t] = make_int4(f, p0 + 128 * t, min(128, h - 128 * t), 0);
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) { carry_p += sp[threadIdx.x]; carry_t += st[threadIdx.x]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) *ntiles = carry_t;
}

int pair_tiles(const int* d_hist, int F, int* d_fcur, int4* d_tiles, int* d_ntiles, cudaStream_t st) {
    pair_tiles_kernel<<<1, 1024, 0, st>>>(d_hist, F, d_fcur, d_tiles, d_ntiles);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

// Bucket the pairs by filter (slot order inside a bucket is irrelevant: every row's
// prediction depends on that row alone) and gather their query rows.
__global__ void pairs_fill_kernel(RoundState s, lf_index idx, const float* __restrict__ queries, int m, int* pcount,
                                  const int* __restrict__ pend, int* fcur, int2* __restrict__ dst,
                                  float* __restrict__ rows) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= s.Q) return;
    const int start = pcount[q], end = pend[q];
    const int Nn = idx.n_nodes;
    const int* lrec = s.leafo + q * Nn;
    const double* lbs = s.lbs + q * Nn;
    const double thr = round_bsf(s, q) * s.f;       // same bound as pass 1: skips its break entry
    for (int i = start; i < end; i += 32) {
        const int k = i + lane;
        const int rec = (k < end && lbs[k] <= thr) ? lrec[k] : -1;
        const bool has = rec >= 0 && (rec & LF_REC_HASF);
        if (has) {
            const int slot = atomicAdd(&fcur[idx.d_leaf_filter[rec & LF_REC_LEAF]], 1);
            dst[slot] = make_int2((int)q, k);
        }
    }
    if (lane == 0) pcount[q] = end;
}

// Gather the query row of every bucketed pair (warp per pair, 128-bit copies).
__global__ void pairs_gather_kernel(const float* __restrict__ queries, int m, const int2* __restrict__ dst, int64_t P,
                                    float* __restrict__ rows) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= P) return;
    const float4* src = reinterpret_cast<const float4*>(queries + (int64_t)dst[i].x * m);
    float4* out = reinterpret_cast<float4*>(rows + i * m);
    for (int c = lane; c < m / 4; c += 32) out[c] = __ldg(src + c);
}

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

// ------------------------------------------------------------ q8 scan ----
// Bounded scan over the int8 shadow (lf_quantize_rows): 1/4 of the bytes of
// every row decide whether the exact fp32 row must be read at all.
//
// Pipeline (one CTA = 1 producer warp + 8 consumer warps, 2 CTAs per SM,
// persistent over the round's task list):
//   producer : one elected lane streams each task's rows in stages of 64 rows
//              (64 x m int8 codes + 64 x 16 B row metadata; the first stage of
//              a task also carries the query's codes and a task header) into a
//              ring of shared-memory stages with cp.async.bulk (TMA bulk
//              copies, L2 evict-first), completion on a full mbarrier.  It runs
//              ahead across task boundaries, so HBM streaming never waits for a
//              task's serial tail, and consumers never wait on a global load to
//              learn what they are scanning.
//   consumers: a warp takes 8 rows of a stage, half a warp per 4 rows, 16 codes
//              per lane per 256-code pass: D = cx . cq with DP4A (exact int32;
//              the query codes cq were quantised once per batch by
//              quantize_queries_kernel).  A transposing butterfly (5 shuffles
//              for 4 rows) leaves every lane with one full row dot, so the bound
//              arithmetic runs once per row on all lanes instead of serially:
//              ||x^ - q^||^2 = sx^2 xx + sq^2 qq - 2 sx sq D (fp32, rounding
//              bounded by tol = 1e-5 (sx^2 xx + sq^2 qq)), and by the triangle
//              inequality the true distance lies in
//              [sqrt(.. - tol) - ex - eq, sqrt(.. + tol) + ex + eq] (widened 1e-6).
//              One arrive per warp releases the stage to the producer.
//   tail     : for k = 1 the task's best row is within min_r hi_r, so a row whose
//              lo exceeds min(bsf, min hi) can never be the answer; every other
//              row (the few that remain) is re-read whole from HBM and summed
//              EXACTLY in fp64 -- kept distances are exact, dropped rows
//              provably worse.
constexpr int Q8_ROWS = 64;
constexpr int Q8_CONS_WARPS = 8;
constexpr int Q8_CONS = 32 * Q8_CONS_WARPS;
constexpr int Q8_THREADS = Q8_CONS + 32;
static_assert(Q8_ROWS == 8 * Q8_CONS_WARPS, "8 rows per consumer warp per stage");

template <int NCH>
struct Q8Cfg {
    static constexpr int M = NCH * 64;
    static constexpr int P = (M + 255) / 256;              // 256-code passes per row (16 codes per lane)
    static constexpr int CODE_BYTES = Q8_ROWS * M;
    static constexpr int META_OFF = CODE_BYTES;             // 64 x float4 row metadata
    static constexpr int QC_OFF = META_OFF + Q8_ROWS * 16;  // query codes (first stage of a task)
    static constexpr int QM_OFF = QC_OFF + P * 256;         // query metadata float4
    static constexpr int HDR_OFF = QM_OFF + 16;             // {r0 (i64), q (i32), nrows (i32)}
    static constexpr int STAGE_BYTES = (HDR_OFF + 16 + 127) / 128 * 128;
    static constexpr int STAGES = (81920 / CODE_BYTES) < 2 ? 2 : ((81920 / CODE_BYTES) > 8 ? 8 : 81920 / CODE_BYTES);
    static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
    static constexpr int LO_OFF = BAR_OFF + 2 * STAGES * 8;
    static constexpr int SR_OFF = LO_OFF + CH * 4;
    static constexpr int SD_OFF = SR_OFF + CH * 4;
    static constexpr int HI_OFF = SD_OFF + CH * 8;                   // upper ends (k > 1)
    static constexpr int HIST_OFF = HI_OFF + CH * 4;                 // 256-bin radix-select histogram
    static constexpr int MISC_OFF = HIST_OFF + 256 * 4;
    static constexpr int SMEM = MISC_OFF + 32;
};

__device__ __forceinline__ uint32_t q8_su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void q8_bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(q8_su32(b)), "r"(n));
}
__device__ __forceinline__ void q8_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(q8_su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void q8_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(q8_su32(b)) : "memory");
}
__device__ __forceinline__ void q8_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LF_Q8W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LF_Q8W_%=;\n}" ::"r"(q8_su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void q8_bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            q8_su32(dst)),
        "l"(src), "r"(bytes), "r"(q8_su32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void q8_cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(Q8_CONS) : "memory"); }

template <int NCH>
__global__ void __launch_bounds__(Q8_THREADS, 2) scan_q8_kernel(RoundState s, lf_index idx,
                                                                const float* __restrict__ queries,
                                                                const int8_t* __restrict__ qcodes,
                                                                const float4* __restrict__ qmeta) {
    using Cfg = Q8Cfg<NCH>;
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
    const int hl = lane & 15;
    const int rbase = cw * 8 + (lane >> 4) * 4;        // this half-warp's 4 rows of a stage
    const bool b8 = (hl & 8) != 0, b4 = (hl & 4) != 0;
    const int myrow = rbase + (b8 ? 2 : 0) + (b4 ? 1 : 0);   // row whose total this lane ends with
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
            if (myrow < rows) {
                const float4 mr = *reinterpret_cast<const float4*>(stg + Cfg::META_OFF + myrow * 16);
                const float sx2xx = mr.x * mr.x * mr.y;
                const float e = mr.z + eq;
                const float d2 = sx2xx + sq2qq - 2.f * (mr.x * sq) * (float)d[0];
                const float tol = 1e-5f * (sx2xx + sq2qq);
                const float lo = (sqrtf(fmaxf(d2 - tol, 0.f)) - e) * (1.f - 1e-6f);
                const float hi = (sqrtf(fmaxf(d2 + tol, 0.f)) + e) * (1.f + 1e-6f);
                hmin = fminf(hmin, hi);
                if ((hl & 3) == 0) {
                    lo_s[j + myrow] = lo;
                    if (s.k > 1) hi_s[j + myrow] = hi;
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
            for (int b0 = 0; b0 < ns; b0 += 16) {
                const int jj = b0 + hslot;
                const bool v = jj < ns;
                const int r = v ? surv_r[jj] : 0;
                float4 x[NCH];
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
                    x[ch] = (v && ch * 64 + hl * 4 < mr)
                                ? __ldg(reinterpret_cast<const float4*>(X0 + (int64_t)r * mr) + ch * 16 + hl)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
                double acc = 0.0;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const float4 qv = ch * 64 + hl * 4 < mr
                                          ? __ldg(reinterpret_cast<const float4*>(qrow) + ch * 16 + hl)
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

constexpr int PQ_SQ = 64;                     // survivors of a task handed to survivor_exact_kernel

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

// --------------------------------------------------------------- merge ----
// One warp per query: k smallest (d, id) among the running top-k and this
// round's candidates (each series is scanned at most once per query, so all
// (d, id) pairs are distinct and repeated "next larger than the last pick"
// selection is exact).  Reads top_* (round-start state), writes top_*_out.
__global__ void merge_kernel(RoundState s) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= s.Q) return;
    const int ns = s.n_sel[q];
    const double* td = s.top_d + q * s.k;
    const long long* ti = s.top_i + q * s.k;
    double* od = s.top_d_out + q * s.k;
    long long* oi = s.top_i_out + q * s.k;
    const int tn = s.top_n[q];
    if (ns == 0) {
        for (int i = lane; i < tn; i += 32) { od[i] = td[i]; oi[i] = ti[i]; }
        if (lane == 0) s.top_n_out[q] = tn;
        return;
    }
    const long long c0 = s.chunk_off[q], c1 = s.chunk_off[q + 1];
    const long long nc = (c1 - c0) * s.kc;
    const double* cd = s.cand_d + c0 * s.kc;
    const long long* ci = s.cand_i + c0 * s.kc;

    if (s.want_trace) {
        const int* pre = s.sel_pre + q * (s.Rcap + 1);
        for (int j = lane; j < ns; j += 32) {
            double mn = kInf;
            for (int c = pre[j]; c < pre[j + 1]; ++c) mn = fmin(mn, s.task_min[c0 + c]);
            const int te = s.sel_trace[q * s.Rcap + j];
            s.tr.d_leaf_nn[q * (int64_t)s.n_leaves + te] = mn;
        }
    }

    double last_d = -1.0;
    long long last_i = -1;
    int filled = 0;
    for (int sel = 0; sel < s.k; ++sel) {
        double bd = kInf;
        long long bi = LLONG_MAX;
        for (int i = lane; i < tn; i += 32) {
            const double d = td[i];
            const long long id = ti[i];
            if (pair_less(last_d, last_i, d, id) && pair_less(d, id, bd, bi)) { bd = d; bi = id; }
        }
        for (long long i = lane; i < nc; i += 32) {
            const long long id = ci[i];
            if (id < 0) continue;
            const double d = cd[i];
            if (pair_less(last_d, last_i, d, id) && pair_less(d, id, bd, bi)) { bd = d; bi = id; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double xd = __shfl_xor_sync(0xffffffffu, bd, o);
            const long long xi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (pair_less(xd, xi, bd, bi)) { bd = xd; bi = xi; }
        }
        if (bi == LLONG_MAX) break;
        if (lane == 0) { od[sel] = bd; oi[sel] = bi; }
        last_d = bd;
        last_i = bi;
        ++filled;
    }
    if (lane == 0) s.top_n_out[q] = filled;
}

__global__ void init_state_kernel(RoundState s) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= s.Q) return;
    s.cursor[q] = 0;
    s.done[q] = 0;
    s.top_n[q] = 0;
    for (int i = 0; i < LF_N_STATS; ++i) s.stats[q * LF_N_STATS + i] = 0;
    if (s.want_trace) s.tr.d_len[q] = 0;
}

__global__ void finish_kernel(RoundState s, int64_t* out_ids, double* out_d) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= s.Q * s.k) return;
    int64_t q = t / s.k;
    int i = (int)(t - q * s.k);
    bool ok = i < s.top_n[q];
    out_ids[t] = ok ? s.top_i[t] : -1;
    out_d[t] = ok ? s.top_d[t] : kInf;
}

// Visit orders as full per-query sorts (default) or sorted prefixes + refill
// (LF_FULL_ORDER=0).  LeaFi walks deep into the order -- its filters prune most
// visited leaves (bench: 281 leaves visited per query, 1,202 at most), so a
// 1,024-entry prefix sends ~27% of the queries to a refill and the full sort wins.
static bool prefix_orders() {
    const char* e = getenv("LF_FULL_ORDER");
    return e && e[0] == '0';
}

// Scan variant (experiments): LF_SCAN_VARIANT = q8 (default) | ea2 | ea3 | full.
// Scan variant: LF_SCAN_VARIANT = q8 (default: full-length int8 shadow, at the HBM
// roofline) | pq (projected shadow after round 0: ~3x fewer bytes, but latency-bound
// on the survivor re-reads -- measured 0.96-1.05x of q8 depending on the box) |
// ea2 | ea3 | full.
static int scan_variant() {
    const char* e = getenv("LF_SCAN_VARIANT");
    if (e && strcmp(e, "pq") == 0) return 8;       // projected stage when the shadow exists
    if (!e || strcmp(e, "q8") == 0) return 9;      // int8 shadow only
    if (e && strcmp(e, "ea3") == 0) return 3;
    if (e && strcmp(e, "full") == 0) return 0;
    if (e && strcmp(e, "ea2") == 0) return 2;
    return 8;                                      // default: int8-bounded scan when the shadow exists
}

template <int NCH>
static cudaError_t launch_scan_ea(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc8,
                                  const float4* qm8, int sms, cudaStream_t st) {
    if (qc8 != nullptr) {
        static bool attr = false;       // one instantiation per NCH
        if (!attr) {
            cudaError_t e = cudaFuncSetAttribute(scan_q8_kernel<NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 Q8Cfg<NCH>::SMEM);
            if (e != cudaSuccess) return e;
            attr = true;
        }
        scan_q8_kernel<NCH><<<sms * 2, Q8_THREADS, Q8Cfg<NCH>::SMEM, st>>>(s, idx, q, qc8, qm8);
    } else if (scan_variant() == 3)
        scan_ea3_kernel<NCH><<<sms * 4, SCAN_THREADS, 0, st>>>(s, idx, q);
    else
        scan_ea2_kernel<NCH><<<sms * 3, SCAN_THREADS, 0, st>>>(s, idx, q);
    return cudaGetLastError();
}

template <int VEC>
static cudaError_t launch_scan(const RoundState& s, const lf_index& idx, const float* q, int grid,
                               cudaStream_t st) {
    scan_kernel<VEC><<<grid, SCAN_THREADS, 0, st>>>(s, idx, q);
    return cudaGetLastError();
}

}  // namespace lf

// A search over one query batch, split into begin / rounds / end so a caller can
// exchange the per-query best-so-far between rounds (leaf-sharded multi-GPU).
struct lf_session {
    lf_index idx{};
    lf_search_opts opts{};
    lf_trace tr{};
    cudaStream_t st = nullptr;
    int64_t Q = 0;
    const float* d_q = nullptr;
    lf::RoundState s{};
    lf::Scratch qsumm, lb, lbs, order, cursor, done, topd, topi, topn, topd2, topi2, topn2, sel_leaf,
        sel_trace, sel_pre, n_sel, chunk_off, cand_d, cand_i, task_min, n_active, tasks, ea_count, qc8, qm8,
        leafo, adj, olen, refill, pcount, pend, preq, pwin, fhist, fcur, ntiles, ptotal;
    lf::OrderArgs oa{};
    bool lazy = false;               // lazy filter inference (opts.d_W1T instead of predictions)
    long long pairs = 0;             // predictions computed lazily
    int predict_steps = 0;
    double predict_ms = 0.0;
    bool q8 = false;                 // int8-bounded scan (query codes quantised once in begin)
    bool grouped = false;            // q8 scan with the round's tasks grouped by (leaf, chunk)
    bool pq = false;                 // two-stage scan over the projected shadow (d_Xp)
    lf::Scratch qcp, qmp, pq_cnt, pq_rows, pq_trows;
    lf::Scratch cbase, ghist, gcur, gsorted, glist, gcount, gbsum, ginfo;
    int n_keys = 0;
    long long refills = 0;           // queries whose visit order was completed after the prefix
    int* h_active = nullptr;         // pinned [2 slots][4]: active, refill, predict requests
    int round = 0;                   // rounds enqueued
    int harvested = 0;               // rounds whose counts were read back
    cudaEvent_t rev[2][4] = {};      // per slot: plan start, scan start, merge start, merge end
    cudaEvent_t done_ev[2] = {};     // per slot: counts copied back
    long long kernels = 0;
    cudaEvent_t ev[6] = {};
    bool prof = false;
};

namespace lf {

static int session_begin(lf_session* ss) {
    const lf_index& idx = ss->idx;
    const lf_search_opts& o = ss->opts;
    cudaStream_t st = ss->st;
    const int64_t Q = ss->Q;
    const int Nn = idx.n_nodes;
    RoundState& s = ss->s;
    s.Q = Q;
    s.k = o.k;
    s.kc = std::min(o.k, CH);
    s.f = o.bsf_factor;
    s.Rcap = o.sequential ? 1 : std::max(1, std::min(o.max_round_leaves, std::max(1, idx.n_leaves)));
    s.pred = o.d_pred;
    s.pred64 = o.d_pred_f64;
    s.offset = o.d_offset;
    s.F = o.n_filters;
    s.want_trace = o.want_trace ? 1 : 0;
    if (s.want_trace) s.tr = ss->tr;
    s.n_leaves = idx.n_leaves;
    s.bound = nullptr;

    const int64_t max_chunks_leaf = std::max<int64_t>(1, (idx.max_leaf_rows + CH - 1) / CH);
    const int64_t max_tasks = std::max<int64_t>(1, Q * s.Rcap * max_chunks_leaf);
    LF_CUDA(ss->qsumm.alloc(sizeof(double) * Q * idx.n_seg, st));
    LF_CUDA(ss->lb.alloc(Nn > 8192 ? sizeof(double) * Q * Nn : 16, st));   // only the unfused path uses it
    LF_CUDA(ss->lbs.alloc(sizeof(double) * Q * Nn, st));
    LF_CUDA(ss->order.alloc(sizeof(int) * Q * Nn, st));
    LF_CUDA(ss->leafo.alloc(sizeof(int) * Q * Nn, st));
    LF_CUDA(ss->adj.alloc(sizeof(double) * Q * Nn, st));
    LF_CUDA(ss->olen.alloc(sizeof(int) * Q, st));
    LF_CUDA(ss->refill.alloc(sizeof(int) * Q, st));
    LF_CUDA(cudaMemsetAsync(ss->refill.p, 0, sizeof(int) * Q, st));
    LF_CUDA(ss->cursor.alloc(sizeof(int) * Q, st));
    LF_CUDA(ss->done.alloc(sizeof(int) * Q, st));
    LF_CUDA(ss->topd.alloc(sizeof(double) * Q * s.k, st));
    LF_CUDA(ss->topi.alloc(sizeof(long long) * Q * s.k, st));
    LF_CUDA(ss->topn.alloc(sizeof(int) * Q, st));
    LF_CUDA(ss->topd2.alloc(sizeof(double) * Q * s.k, st));
    LF_CUDA(ss->topi2.alloc(sizeof(long long) * Q * s.k, st));
    LF_CUDA(ss->topn2.alloc(sizeof(int) * Q, st));
    LF_CUDA(ss->sel_leaf.alloc(sizeof(int) * Q * s.Rcap, st));
    LF_CUDA(ss->sel_trace.alloc(sizeof(int) * Q * s.Rcap, st));
    LF_CUDA(ss->sel_pre.alloc(sizeof(int) * Q * (s.Rcap + 1), st));
    LF_CUDA(ss->n_sel.alloc(sizeof(int) * Q, st));
    LF_CUDA(ss->chunk_off.alloc(sizeof(long long) * (Q + 1), st));
    LF_CUDA(ss->cand_d.alloc(sizeof(double) * max_tasks * s.kc, st));
    LF_CUDA(ss->cand_i.alloc(sizeof(long long) * max_tasks * s.kc, st));
    LF_CUDA(ss->task_min.alloc(sizeof(double) * (s.want_trace ? max_tasks : 1), st));
    LF_CUDA(ss->n_active.alloc(sizeof(int) * 8, st));   // [2 slots][active, refill, predict requests, -]
    for (int sl = 0; sl < 2; ++sl) {
        LF_CUDA(cudaEventCreateWithFlags(&ss->done_ev[sl], cudaEventDisableTiming));
        if (o.h_profile)
            for (auto& e : ss->rev[sl]) LF_CUDA(cudaEventCreate(&e));
    }
    ss->lazy = o.d_pred == nullptr && o.d_pred_f64 == nullptr && o.d_W1T != nullptr;
    if (ss->lazy) {
        LF_CUDA(ss->pcount.alloc(sizeof(int) * Q, st));
        LF_CUDA(cudaMemsetAsync(ss->pcount.p, 0, sizeof(int) * Q, st));
        LF_CUDA(ss->pend.alloc(sizeof(int) * Q, st));
        LF_CUDA(ss->preq.alloc(sizeof(int) * Q, st));
        LF_CUDA(cudaMemsetAsync(ss->preq.p, 0, sizeof(int) * Q, st));
        LF_CUDA(ss->pwin.alloc(sizeof(int) * Q, st));
        fill_int_kernel<<<(unsigned)((Q + 255) / 256), 256, 0, st>>>(ss->pwin.as<int>(), Q, PRED_WINDOW);
        LF_CUDA(cudaGetLastError());
        LF_CUDA(ss->fhist.alloc(sizeof(int) * std::max(1, o.n_filters), st));
        LF_CUDA(ss->fcur.alloc(sizeof(int) * std::max(1, o.n_filters), st));
        LF_CUDA(ss->ntiles.alloc(sizeof(int), st));
        LF_CUDA(ss->ptotal.alloc(sizeof(unsigned long long), st));
    }
    LF_CUDA(ss->tasks.alloc(sizeof(int4) * max_tasks, st));
    LF_CUDA(ss->ea_count.alloc(sizeof(unsigned long long) * 4, st));
    LF_CUDA(cudaMemsetAsync(ss->ea_count.p, 0, sizeof(unsigned long long) * 4, st));
    {   // one pinned word per host thread; a round reads it right after its own sync
        static thread_local int* pinned = nullptr;
        if (pinned == nullptr) LF_CUDA(cudaMallocHost(&pinned, sizeof(int) * 8));
        ss->h_active = pinned;
    }

    if (o.h_profile) {
        ss->prof = true;
        for (int i = 0; i < LF_N_PROF; ++i) o.h_profile[i] = 0.0;
        for (auto& e : ss->ev) LF_CUDA(cudaEventCreate(&e));
        LF_CUDA(cudaEventRecord(ss->ev[0], st));
    }
    int nk = 0;
    OrderArgs& oa = ss->oa;
    oa.lbs = ss->lbs.as<double>();
    oa.order = ss->order.as<int>();
    oa.leafo = ss->leafo.as<int>();
    oa.adj = ss->adj.as<double>();
    oa.olen = ss->olen.as<int>();
    oa.pred = o.d_pred;
    oa.pred64 = o.d_pred_f64;
    oa.offset = o.d_offset;
    oa.F = o.n_filters;
    oa.only = nullptr;
    oa.lazy = ss->lazy ? 1 : 0;
    int rc = bounds_and_order(ss->d_q, Q, idx, ss->qsumm.as<double>(), ss->lb.as<double>(), oa, prefix_orders(),
                              st, &nk);
    if (rc) return rc;
    ss->kernels += nk;

    s.order = ss->order.as<int>();
    s.lbs = ss->lbs.as<double>();
    s.leafo = ss->leafo.as<int>();
    s.adj = ss->adj.as<double>();
    s.olen = ss->olen.as<int>();
    s.refill = ss->refill.as<int>();
    s.n_refill = ss->n_active.as<int>() + 1;
    s.n_predict = ss->n_active.as<int>() + 2;
    s.lazy = ss->lazy ? 1 : 0;
    s.pcount = ss->lazy ? ss->pcount.as<int>() : nullptr;
    s.preq = ss->lazy ? ss->preq.as<int>() : nullptr;
    s.pwin = ss->lazy ? ss->pwin.as<int>() : nullptr;
    s.cursor = ss->cursor.as<int>();
    s.done = ss->done.as<int>();
    s.top_d = ss->topd.as<double>();
    s.top_i = ss->topi.as<long long>();
    s.top_n = ss->topn.as<int>();
    s.top_d_out = ss->topd2.as<double>();
    s.top_i_out = ss->topi2.as<long long>();
    s.top_n_out = ss->topn2.as<int>();
    s.sel_leaf = ss->sel_leaf.as<int>();
    s.sel_trace = ss->sel_trace.as<int>();
    s.sel_pre = ss->sel_pre.as<int>();
    s.n_sel = ss->n_sel.as<int>();
    s.chunk_off = ss->chunk_off.as<long long>();
    s.cand_d = ss->cand_d.as<double>();
    s.cand_i = ss->cand_i.as<long long>();
    s.task_min = ss->task_min.as<double>();
    s.n_active = ss->n_active.as<int>();
    s.tasks = ss->tasks.as<int4>();
    s.ea_count = o.h_profile ? ss->ea_count.as<unsigned long long>() : nullptr;

    init_state_kernel<<<(unsigned)((Q + 127) / 128), 128, 0, st>>>(s);
    LF_CUDA(cudaGetLastError());
    ++ss->kernels;
    ss->q8 = idx.d_X8 != nullptr && idx.d_qmeta != nullptr && o.early_abandon && !s.want_trace &&
             (idx.m % 4) == 0 && idx.m <= 512 && (scan_variant() == 8 || scan_variant() == 9);
    ss->pq = idx.d_Xp != nullptr && idx.d_pmeta != nullptr && (idx.pca_k == 32 || idx.pca_k == 64) &&
             o.early_abandon && !s.want_trace && (idx.m % 4) == 0 && idx.m <= 512 && scan_variant() == 8;
    if (ss->pq) {
        LF_CUDA(ss->qcp.alloc((size_t)Q * idx.pca_k, st));
        LF_CUDA(ss->qmp.alloc(sizeof(float4) * Q, st));
        LF_CUDA(ss->pq_cnt.alloc(sizeof(int) * max_tasks, st));
        LF_CUDA(ss->pq_trows.alloc(sizeof(int4) * max_tasks, st));
        s.task_rows = ss->pq_trows.as<int4>();
        LF_CUDA(ss->pq_rows.alloc(sizeof(unsigned short) * PQ_SQ * max_tasks, st));
        project_queries_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(
            ss->d_q, Q, idx.m, idx.pca_k, idx.pca_k, idx.d_P, idx.d_mu, ss->qcp.as<int8_t>(), ss->qmp.as<float4>());
        LF_CUDA(cudaGetLastError());
        ++ss->kernels;
    }
    if (ss->q8) {
        // grouping by (leaf, chunk) reads ~1/3 fewer int8 bytes on the bench workload but its
        // round overhead (~30 us) eats the gain there (scan 3.95 -> 3.82 ms, +0.27 ms grouping),
        // so it is opt-in: LF_SCAN_GROUP=1
        const char* ge = getenv("LF_SCAN_GROUP");
        ss->grouped = ge && ge[0] == '1';
        if (ss->grouped) {
            LF_CUDA(ss->cbase.alloc(sizeof(int) * (idx.n_leaves + 1), st));
            chunk_base_kernel<<<1, 1024, 0, st>>>(idx.d_leaf_ptr, idx.n_leaves, ss->cbase.as<int>());
            LF_CUDA(cudaGetLastError());
            LF_CUDA(cudaMemcpyAsync(&ss->n_keys, ss->cbase.as<int>() + idx.n_leaves, sizeof(int),
                                    cudaMemcpyDeviceToHost, st));
            LF_CUDA(cudaStreamSynchronize(st));
            LF_CUDA(ss->ghist.alloc(sizeof(int) * std::max(1, ss->n_keys), st));
            LF_CUDA(ss->gcur.alloc(sizeof(int) * std::max(1, ss->n_keys), st));
            LF_CUDA(ss->gsorted.alloc(sizeof(int) * max_tasks, st));
            LF_CUDA(ss->glist.alloc(sizeof(int2) * max_tasks, st));
            LF_CUDA(ss->ginfo.alloc(sizeof(GroupInfo) * max_tasks, st));
            LF_CUDA(ss->gcount.alloc(sizeof(int), st));
            LF_CUDA(ss->gbsum.alloc(sizeof(int2) * ((ss->n_keys + GL_THREADS - 1) / GL_THREADS + 1), st));
            ++ss->kernels;
        }
        const int MP = (idx.m + 255) / 256 * 256;
        LF_CUDA(ss->qc8.alloc((size_t)Q * MP, st));
        LF_CUDA(ss->qm8.alloc(sizeof(float4) * Q, st));
        int rq = quantize_queries(ss->d_q, Q, idx.m, MP, ss->qc8.as<int8_t>(), ss->qm8.as<float4>(), st);
        if (rq) return rq;
        ++ss->kernels;
    }
    if (ss->prof) LF_CUDA(cudaEventRecord(ss->ev[1], st));
    return LF_OK;
}

static float ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

__global__ void bsf_out_kernel(RoundState s, double* out) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q < s.Q) out[q] = query_bsf(s, q);
}

// Lazy filter inference for every query with a finite bsf (see pairs_count_kernel).
static int predict_step(lf_session* ss) {
    RoundState& s = ss->s;
    const lf_index& idx = ss->idx;
    const lf_search_opts& o = ss->opts;
    cudaStream_t st = ss->st;
    const int64_t Q = ss->Q;
    const int F = o.n_filters;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ss->prof) {
        LF_CUDA(cudaEventCreate(&e0));
        LF_CUDA(cudaEventCreate(&e1));
        LF_CUDA(cudaEventRecord(e0, st));
    }
    LF_CUDA(cudaMemsetAsync(ss->fhist.p, 0, sizeof(int) * std::max(1, F), st));
    LF_CUDA(cudaMemsetAsync(ss->ptotal.p, 0, sizeof(unsigned long long), st));
    const unsigned wgrid = (unsigned)((Q * 32 + 255) / 256);
    pairs_count_kernel<<<wgrid, 256, 0, st>>>(s, ss->pend.as<int>(), ss->fhist.as<int>(),
                                              ss->ptotal.as<unsigned long long>(), idx, ss->round == 0 ? 1 : 0);
    LF_CUDA(cudaGetLastError());
    unsigned long long total = 0;
    LF_CUDA(cudaMemcpyAsync(&total, ss->ptotal.p, sizeof(total), cudaMemcpyDeviceToHost, st));
    LF_CUDA(cudaStreamSynchronize(st));
    ss->kernels += 1;
    if (total == 0) {
        LF_CUDA(cudaMemcpyAsync(ss->pcount.p, ss->pend.p, sizeof(int) * Q, cudaMemcpyDeviceToDevice, st));
    } else {
        const int64_t P = (int64_t)total;
        Scratch rows, dst, tiles;
        LF_CUDA(rows.alloc(sizeof(float) * (size_t)P * idx.m, st));
        LF_CUDA(dst.alloc(sizeof(int2) * (size_t)P, st));
        LF_CUDA(tiles.alloc(sizeof(int4) * (size_t)(P / 128 + F + 1), st));
        pair_tiles_kernel<<<1, 1024, 0, st>>>(ss->fhist.as<int>(), F, ss->fcur.as<int>(), tiles.as<int4>(),
                                              ss->ntiles.as<int>());
        LF_CUDA(cudaGetLastError());
        pairs_fill_kernel<<<wgrid, 256, 0, st>>>(s, idx, ss->d_q, idx.m, ss->pcount.as<int>(), ss->pend.as<int>(),
                                                 ss->fcur.as<int>(), dst.as<int2>(), rows.as<float>());
        LF_CUDA(cudaGetLastError());
        pairs_gather_kernel<<<(unsigned)((P * 32 + 255) / 256), 256, 0, st>>>(ss->d_q, idx.m, dst.as<int2>(), P,
                                                                             rows.as<float>());
        LF_CUDA(cudaGetLastError());
        int rc = filter_pairs_tc(rows.as<float>(), P, idx.m, o.d_W1T, o.d_b1, o.d_W2, o.d_b2, F, tiles.as<int4>(),
                                 ss->ntiles.as<int>(), dst.as<int2>(), o.d_offset, ss->adj.as<double>(), idx.n_nodes,
                                 st);
        if (rc) return rc;
        ss->kernels += 4;
        ss->pairs += P;
        ++ss->predict_steps;
    }
    if (ss->prof) {
        LF_CUDA(cudaEventRecord(e1, st));
        LF_CUDA(cudaEventSynchronize(e1));
        ss->predict_ms += ev_ms(e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    return LF_OK;
}

// Enqueue one round (plan, scan, merge) into count slot round & 1; the counts are
// copied back asynchronously (done_ev).  session_harvest reads them.
static int session_enqueue(lf_session* ss, const double* d_bound, double* d_bsf_out) {
    RoundState& s = ss->s;
    const lf_index& idx = ss->idx;
    const lf_search_opts& o = ss->opts;
    cudaStream_t st = ss->st;
    const int64_t Q = ss->Q;
    const int slot = ss->round & 1;
    int* counts = ss->n_active.as<int>() + 4 * slot;
    s.n_active = counts;
    s.n_refill = counts + 1;
    s.n_predict = counts + 2;
    cudaEvent_t* ev = ss->rev[slot];
    s.bound = d_bound;
    s.R = o.sequential ? 1 : (int)std::min<int64_t>(s.Rcap, (int64_t)1 << std::min(ss->round, 30));
    LF_CUDA(cudaMemsetAsync(counts, 0, sizeof(int) * 3, st));
    if (ss->prof) cudaEventRecord(ev[0], st);
    plan_warp_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(s, idx);
    offsets_kernel<<<1, 1024, 0, st>>>(s.chunk_off, Q);
    expand_tasks_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(s, idx.d_leaf_ptr);
    if (ss->prof) cudaEventRecord(ev[1], st);
    const int grid = sm_count() * 4;
    const int m4 = idx.m / 4;
    cudaError_t ce;
    // the int8-bounded scan takes m % 4 == 0 (codes zero-padded to a multiple of 64); the fp32
    // early-abandon variants need m % 64 == 0
    const bool ea = o.early_abandon && !s.want_trace && idx.m <= 512 && scan_variant() != 0 &&
                    ((idx.m % 64) == 0 || (ss->q8 && (idx.m % 4) == 0));
    const int nch = (idx.m + 63) / 64;
    // round 0 has no best-so-far yet: the projected bound's loose upper end would let
    // most rows through, so the first round runs the full-length int8 scan
    if (ea && ss->pq && !(ss->round == 0 && ss->q8)) {
        const int sms = sm_count();
        if (idx.pca_k == 32) {
            static bool attr = false;
            if (!attr) {
                LF_CUDA(cudaFuncSetAttribute(scan_pq_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             PQCfg<32>::SMEM));
                attr = true;
            }
            scan_pq_kernel<32><<<sms * 2, Q8_THREADS, PQCfg<32>::SMEM, st>>>(
                s, idx, ss->d_q, ss->qcp.as<int8_t>(), ss->qmp.as<float4>(), ss->pq_cnt.as<int>(),
                ss->pq_rows.as<unsigned short>());
        } else {
            static bool attr = false;
            if (!attr) {
                LF_CUDA(cudaFuncSetAttribute(scan_pq_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             PQCfg<64>::SMEM));
                attr = true;
            }
            scan_pq_kernel<64><<<sms * 2, Q8_THREADS, PQCfg<64>::SMEM, st>>>(
                s, idx, ss->d_q, ss->qcp.as<int8_t>(), ss->qmp.as<float4>(), ss->pq_cnt.as<int>(),
                ss->pq_rows.as<unsigned short>());
        }
        const int64_t max_tasks = std::max<int64_t>(
            1, Q * s.Rcap * std::max<int64_t>(1, (idx.max_leaf_rows + CH - 1) / CH));
        survivor_exact_kernel<<<(unsigned)((max_tasks * 32 + 255) / 256), 256, 0, st>>>(
            s, idx, ss->d_q, ss->pq_cnt.as<int>(), ss->pq_rows.as<unsigned short>());
        ++ss->kernels;
        ce = cudaGetLastError();
    } else if (ea && ss->q8 && ss->grouped) {
        // group the round's tasks by (leaf, chunk), then one pass per chunk serves them all
        const int64_t max_tasks = std::max<int64_t>(
            1, Q * s.Rcap * std::max<int64_t>(1, (idx.max_leaf_rows + CH - 1) / CH));
        const unsigned tgrid = (unsigned)((max_tasks + 255) / 256);
        LF_CUDA(cudaMemsetAsync(ss->ghist.p, 0, sizeof(int) * std::max(1, ss->n_keys), st));
        group_hist_kernel<<<tgrid, 256, 0, st>>>(s, ss->cbase.as<int>(), ss->ghist.as<int>());
        {
            const int nb = (ss->n_keys + GL_THREADS - 1) / GL_THREADS;
            group_blocksum_kernel<<<nb, GL_THREADS, 0, st>>>(ss->ghist.as<int>(), ss->n_keys, ss->gbsum.as<int2>());
            group_blockscan_kernel<<<1, 1024, 0, st>>>(ss->gbsum.as<int2>(), nb, ss->gcount.as<int>());
            group_write_kernel<<<nb, GL_THREADS, 0, st>>>(ss->ghist.as<int>(), ss->n_keys, ss->gbsum.as<int2>(),
                                                          ss->gcur.as<int>(), ss->glist.as<int2>());
        }
        group_scatter_kernel<<<tgrid, 256, 0, st>>>(s, ss->cbase.as<int>(), ss->gcur.as<int>(),
                                                    ss->gsorted.as<int>());
        group_info_kernel<<<tgrid, 256, 0, st>>>(s, idx, ss->gsorted.as<int>(), ss->glist.as<int2>(),
                                                 ss->gcount.as<int>(), ss->ginfo.as<GroupInfo>());
        LF_CUDA(cudaGetLastError());
        ss->kernels += 6;
        if (ss->prof) cudaEventRecord(ev[1], st);          // grouping counts as planning
        const int sms = sm_count();
        switch (nch) {
#define LF_GROUPED(N)                                                                                          \
    case N: {                                                                                                 \
        static bool attr = false;                                                                             \
        if (!attr) {                                                                                          \
            LF_CUDA(cudaFuncSetAttribute(scan_q8g_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                                         Q8GCfg<N>::SMEM));                                                   \
            attr = true;                                                                                      \
        }                                                                                                     \
        scan_q8g_kernel<N><<<sms, G_THREADS, Q8GCfg<N>::SMEM, st>>>(                                          \
            s, idx, ss->d_q, ss->qc8.as<int8_t>(), ss->qm8.as<float4>(), ss->gsorted.as<int>(),               \
            ss->ginfo.as<GroupInfo>(), ss->gcount.as<int>());                                                 \
        break;                                                                                                \
    }
            LF_GROUPED(1) LF_GROUPED(2) LF_GROUPED(3) LF_GROUPED(4)
            LF_GROUPED(5) LF_GROUPED(6) LF_GROUPED(7) LF_GROUPED(8)
#undef LF_GROUPED
            default: return fail(LF_EINVAL, "series length not supported by the grouped scan");
        }
        ce = cudaGetLastError();
    } else if (ea) {
        const int g3 = sm_count();                // launch_scan_ea sizes the grid to the variant's residency
        const int8_t* qc8 = ss->q8 ? ss->qc8.as<int8_t>() : nullptr;
        const float4* qm8 = ss->q8 ? ss->qm8.as<float4>() : nullptr;
        switch (nch) {
            case 1: ce = launch_scan_ea<1>(s, idx, ss->d_q, qc8, qm8, g3, st); break;
            case 2: ce = launch_scan_ea<2>(s, idx, ss->d_q, qc8, qm8, g3, st); break;
            case 3: ce = launch_scan_ea<3>(s, idx, ss->d_q, qc8, qm8, g3, st); break;
            case 4: ce = launch_scan_ea<4>(s, idx, ss->d_q, qc8, qm8, g3, st); break;
            case 5: ce = launch_scan_ea<5>(s, idx, ss->d_q, qc8, qm8, g3, st); break;
            case 6: ce = launch_scan_ea<6>(s, idx, ss->d_q, qc8, qm8, g3, st); break;
            case 7: ce = launch_scan_ea<7>(s, idx, ss->d_q, qc8, qm8, g3, st); break;
            default: ce = launch_scan_ea<8>(s, idx, ss->d_q, qc8, qm8, g3, st); break;
        }
    } else if ((idx.m & 3) != 0 || m4 <= 32) ce = launch_scan<1>(s, idx, ss->d_q, grid, st);
    else if (m4 <= 64) ce = launch_scan<2>(s, idx, ss->d_q, grid, st);
    else if (m4 <= 128) ce = launch_scan<4>(s, idx, ss->d_q, grid, st);
    else if (m4 <= 256) ce = launch_scan<8>(s, idx, ss->d_q, grid, st);
    else return fail(LF_EINVAL, "series length > 1024 not supported");
    if (ce != cudaSuccess) return fail(LF_ECUDA, cudaGetErrorString(ce));
    if (ss->prof) cudaEventRecord(ev[2], st);
    merge_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(s);
    LF_CUDA(cudaGetLastError());
    if (ss->prof) cudaEventRecord(ev[3], st);
    ss->kernels += 5;
    std::swap(s.top_d, s.top_d_out);
    std::swap(s.top_i, s.top_i_out);
    std::swap(s.top_n, s.top_n_out);
    if (d_bsf_out) {
        bsf_out_kernel<<<(unsigned)((Q + 255) / 256), 256, 0, st>>>(s, d_bsf_out);
        LF_CUDA(cudaGetLastError());
        ++ss->kernels;
    }
    LF_CUDA(cudaMemcpyAsync(ss->h_active + 4 * slot, counts, sizeof(int) * 3, cudaMemcpyDeviceToHost, st));
    LF_CUDA(cudaEventRecord(ss->done_ev[slot], st));
    ++ss->round;
    return LF_OK;
}

// Wait for the oldest enqueued round's counts, run the host-decided follow-ups
// (lazy prediction pass, order refill) and accumulate its profile.
static int session_harvest(lf_session* ss, int* active_out) {
    RoundState& s = ss->s;
    const lf_index& idx = ss->idx;
    const lf_search_opts& o = ss->opts;
    cudaStream_t st = ss->st;
    const int64_t Q = ss->Q;
    const int r = ss->harvested;
    const int slot = r & 1;
    int* h = ss->h_active + 4 * slot;
    LF_CUDA(cudaEventSynchronize(ss->done_ev[slot]));
    if (ss->lazy && h[0] > 0 && (r == 0 || h[2] > 0)) {
        int rc = predict_step(ss);     // after round 0 every bsf is finite: predict what is reachable
        if (rc) return rc;
    }
    if (h[1] > 0) {                    // some walks reached the end of their sorted prefix
        OrderArgs oa = ss->oa;
        oa.only = s.refill;
        int nk = 0;
        int rc = refill_order(ss->d_q, Q, idx, ss->qsumm.as<double>(), ss->lb.as<double>(), oa, st, &nk);
        if (rc) return rc;
        ss->kernels += nk;
        ss->refills += h[1];
    }
    if (ss->prof) {
        double* p = o.h_profile;
        cudaEvent_t* ev = ss->rev[slot];
        if (r == 0) p[LF_PROF_BOUNDS_MS] = ev_ms(ss->ev[0], ss->ev[1]);
        p[LF_PROF_PLAN_MS] += ev_ms(ev[0], ev[1]);
        p[LF_PROF_SCAN_MS] += ev_ms(ev[1], ev[2]);
        p[LF_PROF_MERGE_MS] += ev_ms(ev[2], ev[3]);
    }
    ++ss->harvested;
    *active_out = h[0];
    return LF_OK;
}

static int session_round(lf_session* ss, const double* d_bound, double* d_bsf_out, int* active_out) {
    int rc = session_enqueue(ss, d_bound, d_bsf_out);
    if (rc) return rc;
    return session_harvest(ss, active_out);
}

static int session_end(lf_session* ss, int64_t* out_ids, double* out_d, int64_t* out_stats) {
    RoundState& s = ss->s;
    cudaStream_t st = ss->st;
    const int64_t n = ss->Q * s.k;
    finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s, out_ids, out_d);
    LF_CUDA(cudaGetLastError());
    ++ss->kernels;
    (void)out_stats;   // counters were accumulated in place (d_stats of lf_search_begin)
    if (ss->prof) {
        double* p = ss->opts.h_profile;
        cudaEventRecord(ss->ev[5], st);
        cudaEventSynchronize(ss->ev[5]);
        p[LF_PROF_ROUNDS] = ss->harvested;
        p[LF_PROF_KERNELS] = (double)ss->kernels;
        p[LF_PROF_TOTAL_MS] = ev_ms(ss->ev[0], ss->ev[5]);
        p[LF_PROF_REFILLS] = (double)ss->refills;
        p[LF_PROF_PREDICT_MS] = ss->predict_ms;
        p[LF_PROF_PAIRS] = (double)ss->pairs;
        p[LF_PROF_PREDICT_STEPS] = (double)ss->predict_steps;
        unsigned long long c[4] = {0, 0, 0, 0};
        cudaMemcpy(c, ss->ea_count.p, sizeof(c), cudaMemcpyDeviceToHost);
        p[LF_PROF_EA_ROWS] = (double)c[0];
        p[LF_PROF_EA_SURVIVORS] = (double)c[1];
        p[LF_PROF_SCAN_STREAM_BYTES] = (double)c[2];
        p[LF_PROF_SCAN_EXACT_BYTES] = (double)c[3];
    }
    return LF_OK;
}

static void session_free(lf_session* ss) {
    if (!ss) return;
    for (auto& e : ss->ev)
        if (e) cudaEventDestroy(e);
    for (int sl = 0; sl < 2; ++sl) {
        if (ss->done_ev[sl]) cudaEventDestroy(ss->done_ev[sl]);
        for (auto& e : ss->rev[sl])
            if (e) cudaEventDestroy(e);
    }
    delete ss;   // Scratch members free their device buffers stream-ordered
}

static int check_args(const lf_index* idx, int64_t Q, const lf_search_opts* opts) {
    LF_REQUIRE(idx != nullptr && opts != nullptr, "NULL argument");
    LF_REQUIRE(Q >= 0, "negative query count");
    LF_REQUIRE(opts->k >= 1 && opts->k <= idx->n_series, "k must be in [1, n]");
    LF_REQUIRE(idx->n_seg >= 1 && idx->n_seg <= LF_MAX_SEG, "bad segment count");
    LF_REQUIRE((opts->d_pred == nullptr && opts->d_pred_f64 == nullptr && opts->d_W1T == nullptr) ||
                   (opts->d_offset != nullptr && idx->d_leaf_filter != nullptr),
               "filter predictions need offsets and a leaf->filter map");
    LF_REQUIRE(opts->d_W1T == nullptr || opts->d_pred != nullptr || opts->d_pred_f64 != nullptr ||
                   (opts->d_b1 != nullptr && opts->d_W2 != nullptr && opts->d_b2 != nullptr && idx->m % 32 == 0 &&
                    idx->m >= 32 && idx->m <= 256 && opts->n_filters >= 1),
               "lazy filter inference needs W1T, b1, W2, b2 and m in {32, 64, ..., 256}");
    LF_REQUIRE(opts->sequential || opts->max_round_leaves >= 1, "max_round_leaves must be >= 1");
    return LF_OK;
}

}  // namespace lf

extern "C" {

lf_session* lf_search_begin(const lf_index* idx, const float* d_queries, int64_t Q,
                            const lf_search_opts* opts, const lf_trace* trace, int64_t* d_stats,
                            void* stream) {
    if (lf::check_args(idx, Q, opts) != LF_OK) return nullptr;
    if (Q < 1) { lf::fail(LF_EINVAL, "empty query batch"); return nullptr; }
    auto* ss = new lf_session();
    ss->idx = *idx;
    ss->opts = *opts;
    ss->opts.want_trace = (opts->want_trace && trace != nullptr) ? 1 : 0;
    if (ss->opts.want_trace) ss->tr = *trace;
    ss->st = lf::as_stream(stream);
    ss->Q = Q;
    ss->d_q = d_queries;
    ss->s.stats = reinterpret_cast<long long*>(d_stats);
    if (lf::session_begin(ss) != LF_OK) {
        lf::session_free(ss);
        return nullptr;
    }
    return ss;
}

int lf_search_round(lf_session* ss, const double* d_bound, double* d_bsf_out, int32_t* h_active) {
    LF_REQUIRE(ss != nullptr && h_active != nullptr, "NULL argument");
    return lf::session_round(ss, d_bound, d_bsf_out, h_active);
}

int lf_search_end(lf_session* ss, int64_t* d_out_ids, double* d_out_dists) {
    LF_REQUIRE(ss != nullptr, "NULL session");
    int rc = lf::session_end(ss, d_out_ids, d_out_dists, nullptr);
    return rc;
}

void lf_search_free(lf_session* ss) { lf::session_free(ss); }

int lf_search(const lf_index* idx, const float* d_queries, int64_t Q, const lf_search_opts* opts,
              int64_t* d_out_ids, double* d_out_dists, int64_t* d_out_stats, const lf_trace* trace,
              void* stream) {
    int rc = lf::check_args(idx, Q, opts);
    if (rc) return rc;
    if (Q == 0) return LF_OK;
    auto* ss = new lf_session();
    ss->idx = *idx;
    ss->opts = *opts;
    ss->opts.want_trace = (opts->want_trace && trace != nullptr) ? 1 : 0;
    if (ss->opts.want_trace) ss->tr = *trace;
    ss->st = lf::as_stream(stream);
    ss->Q = Q;
    ss->d_q = d_queries;
    ss->s.stats = reinterpret_cast<long long*>(d_out_stats);
    rc = lf::session_begin(ss);
    if (rc) {
        lf::session_free(ss);
        return rc;
    }
    int active = 0;
    if (ss->lazy || lf::prefix_orders()) {
        do {   // host decisions after every round (prediction passes, refills): no pipelining
            rc = lf_search_round(ss, nullptr, nullptr, &active);
            if (rc) break;
        } while (active > 0);
    } else {
        // one round in flight ahead of the count read-back: the host never idles the GPU
        // between rounds; a round enqueued after the last active one finds every query done
        // and changes nothing
        rc = lf::session_enqueue(ss, nullptr, nullptr);
        while (rc == LF_OK) {
            rc = lf::session_enqueue(ss, nullptr, nullptr);
            if (rc) break;
            rc = lf::session_harvest(ss, &active);
            if (rc || active == 0) break;
        }
    }
    if (rc == LF_OK) rc = lf_search_end(ss, d_out_ids, d_out_dists);
    lf_search_free(ss);
    return rc;
}

}  // extern "C"
