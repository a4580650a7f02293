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
#include "round.cuh"
#include "tc.cuh"

namespace lf {

// Warp-parallel plan: one warp per query evaluates 32 consecutive visit-order
// entries at a time.  Within a round every decision uses the round-start bsf,
// so the entries are independent; ballots locate the first break (lb > bsf*f)
// and the R-th selected leaf, and prefix counts place selections and trace
// entries in visit order.  Counters, selections and traces are identical to a
// serial walk of the same entries (tree.py:256-297 with the round-start bsf).
// k = 1 with the entry tail's (distance, id) pairs: fold the query's tasks of the round
// just scanned into its best (warp per query, eight pairs in flight per lane).  (Folding
// them in the next round's plan kernel instead, to save the merge launch of every graph
// round >= 1: 1.424 vs 1.427 ms per batch -- not kept.)
__device__ __forceinline__ void merge_pairs_k1(const RoundState& s, int64_t q, int lane) {
    if (s.n_sel[q] == 0) return;
    const int tn = s.top_n[q];
    double bd = tn > 0 ? s.top_d[q] : kInf;
    long long bi = tn > 0 ? s.top_i[q] : LLONG_MAX;
    const long long c0 = s.chunk_off[q], nc = s.chunk_cnt[q];
    const ulonglong2* cp = reinterpret_cast<const ulonglong2*>(s.cand16) + c0;
    for (long long i0 = lane; i0 < nc; i0 += 256) {
        ulonglong2 c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long i = i0 + 32 * u;
            c[u] = i < nc ? cp[i] : make_ulonglong2(0ull, ~0ull);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long id = (long long)c[u].y;
            const double d = __longlong_as_double((long long)c[u].x);
            if (id >= 0 && pair_less(d, id, bd, bi)) { bd = d; bi = id; }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double xd = __shfl_xor_sync(0xffffffffu, bd, o);
        const long long xi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (pair_less(xd, xi, bd, bi)) { bd = xd; bi = xi; }
    }
    if (lane == 0 && bi != LLONG_MAX) {
        s.top_d[q] = bd;
        s.top_i[q] = bi;
        s.top_n[q] = 1;
    }
    __syncwarp();
}

#ifndef LF_PLAN_PF
#define LF_PLAN_PF 8
#endif
constexpr int PLAN_PF = LF_PLAN_PF;
__global__ void plan_warp_kernel(RoundState s, lf_index idx) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0 && s.pq_n != nullptr) *s.pq_n = 0;   // the scan's entry counter
    if (q >= s.Q) return;
    const unsigned below = (1u << lane) - 1u;
    const int Lr = s.n_leaves;                 // records per query: the leaf slots
    const int R = s.d_round == nullptr ? s.R
                  : s.seq ? 1 : (int)min((long long)s.Rcap, 1ll << min(*s.d_round * s.growth, 30));
    int* pre = s.sel_pre + q * (s.Rcap + 1);
    int ns = 0, nch = 0;
    if (!s.done[q]) {
        const double bsf = round_bsf(s, q);
        const double thr = bsf * s.f;
        const int* ord = s.order + q * Lr;       // node ids (traces only)
        const double* lbs = s.lbs + q * Lr;
        const double* gps = s.gap + q * Lr;
        const int* lrec = s.leafo + q * Lr;
        const double* adj = s.adj + q * Lr;
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
        auto load = [&](int at, double& l_, double& g_, int& r_, double& a_) {
            const int k = at + lane;
            l_ = k < len ? lbs[k] : kInf;
            g_ = k < len ? gps[k] : 0.0;
            r_ = k < len ? lrec[k] : -1;
            a_ = k < len ? adj[k] : 0.0;
        };
        // L2 prefetch of the records PLAN_PF batches ahead (11 lanes: the <= 3 lines of each
        // fp64 array and <= 2 of the records per 32 entries): a walk through a long
        // filter-pruned stretch otherwise waits on DRAM every batch (measured per walk
        // with %globaltimer: 0.63 -> 0.43 us per batch; what remains is the batch's own
        // instruction latency at one warp per scheduler -- a shared-memory cp.async ring
        // or a second register batch in flight change nothing)
        auto prefetch = [&](int at) {
            if (lane < 11 && at < len) {
                const char* p = lane < 3   ? reinterpret_cast<const char*>(lbs + at) + min(lane * 128, 255)
                                : lane < 6 ? reinterpret_cast<const char*>(gps + at) + min((lane - 3) * 128, 255)
                                : lane < 9 ? reinterpret_cast<const char*>(adj + at) + min((lane - 6) * 128, 255)
                                           : reinterpret_cast<const char*>(lrec + at) + (lane - 9) * 127;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
            }
        };
#pragma unroll
        for (int j = 1; j <= PLAN_PF; ++j) prefetch(cur + 32 * j);
        double lb_c, gp_c, ad_c;
        int rec_c;
        load(cur, lb_c, gp_c, rec_c, ad_c);
        while (!fin && cur < len) {
            double lb_n, gp_n, ad_n;
            int rec_n;
            load(cur + 32, lb_n, gp_n, rec_n, ad_n);
            prefetch(cur + 32 * (PLAN_PF + 1));
            const int i = cur + lane;
            const bool valid = i < len;
            const int node = (valid && s.want_trace) ? ord[i] : -1;
            const double lb = lb_c;
            const int rec = rec_c;
            const int leaf = rec >= 0 ? (rec & LF_REC_LEAF) : -1;
            // the walk stops before this leaf if a non-leaf node popped since the previous
            // leaf has lb > bsf * f (gap, uncounted), or at this leaf if its own bound does
            const bool gbrk = valid && gp_c > thr;
            const bool brk = valid && (gbrk || lb > thr);
            const unsigned bmask = __ballot_sync(0xffffffffu, brk);
            const int first_brk = bmask ? __ffs(bmask) - 1 : 32;
            const bool visit = valid && leaf >= 0 && lane < first_brk;
            const int fs = (visit && (rec & LF_REC_HASF)) ? 0 : -1;
            const bool fpr = fs >= 0 && ad_c > thr;        // (pred - offset) > bsf * f, tree.py:282
            const bool scan = visit && !fpr;
            const unsigned smask = __ballot_sync(0xffffffffu, scan);
            if ((bmask | smask) == 0u && !s.want_trace && cur + 32 < len) {
                // a whole batch of filter-pruned leaves (the long stretches of a walk under
                // a tight bound): counters only, no selection bookkeeping.  No break and no
                // scan: every visited leaf has a filter and was pruned by it
                const int nv = __popc(__ballot_sync(0xffffffffu, visit));
                c_vis += nv;
                c_inf += nv;
                c_fp += nv;
                cur += 32;
                lb_c = lb_n; gp_c = gp_n; rec_c = rec_n; ad_c = ad_n;
                continue;
            }
            const int need = R - ns;
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
            const unsigned sm_in = __ballot_sync(0xffffffffu, s_in);
            const unsigned vm_in = __ballot_sync(0xffffffffu, v_in);
            if (sm_in) {            // (a batch without a selected leaf skips the chunk scan)
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
                if (s_in) {
                    const int slot = ns + __popc(sm_in & below);
                    s.sel_leaf[q * s.Rcap + slot] = leaf;
                    pre[slot] = nch + incl - chunks;
                }
                long long rsum = rows;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
                c_rows += rsum;
                nch += __shfl_sync(0xffffffffu, incl, 31);
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
            c_vis += __popc(vm_in);
            c_srch += __popc(sm_in);
            c_inf += __popc(__ballot_sync(0xffffffffu, f_in));
            c_fp += __popc(__ballot_sync(0xffffffffu, p_in));
            tl += __popc(vm_in);
            ns += __popc(sm_in);
            if (quota) {
                cur += end;
                quota_hit = true;
                // the walk's next record already breaks at this round's bound; bsf only
                // shrinks, so the next round would stop there with the same counters:
                // stop now (saves the round that only finds every walk done)
                if (!s.want_trace && cur < len) {
                    const double plb = end < 32 ? __shfl_sync(0xffffffffu, lb_c, end) : __shfl_sync(0xffffffffu, lb_n, 0);
                    const double pgp = end < 32 ? __shfl_sync(0xffffffffu, gp_c, end) : __shfl_sync(0xffffffffu, gp_n, 0);
                    if (pgp > thr || plb > thr) {
                        if (!(pgp > thr)) {               // a leaf: visited + lb-pruned (tree.py:261-269)
                            c_vis += 1;
                            c_lbp += 1;
                        }
                        fin = true;
                    }
                }
            } else if (first_brk < 32 && first_brk < len - cur) {
                // the break entry: a leaf counts as visited + lb-pruned (tree.py:261-269),
                // an internal node (gap) ends the walk uncounted
                const int bnode = __shfl_sync(0xffffffffu, node, first_brk);
                const bool bgap = __shfl_sync(0xffffffffu, gbrk, first_brk);
                const double blb = __shfl_sync(0xffffffffu, lb, first_brk);
                if (!bgap) {
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
                lb_c = lb_n; gp_c = gp_n; rec_c = rec_n; ad_c = ad_n;
            } else {
                load(cur, lb_c, gp_c, rec_c, ad_c);
            }
        }
        if (cur >= olen) fin = true;
        if (lane == 0) {
            st[0] += c_vis; st[1] += c_srch; st[2] += c_lbp; st[3] += c_fp; st[4] += c_inf; st[5] += c_rows;
            s.cursor[q] = cur;
            if (s.want_trace) s.tr.d_len[q] = tl;
            if (fin) s.done[q] = 1;
            else atomicAdd(s.n_active, 1);
            if (!fin && !quota_hit && cur >= len && len < olen) {   // needs predictions further down
                s.preq[q] = 1;
                atomicAdd(s.n_predict, 1);
            }
        }
    }
    // this query's tasks: a contiguous range claimed from the round's task counter
    // (chunk_off[Q]; ranges of different queries land in any order, each stays
    // contiguous), then one lane per selected leaf writes (query, leaf, chunk) and the
    // chunk's row range, so a scan producer needs no dependent loads
    long long base = 0;
    if (lane == 0) {
        pre[ns] = nch;
        s.n_sel[q] = ns;
        if (nch) base = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(s.chunk_off + s.Q),
                                             (unsigned long long)nch);
        s.chunk_off[q] = base;
        s.chunk_cnt[q] = nch;
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    __syncwarp();                                  // sel_leaf / pre of every lane visible
    for (int j = lane; j < ns; j += 32) {
        const int leaf = s.sel_leaf[q * s.Rcap + j];
        const int c0 = pre[j], n = pre[j + 1] - c0;
        const long long lb = idx.d_leaf_ptr[leaf], le = idx.d_leaf_ptr[leaf + 1];
        for (int c = 0; c < n; ++c) {
            s.tasks[base + c0 + c] = make_int4((int)q, leaf, c, j);
            if (s.task_rows != nullptr) {
                const long long r0 = lb + (long long)c * CH;
                s.task_rows[base + c0 + c] = make_int4((int)(r0 & 0xffffffffLL), (int)(r0 >> 32),
                                                       (int)min((long long)CH, le - r0), (int)q);
            }
        }
    }
}

// Round 0 of a pruned-order search (the visit orders are built after round 0): every
// walk pops its first leaf -- the minimum (lb, node id) over the leaves, from
// lb_tile's per-group minima -- and scans it; bsf is +inf, so nothing is pruned
// and the counters are the reference's for one visited, searched leaf.
__global__ void first_leaf_plan_kernel(RoundState s, lf_index idx, const double* __restrict__ plb,
                                       const int* __restrict__ pnode, int W) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0 && s.pq_n != nullptr) *s.pq_n = 0;   // the scan's entry counter
    if (q >= s.Q) return;
    double bv = kInf;
    int bn = 0x7fffffff;
    for (int w = lane; w < W; w += 32) {
        const int nd = pnode[q * W + w];
        if (nd < 0) continue;
        const double v = plb[q * W + w];
        if (v < bv || (v == bv && nd < bn)) { bv = v; bn = nd; }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, d);
        const int on = __shfl_xor_sync(0xffffffffu, bn, d);
        if (ov < bv || (ov == bv && on < bn)) { bv = ov; bn = on; }
    }
    int* pre = s.sel_pre + q * (s.Rcap + 1);
    if (bn == 0x7fffffff) {                            // no leaf on this shard
        if (lane == 0) {
            s.n_sel[q] = 0;
            pre[0] = 0;
            s.chunk_off[q] = 0;
            s.chunk_cnt[q] = 0;
            s.done[q] = 1;
        }
        return;
    }
    const int leaf = idx.d_node_leaf[bn];
    const long long lb0 = idx.d_leaf_ptr[leaf], le0 = idx.d_leaf_ptr[leaf + 1];
    const int nch = (int)((le0 - lb0 + CH - 1) / CH);
    long long base = 0;
    if (lane == 0) {
        long long* st = s.stats + q * LF_N_STATS;
        st[0] += 1;                                    // visited
        st[1] += 1;                                    // searched
        if (idx.d_leaf_filter != nullptr && s.F > 0 && idx.d_leaf_filter[leaf] >= 0) st[4] += 1;   // inference
        st[5] += le0 - lb0;
        s.cursor[q] = 1;
        atomicAdd(s.n_active, 1);
        s.sel_leaf[q * s.Rcap] = leaf;
        pre[0] = 0;
        pre[1] = nch;
        s.n_sel[q] = 1;
        base = (long long)atomicAdd(reinterpret_cast<unsigned long long*>(s.chunk_off + s.Q), (unsigned long long)nch);
        s.chunk_off[q] = base;
        s.chunk_cnt[q] = nch;
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int c = lane; c < nch; c += 32) {
        s.tasks[base + c] = make_int4((int)q, leaf, c, 0);
        if (s.task_rows != nullptr) {
            const long long r0 = lb0 + (long long)c * CH;
            s.task_rows[base + c] = make_int4((int)(r0 & 0xffffffffLL), (int)(r0 >> 32), (int)min((long long)CH, le0 - r0),
                                              (int)q);
        }
    }
}

// ------------------------------------------------- in-search inference ----
// Round 0 needs no prediction (bsf = +inf: the filter rule never fires).  After it,
// a query with a finite bsf0 can only ever reach the visit-order positions
// [pcount, pend), pend = one past the first position whose bound exceeds bsf0 * f
// (bsf only decreases, so every later break comes no later).  The leaves with a
// filter in that range are a superset of the (query, leaf) pairs whose prediction
// the cascade may evaluate (tree.py:277-286).  One pass predicts them all: pass 1
// counts them per filter, a single-CTA scan turns the counts into filter buckets and
// a 128-pair tile list, pass 2 fills the buckets, and filter_reach_f16 (tcgen05
// kind::f16, the dense kernel's arithmetic, query rows gathered with cp.async)
// writes pred - offset into the records.  On the bench workload that is 0.42M pairs
// instead of the 4.1M of a dense pass.  All on the device: rounds stay pipelined.
// Thread per query: the range of the visit order the walk can still reach.  The
// order is sorted by (lb, node id), so the first position whose bound exceeds
// bsf * f is a binary search; pairs are [pstart, pair_end), and the walk may go up to
// pend = pair_end + 1 (the break entry itself: its bound alone decides).
// Warp per query: a 32-way search (one ballot per step, ~3 dependent loads for 4,096
// records instead of 12).
__global__ void pairs_range_kernel(RoundState s, int* __restrict__ pcount, int* __restrict__ pstart,
                                   int* __restrict__ pair_end, int all, int* __restrict__ fhist, int F) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < F; f += (int64_t)gridDim.x * blockDim.x)
        fhist[f] = 0;                                    // the pass's filter buckets (no memset node)
    if (q >= s.Q) return;
    const int pc = pcount[q];
    const int start = max(pc, s.cursor[q]);              // the walk never goes back
    const double thr = round_bsf(s, q) * s.f;
    const bool want = all || s.preq[q];
    int pe = start, walk = start;
    if (!s.done[q] && thr < kInf && want) {
        const double* lbs = s.lbs + q * s.n_leaves;
        const int len = s.olen[q];
        int lo = start, hi = len;                        // the answer lies in [lo, hi]
        while (hi - lo > 32) {
            const int step = (hi - lo + 31) >> 5;
            const int p = min(lo + (lane + 1) * step - 1, hi - 1);
            const unsigned b = __ballot_sync(0xffffffffu, lbs[p] > thr);
            if (b == 0u) {
                lo = hi;                                 // every probe (the last is hi - 1) <= thr
            } else {
                const int f = __ffs(b) - 1;
                const int nlo = f == 0 ? lo : min(lo + f * step - 1, hi - 1) + 1;
                hi = min(lo + (f + 1) * step - 1, hi - 1);   // lbs[hi] > thr
                lo = nlo;
            }
        }
        const bool gt = lo + lane < hi && lbs[lo + lane] > thr;
        const unsigned b = __ballot_sync(0xffffffffu, gt);
        pe = b ? lo + __ffs(b) - 1 : hi;
        walk = pe < len ? pe + 1 : len;
    }
    if (lane == 0) {
        s.preq[q] = 0;
        pstart[q] = start;
        pair_end[q] = pe;
        pcount[q] = max(pc, walk);
    }
}

// Warp per (query, 256 positions): FILL = 0 counts the filtered leaves of the
// reachable range per filter, FILL = 1 places each (query, position) pair in its
// filter's bucket.
constexpr int PAIR_SPAN = 256;
template <bool FILL>
__global__ void pairs_pos_kernel(int64_t Q, int Lr, const int* __restrict__ pstart, const int* __restrict__ pair_end,
                                 const int* __restrict__ leafo, const int* __restrict__ leaf_filter,
                                 int* __restrict__ cnt, int2* __restrict__ dst, unsigned long long* total,
                                 int stride) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int spans = (Lr + PAIR_SPAN - 1) / PAIR_SPAN;
    const int64_t q = w / spans;
    if (q >= Q) return;
    const int c0 = (int)(w % spans) * PAIR_SPAN;
    const int a = max(pstart[q], c0), b = min(pair_end[q], c0 + PAIR_SPAN);
    if (a >= b) return;
    const int* lrec = leafo + q * Lr;
    int n = 0;
    for (int k = a + lane; k < b; k += 32) {
        const int rec = lrec[k];
        if (rec >= 0 && (rec & LF_REC_HASF)) {
            const int f = leaf_filter[rec & LF_REC_LEAF];
            if (FILL) dst[(int64_t)f * stride + atomicAdd(&cnt[f], 1)] = make_int2((int)q, k);
            else atomicAdd(&cnt[f], 1);
            ++n;
        }
    }
    if (total) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
        if (lane == 0 && n) atomicAdd(total, (unsigned long long)n);
    }
}

// Filter buckets (exclusive scan of the per-filter counts) and the tile list
// (filter, first pair, pairs <= 128) in one CTA: each thread owns PT consecutive
// filters, one block-wide scan of (pairs, tiles) per thread.
constexpr int PT_THREADS = 1024, PT_ITEMS = 8;
__global__ void __launch_bounds__(PT_THREADS) pair_tiles_kernel(const int* __restrict__ fhist, int F,
                                                                int* __restrict__ fcur, int4* __restrict__ tiles,
                                                                int* __restrict__ ntiles, int stride) {
    using Scan = cub::BlockScan<int2, PT_THREADS>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int2 carry;
    if (threadIdx.x == 0) carry = make_int2(0, 0);
    __syncthreads();
    struct Add2 {
        __device__ int2 operator()(const int2& a, const int2& b) const { return make_int2(a.x + b.x, a.y + b.y); }
    };
    for (int base = 0; base < F; base += PT_THREADS * PT_ITEMS) {
        int h[PT_ITEMS];
        int2 mine = make_int2(0, 0);
#pragma unroll
        for (int i = 0; i < PT_ITEMS; ++i) {
            const int f = base + threadIdx.x * PT_ITEMS + i;
            h[i] = f < F ? fhist[f] : 0;
            mine.x += h[i];
            mine.y += (h[i] + 127) / 128;
        }
        int2 excl, total;
        Scan(tmp).ExclusiveScan(mine, excl, make_int2(0, 0), Add2(), total);
        int p0 = carry.x + excl.x, t0 = carry.y + excl.y;
#pragma unroll
        for (int i = 0; i < PT_ITEMS; ++i) {
            const int f = base + threadIdx.x * PT_ITEMS + i;
            if (f < F) {
                // stride > 0: the buckets were filled in place, bucket f at f * stride
                const int b0 = stride > 0 ? f * stride : p0;
                if (stride == 0) fcur[f] = p0;
                for (int t = 0; t * 128 < h[i]; ++t) tiles[t0 + t] = make_int4(f, b0 + 128 * t, min(128, h[i] - 128 * t), 0);
            }
            p0 += h[i];
            t0 += (h[i] + 127) / 128;
        }
        __syncthreads();
        if (threadIdx.x == 0) carry = make_int2(carry.x + total.x, carry.y + total.y);
        __syncthreads();
    }
    if (threadIdx.x == 0) *ntiles = carry.y;
}

int pair_tiles(const int* d_hist, int F, int* d_fcur, int4* d_tiles, int* d_ntiles, cudaStream_t st, int stride) {
    pair_tiles_kernel<<<1, PT_THREADS, 0, st>>>(d_hist, F, d_fcur, d_tiles, d_ntiles, stride);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

// --------------------------------------------------------------- merge ----
// One warp per query: k smallest (d, id) among the running top-k and this
// round's candidates (each series is scanned at most once per query, so all
// (d, id) pairs are distinct and repeated "next larger than the last pick"
// selection is exact).  Reads top_* (round-start state), writes top_*_out.
constexpr int MERGE_KMAX = 16;                 // k up to this: register top-k per lane
__global__ void merge_kernel(RoundState s) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (blockIdx.x == 0 && threadIdx.x == 0) {     // the next round's task counter and counts
        s.chunk_off[s.Q] = 0;
        if (s.zero_counts != nullptr)
            for (int i = 0; i < 3; ++i) s.zero_counts[i] = 0;
    }
    if (q >= s.Q) return;
    const int ns = s.n_sel[q];
    const double* td = s.top_d + q * s.k;
    const long long* ti = s.top_i + q * s.k;
    double* od = s.top_d_out + q * s.k;
    long long* oi = s.top_i_out + q * s.k;
    const int tn = s.top_n[q];
    if (ns == 0) return;                       // nothing scanned: the top-k stands
    const long long c0 = s.chunk_off[q], c1 = c0 + s.chunk_cnt[q];
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

    if (s.k == 1 && s.cand16 != nullptr) {
        merge_pairs_k1(s, q, lane);
        return;
    }
    if (s.k == 1) {                            // one pass, eight candidates' loads in flight per lane
        double bd = tn > 0 ? td[0] : kInf;
        long long bi = tn > 0 ? ti[0] : LLONG_MAX;
        for (long long i0 = lane; i0 < nc; i0 += 256) {
            double dv[8];
            long long iv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const long long i = i0 + 32 * u;
                iv[u] = i < nc ? ci[i] : -1;
                dv[u] = i < nc ? cd[i] : kInf;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (iv[u] >= 0 && pair_less(dv[u], iv[u], bd, bi)) { bd = dv[u]; bi = iv[u]; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double xd = __shfl_xor_sync(0xffffffffu, bd, o);
            const long long xi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (pair_less(xd, xi, bd, bi)) { bd = xd; bi = xi; }
        }
        if (lane == 0 && bi != LLONG_MAX) {
            s.top_d[q] = bd;
            s.top_i[q] = bi;
            s.top_n[q] = 1;
        }
        return;
    }
    if (s.k <= MERGE_KMAX) {
        // one pass: every lane keeps the k best of its strided share in registers
        // (sorted; candidates and the running top-k alike), then k warp-wide pops
        double ld[MERGE_KMAX];
        long long li[MERGE_KMAX];
#pragma unroll
        for (int j = 0; j < MERGE_KMAX; ++j) { ld[j] = kInf; li[j] = LLONG_MAX; }
        const long long total = (long long)tn + nc;
        double kd = kInf;                                  // the k-th kept (ld[k - 1], kept in registers)
        long long ki = LLONG_MAX;
        for (long long i = lane; i < total; i += 32) {
            const bool top = i < tn;
            const long long id = top ? ti[i] : ci[i - tn];
            if (id < 0) continue;
            const double d = top ? td[i] : cd[i - tn];
            if (!pair_less(d, id, kd, ki)) continue;
            // insert (d, id): the sorted list's "greater than (d, id)" flags are monotone,
            // so slot j takes slot j-1's entry or (d, id) -- static indices only
            bool gt[MERGE_KMAX];
#pragma unroll
            for (int j = 0; j < MERGE_KMAX; ++j) gt[j] = j < s.k && pair_less(d, id, ld[j], li[j]);
#pragma unroll
            for (int j = MERGE_KMAX - 1; j > 0; --j)
                if (gt[j]) {
                    ld[j] = gt[j - 1] ? ld[j - 1] : d;
                    li[j] = gt[j - 1] ? li[j - 1] : id;
                }
            if (gt[0]) { ld[0] = d; li[0] = id; }
            kd = -1.0;                                     // the largest of the first k (sorted: ld[k-1])
            ki = -1;
#pragma unroll
            for (int j = 0; j < MERGE_KMAX; ++j)
                if (j < s.k && pair_less(kd, ki, ld[j], li[j])) { kd = ld[j]; ki = li[j]; }
        }
        int filled = 0;
        for (int sel = 0; sel < s.k; ++sel) {
            double bd = ld[0];
            long long bi = li[0];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double xd = __shfl_xor_sync(0xffffffffu, bd, o);
                const long long xi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (pair_less(xd, xi, bd, bi)) { bd = xd; bi = xi; }
            }
            if (bi == LLONG_MAX) continue;             // (every later pop is empty too)
            if (lane == 0) { od[sel] = bd; oi[sel] = bi; }
            ++filled;
            if (li[0] == bi && ld[0] == bd) {          // the owner pops its head
#pragma unroll
                for (int j = 0; j + 1 < MERGE_KMAX; ++j) { ld[j] = ld[j + 1]; li[j] = li[j + 1]; }
                ld[MERGE_KMAX - 1] = kInf;
                li[MERGE_KMAX - 1] = LLONG_MAX;
            }
        }
        __syncwarp();
        double* wd = s.top_d + q * s.k;
        long long* wi = s.top_i + q * s.k;
        for (int i = lane; i < filled; i += 32) { wd[i] = od[i]; wi[i] = oi[i]; }
        if (lane == 0) s.top_n[q] = filled;
        return;
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
    // the new top-k back into the running state (every lane has finished reading it)
    __syncwarp();
    double* wd = s.top_d + q * s.k;
    long long* wi = s.top_i + q * s.k;
    for (int i = lane; i < filled; i += 32) { wd[i] = od[i]; wi[i] = oi[i]; }
    if (lane == 0) s.top_n[q] = filled;
}

__global__ void init_state_kernel(RoundState s) {
    int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q == 0) {
        s.chunk_off[s.Q] = 0;
        if (s.ea_count != nullptr)
            for (int i = 0; i < 4; ++i) s.ea_count[i] = 0ull;
        if (s.cnt_all != nullptr)
            for (int i = 0; i < 8; ++i) s.cnt_all[i] = 0;
        if (s.rctr != nullptr) *s.rctr = 0;
        if (s.ptotal != nullptr) *s.ptotal = 0ull;
        if (s.pq_n != nullptr) *s.pq_n = 0;
    }
    if (q >= s.Q) return;
    s.cursor[q] = 0;
    s.done[q] = 0;
    s.top_n[q] = 0;
    if (s.lazy) {
        s.pcount[q] = 0;
        s.preq[q] = 0;
    }
    if (s.qbest != nullptr) s.qbest[q] = 0x7f7f7f7fu;          // 3.4e38: above any distance
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

// Scan variant: LF_SCAN_VARIANT unset / pq (default: the full-length int8 shadow in
// round 0, then the projected shadow -- 48 instead of 272 bytes per row -- wherever the
// index carries one) | q8 (int8 shadow only) | full (fp64 over the fp32 rows).
// Leaves per query per round grow as 2^(round * g): LF_ROUND_GROWTH_LOG2 = g (default 2:
// 1, 4, 16, ... up to max_round_leaves).  Measured on the bench workload (1K queries,
// tools/growth_probe.py): x2 / cap 64 -> 9 rounds, 3.47 ms; x4 / cap 256 -> 5 rounds,
// 3.12 ms, 2% more series scanned -- fewer rounds of fixed per-round latency.
static int round_growth_log2() {
    const char* e = getenv("LF_ROUND_GROWTH_LOG2");
    const int g = e ? atoi(e) : 2;
    return g >= 1 && g <= 6 ? g : 2;
}

static bool round0_seeded() {
    const char* e = getenv("LF_SCAN_ROUND0");
    return !(e && strcmp(e, "q8") == 0);
}

static int scan_variant() {
    const char* e = getenv("LF_SCAN_VARIANT");
    if (!e || e[0] == 0 || strcmp(e, "pq") == 0) return 8;   // projected stage when the shadow exists
    if (strcmp(e, "q8") == 0) return 9;            // int8 shadow only
    if (strcmp(e, "full") == 0) return 0;
    return 8;                                      // default: int8-bounded scan when the shadow exists
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
    lf::Scratch qsumm, lb, lbs, gap, order, cursor, done, topd, topi, topn, topd2, topi2, topn2, sel_leaf,
        sel_trace, sel_pre, n_sel, chunk_off, chunk_cnt, cand_d, cand_i, task_min, n_active, tasks, ea_count, qc8, qm8,
        leafo, adj, olen, pcount, pstart, pend, preq, fhist, fcur, ntiles, ptotal, pdst, ptiles, xh, xexp, round_ctr;
    lf::OrderArgs oa{};
    bool pruned = false;             // visit orders built after round 0, only up to bsf0 * f
    lf::Scratch orng, plb, pnode;    // pruned: leaf-bound ranges, per-group first-leaf candidates
    int W = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> oev;   // profiling: the order phase
    bool lazy = false;               // in-search filter inference (opts.d_W1T_h instead of predictions)
    int predict_steps = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pev;   // profiling: per prediction pass
    bool q8 = false;                 // int8-bounded scan (query codes quantised once in begin)
    bool pq = false;                 // two-stage scan over the projected shadow (d_Xp)
    lf::Scratch qcp, qmp, pq_cnt, pq_trows, pq_oent, pq_on, pq_obase, pq_wrows, pq_wdist, pq_lo8, pq_thr, pq_qbest, pq_xlist, pq_xn,
        pq_c16;
    int pq_cap = lf::PQ_OVER_CAP;    // survivor entry capacity (LF_PQ_OVER_CAP: tests of the full-list path)
    int64_t max_tasks = 1;
    int* h_active = nullptr;         // pinned [2 slots][4]: active, -, predict requests
    int round = 0;                   // rounds enqueued
    int harvested = 0;               // rounds whose counts were read back
    cudaEvent_t rev[2][4] = {};      // per slot: plan start, scan start, merge start, merge end
    cudaEvent_t done_ev[2] = {};     // per slot: counts copied back
    long long kernels = 0;
    cudaEvent_t ev[6] = {};
    bool prof = false;
    cudaStream_t st2 = nullptr;      // prologue branch: query codes, concurrent with the bounds
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    // k = 1 seeded round 0: the pruned visit orders are cut at the seed minima (qbest) and
    // built on st2 right after round 0's streaming scan, concurrent with its int8 stage,
    // tail and merge (graph plans); joined before the prediction pass
    bool order_seed = false;
    bool capturing = false;          // plan_capture: the body's rounds share one count slot
    cudaEvent_t scan0_ev = nullptr, order_ev = nullptr;
};

namespace lf {

// Scratch of one search session, sized once for (index, Q, opts); a search plan keeps
// it across calls (lf_search_plan_*), lf_search / lf_search_begin allocate per call.
// the in-search filter operands' width: the pack's (zero-padded) dimension, or m
static int filter_width(const lf_index& idx, const lf_search_opts& o) { return o.filter_m > 0 ? o.filter_m : idx.m; }

static int session_alloc(lf_session* ss) {
    const lf_index& idx = ss->idx;
    const lf_search_opts& o = ss->opts;
    cudaStream_t st = ss->st;
    const int64_t Q = ss->Q;
    const int Nn = idx.n_nodes, L = std::max(1, idx.n_leaves);
    RoundState& s = ss->s;
    s.Q = Q;
    s.k = o.k;
    s.kc = std::min(o.k, CH);
    s.f = o.bsf_factor;
    s.Rcap = o.sequential ? 1 : std::max(1, std::min(o.max_round_leaves, std::max(1, idx.n_leaves)));
    s.seq = o.sequential ? 1 : 0;
    s.growth = round_growth_log2();
    s.d_round = nullptr;
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
    ss->max_tasks = max_tasks;
    LF_CUDA(ss->qsumm.alloc(sizeof(double) * Q * idx.n_seg * (idx.d_sd_min != nullptr ? 2 : 1), st));
    LF_CUDA(ss->lb.alloc(sizeof(double) * Q * Nn, st));        // node bounds (L2-resident at 1K x 8K)
    LF_CUDA(ss->lbs.alloc(sizeof(double) * Q * L, st));        // leaf records in visit order
    LF_CUDA(ss->gap.alloc(sizeof(double) * Q * L, st));
    if (s.want_trace) LF_CUDA(ss->order.alloc(sizeof(int) * Q * L, st));
    LF_CUDA(ss->leafo.alloc(sizeof(int) * Q * L, st));
    LF_CUDA(ss->adj.alloc(sizeof(double) * Q * L, st));
    // NaN once: with in-search inference the visit orders leave adj unset (the pass fills
    // every entry a walk can reach), so nothing ever reads uninitialised memory
    LF_CUDA(cudaMemsetAsync(ss->adj.p, 0xff, sizeof(double) * Q * L, st));
    LF_CUDA(ss->olen.alloc(sizeof(int) * Q, st));
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
    LF_CUDA(ss->chunk_cnt.alloc(sizeof(int) * Q, st));
    LF_CUDA(ss->cand_d.alloc(sizeof(double) * max_tasks * s.kc, st));
    LF_CUDA(ss->cand_i.alloc(sizeof(long long) * max_tasks * s.kc, st));
    LF_CUDA(ss->task_min.alloc(sizeof(double) * (s.want_trace ? max_tasks : 1), st));
    LF_CUDA(ss->n_active.alloc(sizeof(int) * 8, st));   // [2 slots][active, refill, predict requests, -]
    LF_CUDA(ss->round_ctr.alloc(sizeof(int), st));
    LF_CUDA(cudaStreamCreateWithFlags(&ss->st2, cudaStreamNonBlocking));
    LF_CUDA(cudaEventCreateWithFlags(&ss->fork_ev, cudaEventDisableTiming));
    LF_CUDA(cudaEventCreateWithFlags(&ss->join_ev, cudaEventDisableTiming));
    LF_CUDA(cudaEventCreateWithFlags(&ss->scan0_ev, cudaEventDisableTiming));
    LF_CUDA(cudaEventCreateWithFlags(&ss->order_ev, cudaEventDisableTiming));
    for (int sl = 0; sl < 2; ++sl) {
        LF_CUDA(cudaEventCreateWithFlags(&ss->done_ev[sl], cudaEventDisableTiming));
        if (o.h_profile)
            for (auto& e : ss->rev[sl]) LF_CUDA(cudaEventCreate(&e));
    }
    ss->lazy = o.d_pred == nullptr && o.d_pred_f64 == nullptr && o.d_W1T_h != nullptr;
    if (ss->lazy) {
        const int F = std::max(1, o.n_filters);
        LF_CUDA(ss->pcount.alloc(sizeof(int) * Q, st));
        LF_CUDA(ss->pstart.alloc(sizeof(int) * Q, st));
        LF_CUDA(ss->pend.alloc(sizeof(int) * Q, st));
        LF_CUDA(ss->preq.alloc(sizeof(int) * Q, st));
        LF_CUDA(ss->fhist.alloc(sizeof(int) * F, st));
        LF_CUDA(ss->fcur.alloc(sizeof(int) * F, st));
        LF_CUDA(ss->ntiles.alloc(sizeof(int), st));
        LF_CUDA(ss->ptotal.alloc(sizeof(unsigned long long), st));
        const int64_t max_pairs = Q * (int64_t)L;     // every (query, leaf) pair, worst case
        LF_CUDA(ss->pdst.alloc(sizeof(int2) * max_pairs, st));
        LF_CUDA(ss->ptiles.alloc(sizeof(int4) * (max_pairs / 128 + F + 1), st));
        LF_CUDA(ss->xh.alloc(sizeof(__half) * Q * filter_width(idx, o), st));
        LF_CUDA(ss->xexp.alloc(sizeof(int) * Q, st));
    }
    LF_CUDA(ss->tasks.alloc(sizeof(int4) * max_tasks, st));
    LF_CUDA(ss->ea_count.alloc(sizeof(unsigned long long) * 4, st));
    {   // one pinned word per host thread (freed with the thread); a round reads it right after its own sync
        struct Pinned {
            int* p = nullptr;
            ~Pinned() {
                if (p) cudaFreeHost(p);
            }
        };
        static thread_local Pinned pinned;
        if (pinned.p == nullptr) LF_CUDA(cudaMallocHost(&pinned.p, sizeof(int) * 8));
        ss->h_active = pinned.p;
    }
    // pruned visit orders: with the reference's bsf_factor 1, no traces, and a tree the
    // single-CTA order kernel takes (LF_PRUNED_ORDER=0 builds full orders first)
    {
        const char* e = getenv("LF_PRUNED_ORDER");
        ss->pruned = !s.want_trace && o.bsf_factor == 1.0 && fused_order_ok(idx, Q) && !(e && strcmp(e, "0") == 0);
    }
    if (ss->pruned) {
        ss->W = (Nn + 31) / 32;
        LF_CUDA(ss->orng.alloc(sizeof(unsigned) * 2 * Q, st));
        LF_CUDA(ss->plb.alloc(sizeof(double) * Q * ss->W, st));
        LF_CUDA(ss->pnode.alloc(sizeof(int) * Q * ss->W, st));
    }
    OrderArgs& oa = ss->oa;
    oa.prune = ss->pruned ? 1 : 0;
    oa.top_d = ss->topd.as<double>();
    oa.top_n = ss->topn.as<int>();
    oa.k = o.k;
    oa.f = o.bsf_factor;
    oa.bound = nullptr;
    oa.seed = nullptr;
    oa.lbs = ss->lbs.as<double>();
    oa.gap = ss->gap.as<double>();
    oa.order = s.want_trace ? ss->order.as<int>() : nullptr;
    oa.leafo = ss->leafo.as<int>();
    oa.adj = ss->adj.as<double>();
    oa.olen = ss->olen.as<int>();
    oa.pred = o.d_pred;
    oa.pred64 = o.d_pred_f64;
    oa.offset = o.d_offset;
    oa.F = o.n_filters;
    oa.lazy = ss->lazy ? 1 : 0;
    s.order = oa.order;
    s.lbs = ss->lbs.as<double>();
    s.gap = ss->gap.as<double>();
    s.leafo = ss->leafo.as<int>();
    s.adj = ss->adj.as<double>();
    s.olen = ss->olen.as<int>();
    s.n_predict = ss->n_active.as<int>() + 2;
    s.lazy = ss->lazy ? 1 : 0;
    s.pcount = ss->lazy ? ss->pcount.as<int>() : nullptr;
    s.preq = ss->lazy ? ss->preq.as<int>() : nullptr;
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
    s.chunk_cnt = ss->chunk_cnt.as<int>();
    s.cand_d = ss->cand_d.as<double>();
    s.cand_i = ss->cand_i.as<long long>();
    s.task_min = ss->task_min.as<double>();
    s.n_active = ss->n_active.as<int>();
    s.tasks = ss->tasks.as<int4>();
    s.ea_count = o.h_profile ? ss->ea_count.as<unsigned long long>() : nullptr;
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
        if (const char* e = getenv("LF_PQ_OVER_CAP")) ss->pq_cap = std::max(1, std::min(PQ_OVER_CAP, atoi(e)));
        LF_CUDA(ss->pq_oent.alloc(sizeof(int4) * ss->pq_cap, st));
        LF_CUDA(ss->pq_on.alloc(sizeof(int), st));
        LF_CUDA(ss->pq_obase.alloc(sizeof(int) * max_tasks, st));
        LF_CUDA(ss->pq_wrows.alloc(sizeof(unsigned short) * CH * pq_scan_warps(), st));
        LF_CUDA(ss->pq_wdist.alloc(sizeof(double) * CH * pq_scan_warps(), st));
        LF_CUDA(ss->pq_lo8.alloc(sizeof(float) * ss->pq_cap, st));
        LF_CUDA(ss->pq_thr.alloc(sizeof(unsigned) * max_tasks, st));
        LF_CUDA(ss->pq_qbest.alloc(sizeof(unsigned) * Q, st));
        if (s.k == 1 && ss->q8) {
            LF_CUDA(ss->pq_xlist.alloc(sizeof(int) * ss->pq_cap, st));
            LF_CUDA(ss->pq_xn.alloc(sizeof(int), st));
            LF_CUDA(ss->pq_c16.alloc(16 * max_tasks, st));
        }
    }
    if (ss->q8) {
        const int MP = (idx.m + 255) / 256 * 256;
        LF_CUDA(ss->qc8.alloc((size_t)Q * MP, st));
        LF_CUDA(ss->qm8.alloc(sizeof(float4) * Q, st));
    }
    // counters zeroed inside kernels (RoundState)
    s.pq_n = ss->pq ? ss->pq_on.as<int>() : nullptr;
    s.pq_xn = ss->pq_xn.p ? ss->pq_xn.as<int>() : nullptr;
    s.cnt_all = ss->n_active.as<int>();
    s.rctr = ss->round_ctr.as<int>();
    s.ptotal = ss->lazy ? ss->ptotal.as<unsigned long long>() : nullptr;
    s.qbest = ss->pq ? ss->pq_qbest.as<unsigned>() : nullptr;
    return LF_OK;
}

// Per-batch work before round 0: query summaries, bounds, visit orders, state reset,
// query codes (stream-ordered; captured into the plan's graph).
static int session_prologue(lf_session* ss) {
    const lf_index& idx = ss->idx;
    const lf_search_opts& o = ss->opts;
    cudaStream_t st = ss->st;
    const int64_t Q = ss->Q;
    RoundState& s = ss->s;
    // the query-side codes (fp16 rows, projected and int8 codes) do not depend on the
    // bounds: a second stream computes them while the bound matrix is built (a parallel
    // branch of the plan's graph), joined before round 0
    cudaStream_t st2 = ss->st2;
    LF_CUDA(cudaEventRecord(ss->fork_ev, st));
    LF_CUDA(cudaStreamWaitEvent(st2, ss->fork_ev, 0));
    if (ss->lazy) {
        int rc = rows_to_f16(ss->d_q, Q, idx.m, ss->xh.as<__half>(), ss->xexp.as<int>(), st2, filter_width(idx, o));
        if (rc) return rc;
        ++ss->kernels;
    }
    if (ss->pq) {
        LF_CUDA(launch_project_queries(ss->d_q, Q, idx, ss->qcp.as<int8_t>(), ss->qmp.as<float4>(), st2));
        ++ss->kernels;
    }
    if (ss->q8) {
        const int MP = (idx.m + 255) / 256 * 256;
        int rq = quantize_queries(ss->d_q, Q, idx.m, MP, ss->qc8.as<int8_t>(), ss->qm8.as<float4>(), st2);
        if (rq) return rq;
        ++ss->kernels;
    }
    LF_CUDA(cudaEventRecord(ss->join_ev, st2));
    // (ea_count, round counter, pcount / preq / ptotal, qbest, counters: init_state_kernel)
    if (o.h_profile) {
        ss->prof = true;
        for (int i = 0; i < LF_N_PROF; ++i) o.h_profile[i] = 0.0;
        for (auto& e : ss->ev) LF_CUDA(cudaEventCreate(&e));
        LF_CUDA(cudaEventRecord(ss->ev[0], st));
    }
    int nk = 0;
    int rc;
    if (ss->pruned) {
        unsigned* qmax = ss->orng.as<unsigned>();     // zeroed by launch_bounds
        rc = bounds_phase(ss->d_q, Q, idx, ss->qsumm.as<double>(), ss->lb.as<double>(), qmax, qmax + Q,
                          ss->plb.as<double>(), ss->pnode.as<int>(), st, &nk);
    } else {
        rc = bounds_and_order(ss->d_q, Q, idx, ss->qsumm.as<double>(), ss->lb.as<double>(), ss->oa, st, &nk);
    }
    if (rc) return rc;
    if (ss->prof) LF_CUDA(cudaEventRecord(ss->ev[1], st));     // LF_PROF_BOUNDS_MS: means + bounds + order
    ss->kernels += nk;
    init_state_kernel<<<(unsigned)((Q + 127) / 128), 128, 0, st>>>(s);
    LF_CUDA(cudaGetLastError());
    ++ss->kernels;
    LF_CUDA(cudaStreamWaitEvent(st, ss->join_ev, 0));
    if (ss->prof) LF_CUDA(cudaEventRecord(ss->ev[2], st));
    return LF_OK;
}

static int session_begin(lf_session* ss) {
    int rc = session_alloc(ss);
    return rc ? rc : session_prologue(ss);
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

// One in-search prediction pass (see pairs_range_kernel), enqueued on the device only:
// all = 1 right after round 0 (every query with a finite bsf), all = 0 for the queries
// that asked for one (their bsf was still +inf after round 0).
// Pruned orders: the leaf records, built right after round 0 with thr = bsf0 * f
// (bound: the other shards' best-so-far, tightening it).
static int order_after_round0(lf_session* ss, const double* d_bound) {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ss->prof) {
        LF_CUDA(cudaEventCreate(&e0));
        LF_CUDA(cudaEventCreate(&e1));
        LF_CUDA(cudaEventRecord(e0, ss->st));
    }
    ss->oa.bound = d_bound;
    ss->oa.seed = ss->order_seed ? ss->pq_qbest.as<unsigned>() : nullptr;
    const unsigned* qmax = ss->orng.as<unsigned>();
    int rc = order_phase(ss->lb.as<double>(), ss->Q, ss->idx, qmax, qmax + ss->Q, ss->oa, ss->st);
    if (rc) return rc;
    ++ss->kernels;
    if (ss->prof) {
        LF_CUDA(cudaEventRecord(e1, ss->st));
        ss->oev.emplace_back(e0, e1);
    }
    return LF_OK;
}

static int predict_pass(lf_session* ss, int all) {
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
    pairs_range_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(s, ss->pcount.as<int>(), ss->pstart.as<int>(),
                                                                         ss->pend.as<int>(), all, ss->fhist.as<int>(), F);
    LF_CUDA(cudaGetLastError());
    const int64_t Lr = idx.n_leaves;
    const unsigned pgrid = (unsigned)((Q * ((Lr + PAIR_SPAN - 1) / PAIR_SPAN) * 32 + 255) / 256);
    // each query contributes at most one pair per filter: bucket f is filled in place at
    // f * Q (no counting pass), then the tile list is built from the bucket sizes
    pairs_pos_kernel<true><<<pgrid, 256, 0, st>>>(Q, (int)Lr, ss->pstart.as<int>(), ss->pend.as<int>(), s.leafo,
                                                  idx.d_leaf_filter, ss->fhist.as<int>(), ss->pdst.as<int2>(),
                                                  ss->prof ? ss->ptotal.as<unsigned long long>() : nullptr, (int)Q);
    LF_CUDA(cudaGetLastError());
    int rc = pair_tiles(ss->fhist.as<int>(), F, ss->fcur.as<int>(), ss->ptiles.as<int4>(), ss->ntiles.as<int>(), st,
                        (int)Q);
    if (rc) return rc;
    rc = filter_reach_f16(ss->xh.as<__half>(), ss->xexp.as<int>(), Q, filter_width(idx, o), o.d_W1T_h, o.d_wexp, o.d_b1, o.d_W2,
                          o.d_b2, F, ss->ptiles.as<int4>(), ss->ntiles.as<int>(), ss->pdst.as<int2>(), o.d_offset,
                          ss->adj.as<double>(), idx.n_leaves, st);
    if (rc) return rc;
    ss->kernels += 5;
    ++ss->predict_steps;
    if (ss->prof) {
        LF_CUDA(cudaEventRecord(e1, st));
        ss->pev.emplace_back(e0, e1);
    }
    return LF_OK;
}

// The kernels of one round -- plan, chunk offsets, task expansion, scan, merge -- with
// `counts` as the round's counters.  In a graph-launched plan (s.d_round set) the plan
// kernel derives R from the device round counter; otherwise s.R holds it.
static int round_kernels(lf_session* ss, int* counts, bool round0, cudaEvent_t* ev) {
    RoundState& s = ss->s;
    const lf_index& idx = ss->idx;
    const lf_search_opts& o = ss->opts;
    cudaStream_t st = ss->st;
    const int64_t Q = ss->Q;
    s.n_active = counts;
    s.n_predict = counts + 2;
    {   // stream-ordered rounds alternate two count slots: this round's merge zeroes the other
        int* base = ss->n_active.as<int>();
        s.zero_counts = ss->capturing ? nullptr : (counts == base ? base + 4 : base);
    }
    // the round's counters: zeroed by the previous round's consumer (graph: round_cond_kernel
    // after reading them; stream-ordered rounds alternate two slots, each zeroed by the
    // merge two rounds later's predecessor -- here, simply by the merge of the round
    // before, whose slot is the other one); the task counter chunk_off[Q] by the merge
    // of the round before, the entry counter by the plan kernel (init_state for round 0)
    if (ev) cudaEventRecord(ev[0], st);
    // the bounded scans take m % 4 == 0 (codes zero-padded to a multiple of 32)
    const bool ea = o.early_abandon && !s.want_trace && idx.m <= 512 && scan_variant() != 0 && ss->q8;
    // round 0 has no best-so-far yet: for k = 1 the projected scan seeds its threshold
    // with one exactly scored row per task (scan_pq_kernel SEED); for k > 1 (or
    // LF_SCAN_ROUND0=q8) the first round runs the full-length int8 scan
    const bool seed = round0 && s.k == 1 && round0_seeded();
    const bool pq_round = ea && ss->pq && (!round0 || !ss->q8 || seed);
    // k = 1 entry tail: the per-task (d, id) pairs, min'ed by 128-bit CAS (merge reads them)
    s.cand16 = (pq_round && s.k == 1 && ss->q8) ? ss->pq_c16.as<unsigned long long>() : nullptr;
    if (round0 && ss->pruned)
        first_leaf_plan_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(s, idx, ss->plb.as<double>(),
                                                                                   ss->pnode.as<int>(), ss->W);
    else
        plan_warp_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(s, idx);
    if (ev) cudaEventRecord(ev[1], st);
    cudaError_t ce;
    if (pq_round) {
        const PQOverflow ov{ss->pq_oent.as<int4>(), ss->pq_on.as<int>(),
                            ss->pq_obase.as<int>(), ss->pq_cap, ss->pq_wrows.as<unsigned short>(),
                            ss->pq_wdist.as<double>(), ss->q8 ? ss->qc8.as<int8_t>() : nullptr,
                            ss->q8 ? ss->qm8.as<float4>() : nullptr, (idx.m + 255) / 256 * 256,
                            ss->pq_lo8.as<float>(), ss->pq_thr.as<unsigned>(),
                            seed ? ss->pq_qbest.as<unsigned>() : nullptr,
                            s.k == 1 && ss->q8 ? ss->pq_xlist.as<int>() : nullptr,
                            s.k == 1 && ss->q8 ? ss->pq_xn.as<int>() : nullptr};
        if (round0) ss->order_seed = seed && ss->pruned && !std::getenv("LF_ORDER_AFTER_ROUND0");
        ce = launch_scan_pq(s, idx, ss->d_q, ss->qcp.as<int8_t>(), ss->qmp.as<float4>(), ss->pq_cnt.as<int>(), ov,
                            ss->max_tasks, st, round0 && ss->order_seed ? ss->scan0_ev : nullptr);
        ss->kernels += ss->q8 ? 3 : 2;
    } else if (ea) {
        ce = launch_scan_q8(s, idx, ss->d_q, ss->qc8.as<int8_t>(), ss->qm8.as<float4>(), st);
    } else {
        if (idx.m > 1024) return fail(LF_EINVAL, "series length > 1024 not supported");
        ce = launch_scan_full(s, idx, ss->d_q, st);
    }
    if (ce != cudaSuccess) return fail(LF_ECUDA, cudaGetErrorString(ce));
    if (ev) cudaEventRecord(ev[2], st);
    merge_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(s);
    LF_CUDA(cudaGetLastError());
    if (ev) cudaEventRecord(ev[3], st);
    ss->kernels += 3;
    return LF_OK;
}

// Enqueue one round into count slot round & 1; the counts are copied back
// asynchronously (done_ev).  session_harvest reads them.
static int session_enqueue(lf_session* ss, const double* d_bound, double* d_bsf_out) {
    RoundState& s = ss->s;
    const lf_search_opts& o = ss->opts;
    cudaStream_t st = ss->st;
    const int64_t Q = ss->Q;
    const int slot = ss->round & 1;
    int* counts = ss->n_active.as<int>() + 4 * slot;
    if (ss->pruned && ss->round == 1) {
        int rc = order_after_round0(ss, d_bound);
        if (rc) return rc;
    }
    if (ss->lazy && (ss->round == 1 || (ss->round > 1 && s.k > 1))) {
        // after round 0 every query with a finite bsf gets its reachable pairs predicted;
        // with k > 1 a walk whose bsf was still +inf then asks later (preq), and every
        // round starts with a pass over those requests (the same schedule as the graph)
        int rc = predict_pass(ss, ss->round == 1 ? 1 : 0);
        if (rc) return rc;
    }
    s.bound = d_bound;
    s.R = o.sequential ? 1
                       : (int)std::min<int64_t>(s.Rcap, (int64_t)1 << std::min(ss->round * s.growth, 30));
    int rc = round_kernels(ss, counts, ss->round == 0, ss->prof ? ss->rev[slot] : nullptr);
    if (rc) return rc;
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

// Wait for the oldest enqueued round's counts, run the host-decided follow-up
// (lazy prediction pass) and accumulate its profile.
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
        p[LF_PROF_REFILLS] = 0.0;
        for (auto& e : ss->oev) p[LF_PROF_BOUNDS_MS] += ev_ms(e.first, e.second);   // pruned orders
        double pms = 0.0;
        for (auto& e : ss->pev) pms += ev_ms(e.first, e.second);
        p[LF_PROF_PREDICT_MS] = pms;
        unsigned long long pairs = 0;
        if (ss->lazy) cudaMemcpy(&pairs, ss->ptotal.p, sizeof(pairs), cudaMemcpyDeviceToHost);
        p[LF_PROF_PAIRS] = (double)pairs;
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
    if (ss->fork_ev) cudaEventDestroy(ss->fork_ev);
    if (ss->join_ev) cudaEventDestroy(ss->join_ev);
    if (ss->scan0_ev) cudaEventDestroy(ss->scan0_ev);
    if (ss->order_ev) cudaEventDestroy(ss->order_ev);
    if (ss->st2) {
        cudaStreamSynchronize(ss->st2);
        cudaStreamDestroy(ss->st2);
    }
    for (auto* v : {&ss->pev, &ss->oev})
        for (auto& e : *v) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
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
    LF_REQUIRE((opts->d_pred == nullptr && opts->d_pred_f64 == nullptr && opts->d_W1T_h == nullptr) ||
                   (opts->d_offset != nullptr && idx->d_leaf_filter != nullptr),
               "filter predictions need offsets and a leaf->filter map");
    LF_REQUIRE(opts->d_W1T_h == nullptr || opts->d_pred != nullptr || opts->d_pred_f64 != nullptr ||
                   (opts->d_wexp != nullptr && opts->d_b1 != nullptr && opts->d_W2 != nullptr && opts->d_b2 != nullptr &&
                    filter_width(*idx, *opts) % 64 == 0 && filter_width(*idx, *opts) >= 64 &&
                    filter_width(*idx, *opts) <= 256 && filter_width(*idx, *opts) >= idx->m && opts->n_filters >= 1 &&
                    ((uintptr_t)opts->d_W1T_h & 15) == 0 && ((uintptr_t)opts->d_b1 & 15) == 0 &&
                    ((uintptr_t)opts->d_W2 & 15) == 0),
               "in-search filter inference needs W1T_h, wexp, b1, W2, b2 (16-byte aligned) and a filter width "
               "(filter_m, else m) in {64, 128, 192, 256}, >= m");
    LF_REQUIRE(opts->sequential || opts->max_round_leaves >= 1, "max_round_leaves must be >= 1");
    return LF_OK;
}

// ------------------------------------------------------------ search plans ----
// A plan owns one session's scratch for (index, Q, opts) and the whole batched
// search as ONE CUDA graph: prologue (bounds, visit orders, query codes), round 0,
// the in-search prediction pass, then a conditional WHILE node whose body is one
// round followed by round_cond_kernel, which advances the device round counter and
// keeps the loop going while any walk is active.  A search is then a query copy,
// one graph launch and the result copies: no host round trips, no per-call
// allocations, tensor-map encodes or launch latency between rounds.
__global__ void round_cond_kernel(int* __restrict__ counts, int* __restrict__ d_round, int max_rounds,
                                  cudaGraphConditionalHandle h) {
    const int r = *d_round + 1;
    *d_round = r;
    cudaGraphSetConditional(h, (counts[0] > 0 && r < max_rounds) ? 1u : 0u);
    for (int i = 0; i < 3; ++i) counts[i] = 0;     // the next round's counters (no memset node)
}

static int plan_capture(lf_session* ss, cudaStream_t cs, cudaStream_t cs2, int64_t* d_ids, double* d_dists,
                        cudaGraph_t* out) {
    RoundState& s = ss->s;
    const int64_t Q = ss->Q;
    int* counts = ss->n_active.as<int>();
    const int max_rounds = 2 * std::max(1, ss->idx.n_leaves) + 8;
    ss->st = cs;
    ss->capturing = true;
    LF_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed));
    int rc = session_prologue(ss);
    if (!rc) rc = round_kernels(ss, counts, true, nullptr);
    if (!rc && ss->pruned && ss->order_seed) {
        // the order branch: st2 from the seeded scan's end, joined before the prediction pass
        cudaError_t e = cudaStreamWaitEvent(ss->st2, ss->scan0_ev, 0);
        if (e != cudaSuccess) rc = fail(LF_ECUDA, cudaGetErrorString(e));
        if (!rc) {
            ss->st = ss->st2;
            rc = order_after_round0(ss, nullptr);
            ss->st = cs;
        }
        if (!rc && (e = cudaEventRecord(ss->order_ev, ss->st2)) == cudaSuccess)
            e = cudaStreamWaitEvent(cs, ss->order_ev, 0);
        if (!rc && e != cudaSuccess) rc = fail(LF_ECUDA, cudaGetErrorString(e));
    } else if (!rc && ss->pruned) {
        rc = order_after_round0(ss, nullptr);
    }
    if (!rc && ss->lazy) rc = predict_pass(ss, 1);
    cudaGraph_t g = nullptr;
    cudaGraphConditionalHandle h;
    cudaGraphNode_t cnode = nullptr;
    if (!rc) {
        cudaStreamCaptureStatus cst;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        cudaError_t e = cudaStreamGetCaptureInfo(cs, &cst, nullptr, &g, &deps, &nd);
        if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, g, 0, 0);
        if (e == cudaSuccess) {
            round_cond_kernel<<<1, 1, 0, cs>>>(counts, ss->round_ctr.as<int>(), max_rounds, h);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamGetCaptureInfo(cs, &cst, nullptr, &g, &deps, &nd);
        cudaGraphNodeParams cp = {};
        if (e == cudaSuccess) {
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            e = cudaGraphAddNode(&cnode, g, deps, nd, &cp);
        }
        if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(cs2, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                                cudaStreamCaptureModeRelaxed);
        if (e != cudaSuccess) rc = fail(LF_ECUDA, std::string("conditional graph node: ") + cudaGetErrorString(e));
        if (!rc) {
            ss->st = cs2;
            if (ss->lazy && s.k > 1) rc = predict_pass(ss, 0);   // walks whose bsf was +inf after round 0
            if (!rc) rc = round_kernels(ss, counts, false, nullptr);
            if (!rc) {
                round_cond_kernel<<<1, 1, 0, cs2>>>(counts, ss->round_ctr.as<int>(), max_rounds, h);
                if (cudaGetLastError() != cudaSuccess) rc = fail(LF_ECUDA, "round_cond_kernel launch");
            }
            cudaGraph_t body = nullptr;
            const cudaError_t e2 = cudaStreamEndCapture(cs2, &body);
            if (!rc && e2 != cudaSuccess) rc = fail(LF_ECUDA, std::string("body capture: ") + cudaGetErrorString(e2));
            ss->st = cs;
        }
        if (!rc) {
            const cudaError_t e3 = cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies);
            if (e3 != cudaSuccess) rc = fail(LF_ECUDA, std::string("capture dependencies: ") + cudaGetErrorString(e3));
        }
        if (!rc) {
            finish_kernel<<<(unsigned)((Q * s.k + 255) / 256), 256, 0, cs>>>(s, d_ids, d_dists);
            if (cudaGetLastError() != cudaSuccess) rc = fail(LF_ECUDA, "finish_kernel launch");
        }
    }
    cudaGraph_t full = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(cs, &full);
    ss->capturing = false;
    if (!rc && ee != cudaSuccess) rc = fail(LF_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ee));
    if (rc) {
        if (full) cudaGraphDestroy(full);
        return rc;
    }
    *out = full;
    return LF_OK;
}

}  // namespace lf

struct lf_search_plan {
    lf_session* ss = nullptr;
    lf::Scratch qbuf, ids, dists, stats;
    cudaStream_t cs = nullptr, cs2 = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int64_t Q = 0;
    int m = 0, k = 0;
};

static void plan_free(lf_search_plan* p) {
    if (!p) return;
    if (p->exec) cudaGraphExecDestroy(p->exec);
    if (p->graph) cudaGraphDestroy(p->graph);
    if (p->cs) cudaStreamSynchronize(p->cs);
    if (p->ss) lf::session_free(p->ss);              // its scratch is freed on p->cs
    for (lf::Scratch* b : {&p->qbuf, &p->ids, &p->dists, &p->stats})
        if (b->p) {
            cudaFreeAsync(b->p, b->s);
            b->p = nullptr;
        }
    if (p->cs) cudaStreamSynchronize(p->cs);
    if (p->cs) cudaStreamDestroy(p->cs);
    if (p->cs2) cudaStreamDestroy(p->cs2);
    delete p;
}

extern "C" {

lf_search_plan* lf_search_plan_create(const lf_index* idx, int64_t Q, const lf_search_opts* opts, void* stream) {
    if (lf::check_args(idx, Q, opts) != LF_OK) return nullptr;
    if (Q < 1) { lf::fail(LF_EINVAL, "empty query batch"); return nullptr; }
    if (opts->want_trace || opts->h_profile) {
        lf::fail(LF_EINVAL, "search plans do not trace or profile: use lf_search");
        return nullptr;
    }
    auto* p = new lf_search_plan();
    p->Q = Q;
    p->m = idx->m;
    p->k = opts->k;
    cudaStream_t st = lf::as_stream(stream);
    auto bail = [&](const char* what, cudaError_t e) -> lf_search_plan* {
        if (e != cudaSuccess) lf::fail(LF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
        plan_free(p);
        return nullptr;
    };
    cudaError_t e = cudaStreamCreateWithFlags(&p->cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->cs2, cudaStreamNonBlocking);
    if (e != cudaSuccess) return bail("plan streams", e);
    if ((e = p->qbuf.alloc(sizeof(float) * Q * idx->m, p->cs)) != cudaSuccess ||
        (e = p->ids.alloc(sizeof(int64_t) * Q * opts->k, p->cs)) != cudaSuccess ||
        (e = p->dists.alloc(sizeof(double) * Q * opts->k, p->cs)) != cudaSuccess ||
        (e = p->stats.alloc(sizeof(int64_t) * Q * LF_N_STATS, p->cs)) != cudaSuccess)
        return bail("plan buffers", e);
    auto* ss = new lf_session();
    p->ss = ss;
    ss->idx = *idx;
    ss->opts = *opts;
    ss->opts.want_trace = 0;
    ss->st = p->cs;
    ss->Q = Q;
    ss->d_q = p->qbuf.as<float>();
    ss->s.stats = p->stats.as<long long>();
    if (lf::session_alloc(ss) != LF_OK) return bail("", cudaSuccess);
    ss->s.d_round = ss->round_ctr.as<int>();
    if ((e = cudaStreamSynchronize(p->cs)) != cudaSuccess) return bail("plan allocation", e);
    (void)st;
    if (lf::plan_capture(ss, p->cs, p->cs2, p->ids.as<int64_t>(), p->dists.as<double>(), &p->graph) != LF_OK)
        return bail("", cudaSuccess);
    if ((e = cudaGraphInstantiate(&p->exec, p->graph, 0)) != cudaSuccess) return bail("graph instantiate", e);
    return p;
}

int lf_search_plan_run(lf_search_plan* p, const float* d_queries, int64_t* d_out_ids, double* d_out_dists,
                       int64_t* d_out_stats, void* stream) {
    LF_REQUIRE(p != nullptr && d_queries != nullptr, "NULL argument");
    cudaStream_t st = lf::as_stream(stream);
    LF_CUDA(cudaMemcpyAsync(p->qbuf.p, d_queries, sizeof(float) * p->Q * p->m, cudaMemcpyDeviceToDevice, st));
    LF_CUDA(cudaGraphLaunch(p->exec, st));
    if (d_out_ids)
        LF_CUDA(cudaMemcpyAsync(d_out_ids, p->ids.p, sizeof(int64_t) * p->Q * p->k, cudaMemcpyDeviceToDevice, st));
    if (d_out_dists)
        LF_CUDA(cudaMemcpyAsync(d_out_dists, p->dists.p, sizeof(double) * p->Q * p->k, cudaMemcpyDeviceToDevice, st));
    if (d_out_stats)
        LF_CUDA(cudaMemcpyAsync(d_out_stats, p->stats.p, sizeof(int64_t) * p->Q * LF_N_STATS,
                                cudaMemcpyDeviceToDevice, st));
    return LF_OK;
}

void lf_search_plan_free(lf_search_plan* p) { plan_free(p); }

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
    LF_REQUIRE(ss->harvested == ss->round, "rounds in flight: call lf_search_round_wait first");
    return lf::session_round(ss, d_bound, d_bsf_out, h_active);
}

int lf_search_round_async(lf_session* ss, const double* d_bound, double* d_bsf_out, int32_t* d_active) {
    LF_REQUIRE(ss != nullptr, "NULL session");
    LF_REQUIRE(ss->round - ss->harvested < 2, "at most two rounds in flight: call lf_search_round_wait first");
    const int slot = ss->round & 1;
    int rc = lf::session_enqueue(ss, d_bound, d_bsf_out);
    if (rc) return rc;
    if (d_active)
        LF_CUDA(cudaMemcpyAsync(d_active, ss->n_active.as<int>() + 4 * slot, sizeof(int), cudaMemcpyDeviceToDevice,
                                ss->st));
    return LF_OK;
}

int lf_search_round_wait(lf_session* ss, int32_t* h_active) {
    LF_REQUIRE(ss != nullptr && h_active != nullptr, "NULL argument");
    LF_REQUIRE(ss->harvested < ss->round, "no round in flight");
    int act = 0;
    int rc = lf::session_harvest(ss, &act);
    *h_active = act;
    return rc;
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
    if (rc == LF_OK) rc = lf_search_end(ss, d_out_ids, d_out_dists);
    lf_search_free(ss);
    return rc;
}

}  // extern "C"
