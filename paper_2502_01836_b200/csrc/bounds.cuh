#pragma once
#include <cuda_runtime.h>

#include "../../include/leafi_b200.h"

namespace lf {
// mode 0 / 1: the reference's search / traingen bound; 2: EAPCA (sd_min / sd_max).
// d_qmax / d_qmin (nullable, [Q]): per query the range of its leaf bounds as float bits
// (d_qmin complemented, so both are zero-initialised here).
int launch_bounds(const float* d_q, int64_t Q, const lf_index& idx, const double* env_min,
                  const double* env_max, int n_env, int mode, double* d_qsumm, double* d_lb,
                  cudaStream_t st, unsigned* d_qmax = nullptr, unsigned* d_qmin = nullptr,
                  const double* sd_min = nullptr, const double* sd_max = nullptr, double* d_plb = nullptr,
                  int* d_pnode = nullptr);

// Per-query visit-order records [Q][L] over the L LEAF slots of the index, in
// (lb, node id) order -- the pop order of tree.py:256-275 restricted to the
// leaves.  Internal nodes (and, on a leaf shard, the other shards' leaves) are
// not records: the only thing they decide is where the walk stops.  The walk
// stops at the first popped node with lb > bsf * f (tree.py:261); an internal
// node there ends the walk WITHOUT counting a leaf (tree.py:262-265), a leaf
// counts as visited + lb-pruned.  Because bounds are popped in ascending order,
// "some non-leaf node between leaf i-1 and leaf i has lb > thr" is the same as
// gap[i] > thr, gap[i] = the largest such bound (0 if none): the walk at leaf i
// stops uncounted if gap[i] > thr, else counted if lb[i] > thr.
//   leafo = leaf slot | LF_REC_HASF when the leaf has a filter;
//   adj   = prediction - offset of that filter (the exact operand of the filter
//           rule, tree.py:282), gathered once so the plan never chases it;
//   order = node id (written only when `order` is non-NULL: traces).
constexpr int LF_REC_HASF = 1 << 30;
constexpr int LF_REC_LEAF = LF_REC_HASF - 1;
struct OrderArgs {
    double* lbs;
    double* gap;
    int* order;                  // may be NULL
    int* leafo;
    double* adj;
    int* olen;
    const float* pred;           // [Q][F] or NULL
    const double* pred64;        // [Q][F] or NULL
    const double* offset;        // [F]
    int F;
    int lazy;                    // predictions computed later (lazy inference): flag filters, adj = NaN
    // pruned orders (prune = 1, built after round 0): only the leaves with lb <= thr,
    // thr = bsf * f from the running top-k (k-th best, tightened by `bound`), in
    // (lb, id) order, then ONE terminal record: the first leaf past thr, carrying the
    // gap of the internal nodes popped before it.  bsf never rises, so every later
    // walk stops at or before the terminal record; thr = +inf gives the full order.
    int prune;
    const double* top_d;         // [Q][k]
    const int* top_n;            // [Q]
    int k;
    double f;
    const double* bound;         // [Q] or NULL
    // k = 1 seeded round 0: thr = seed * f instead of the top-k, seed = float bits of the
    // exactly scored seed rows' minimum per query (>= bsf0, so the order is a superset of
    // the bsf0-pruned one with the same prefix) -- available before round 0's merge, so
    // the order is built concurrently with the rest of round 0
    const unsigned* seed;        // [Q] or NULL
};
// Two phases of bounds_and_order, for orders built after round 0:
//   bounds_phase: segment means, bound matrix, the range of each query's leaf
//                 bounds (qmax / qmin float bits), and per (query, 32-node group)
//                 the minimum (lb, node id) over its leaves (plb / pnode [Q][W],
//                 W = ceil(n_nodes / 32); +inf / -1: no leaf) -- the first leaf a
//                 walk pops, for round 0's plan;
//   order_phase:  the records (leaf_order_kernel).
// fused_order_ok: the tree fits leaf_order_kernel (<= 8192 nodes, <= 4096 leaf
// slots, <= 8 segments).
bool fused_order_ok(const lf_index& idx, int64_t Q);
int bounds_phase(const float* d_q, int64_t Q, const lf_index& idx, double* d_qsumm, double* d_lb, unsigned* qmax,
                 unsigned* qmin, double* plb, int* pnode, cudaStream_t st, int* kernels);
int order_phase(const double* d_lb, int64_t Q, const lf_index& idx, const unsigned* qmax, const unsigned* qmin,
                const OrderArgs& oa, cudaStream_t st);
// Segment means (d_qsumm [Q][n_seg]), node bounds (d_lb [Q][n_nodes], the search
// bound of summarize.py:97-107) and the leaf records above.
int bounds_and_order(const float* d_q, int64_t Q, const lf_index& idx, double* d_qsumm, double* d_lb,
                     const OrderArgs& oa, cudaStream_t st, int* kernels);
int sort_visit_order(const double* d_lb, int64_t Q, int n, double* d_lb_sorted, int* d_order,
                     cudaStream_t st);
}  // namespace lf
