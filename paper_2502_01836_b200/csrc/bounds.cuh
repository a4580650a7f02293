#pragma once
#include <cuda_runtime.h>

#include "../../include/leafi_b200.h"

namespace lf {
int launch_bounds(const float* d_q, int64_t Q, const lf_index& idx, const double* env_min,
                  const double* env_max, int n_env, int mode, double* d_qsumm, double* d_lb,
                  cudaStream_t st);
// Per-query visit-order records [Q][n_nodes] in (lb, node id) order; only the
// first olen[q] entries are valid (a sorted PREFIX of the full order, or all of
// it).  leafo = leaf slot | LF_REC_HASF when the leaf has a filter, -1 for an
// internal node; adj = prediction - offset of that filter (the exact operand of
// the filter rule, tree.py:282), gathered once so the plan never chases it.
constexpr int LF_REC_HASF = 1 << 30;
constexpr int LF_REC_LEAF = LF_REC_HASF - 1;
struct OrderArgs {
    double* lbs;
    int* order;
    int* leafo;
    double* adj;
    int* olen;
    const float* pred;           // [Q][F] or NULL
    const double* pred64;        // [Q][F] or NULL
    const double* offset;        // [F]
    int F;
    int* only;                   // refill: queries with only[q] != 0 (cleared when done); NULL = all
    int lazy;                    // predictions computed later (lazy inference): flag filters, adj = NaN
};
// prefix = true: sort only the first ~PF_K entries of each order (olen[q] < n_nodes
// possible); the plan asks for the rest with refill_order when it gets there.
int bounds_and_order(const float* d_q, int64_t Q, const lf_index& idx, double* d_qsumm, double* d_lb_scratch,
                     const OrderArgs& oa, bool prefix, cudaStream_t st, int* kernels);
// Full order for the queries flagged in oa.only (the first olen[q] entries are
// unchanged: the prefix is the head of the full order).
int refill_order(const float* d_q, int64_t Q, const lf_index& idx, const double* d_qsumm, double* d_lb_scratch,
                 const OrderArgs& oa, cudaStream_t st, int* kernels);
int sort_visit_order(const double* d_lb, int64_t Q, int n, double* d_lb_sorted, int* d_order,
                     cudaStream_t st);
}  // namespace lf
