// Shared state and helpers of the round-driven batched search (search.cu and the
// scan kernels in scan_*.cu): the per-round state every kernel reads, the bound a
// round prunes with, the TMA bulk-copy / mbarrier helpers of the pipelined scans,
// and the host launchers each scan file exports.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <climits>

#include "common.cuh"

namespace lf {

constexpr int CH = 512;          // rows per scan task (512 KiB at m = 256)
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_WARPS = SCAN_THREADS / 32;

struct RoundState {
    int64_t Q;
    int k, kc;                   // kc = candidates kept per task = min(k, CH)
    int R, Rcap;                 // leaves per query this round, and the buffer stride
    int seq, growth;             // sequential schedule; leaves per round grow as 2^(round * growth)
    const int* d_round;          // device round counter (graph-launched plans): R derived from it, else s.R
    double f;                    // bsf_factor
    const int* order;            // [Q][L] visit-order leaf records (bounds.cuh OrderArgs): node ids (traces)
    const double* lbs;           // [Q][L] leaf bound
    const double* gap;           // [Q][L] largest non-leaf bound popped since the previous leaf (0: none)
    const int* leafo;            // [Q][L] leaf slot | LF_REC_HASF
    const double* adj;           // [Q][L] pred - offset of the leaf's filter
    const int* olen;             // [Q] records of the order (= L)
    int lazy;                    // in-search filter inference: adj valid for positions < pcount[q]
    int* pcount;                 // [Q]
    int* preq;                   // [Q] set when the walk stopped at pcount (more predictions needed)
    int* n_predict;              // walks that reached pcount with a finite bsf (= n_active + 2)
    int* cursor;                 // [Q]
    int* done;                   // [Q]
    double* top_d;               // [Q][k]   running top-k (round-start state)
    long long* top_i;            // [Q][k]
    int* top_n;                  // [Q]
    double* top_d_out;           // merge's scratch: the new top-k, copied back into top_d
    long long* top_i_out;
    int* top_n_out;
    int n_leaves;
    const double* bound;         // [Q] external best-so-far bound (other shards), or NULL
    long long* stats;            // [Q][6]
    int* sel_leaf;               // [Q][Rcap]
    int* sel_trace;              // [Q][Rcap]
    int* sel_pre;                // [Q][Rcap+1] chunk prefix within the query
    int* n_sel;                  // [Q]
    long long* chunk_off;        // [Q+1]: first task of query q; [Q] = the round's task count (atomic)
    int* chunk_cnt;              // [Q] tasks of query q this round
    int4* tasks;                 // [max_tasks] (query, leaf slot, chunk, selection index)
    int4* task_rows;             // [max_tasks] (r0 lo, r0 hi, rows, query) or NULL
    unsigned long long* ea_count;  // [2] rows tested / survivors (profiling only, may be NULL)
    double* cand_d;              // [max_tasks][kc]
    long long* cand_i;
    double* task_min;            // [max_tasks] (trace only)
    int* n_active;
    // counters zeroed inside kernels instead of graph memset nodes (~0.85 us per node):
    int* pq_n;                   // projected-scan entry count: zeroed by the plan kernels
    int* pq_xn;                  // exact-tail list length: zeroed by the int8 stage
    int* cnt_all;                // [8] round counters (both slots): zeroed by init_state
    int* zero_counts;            // stream-ordered rounds: the next round's counter slot, zeroed by merge
    unsigned long long* cand16;  // k = 1 entry tail: per task (d bits, id), 16-byte aligned, min'ed by a 128-bit CAS, or NULL
    int* rctr;                   // graph round counter, or NULL: zeroed by init_state
    unsigned long long* ptotal;  // pair total (profiling), or NULL: zeroed by init_state
    unsigned* qbest;             // seeded round 0: per-query seed minimum, set to 3.4e38 by init_state
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

// ---- host launchers (one per scan file); each returns the launch error
// scan_fp32.cu: fp64 full scan (VEC float4 per lane): traces, and indexes without a shadow
cudaError_t launch_scan_full(const RoundState& s, const lf_index& idx, const float* q, cudaStream_t st);
// scan_q8.cu: TMA-pipelined int8-bounded scan
cudaError_t launch_scan_q8(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc8,
                           const float4* qm8, cudaStream_t st);
// scan_pq.cu: projected two-stage scan
cudaError_t launch_project_queries(const float* q, int64_t Q, const lf_index& idx, int8_t* qc, float4* qm,
                                   cudaStream_t st);
// Survivors of the projected scan: (task, row) entries, contiguous per task, for pq_tail_kernel.
struct PQOverflow {
    int4* ent;                                // [cap] (task, query, absolute row lo, hi); task < 0: unused
    int* n;                                   // entries claimed this launch (device counter)
    int* base;                                // [max_tasks] first entry of a task
    int cap;
    unsigned short* wrows;                    // [scan warps][CH] rows / distances of a task whose
    double* wdist;                            //   entries did not fit (re-read in the scan warp)
    // second stage: the full-length int8 interval of every entry (nullptr qc8: no stage)
    const int8_t* qc8;                        // [Q][mp] query codes (quantize_queries)
    const float4* qm8;                        // [Q] query code metadata
    int mp;
    float* lo8;                               // [cap] int8 lower bound of each entry
    unsigned* thr;                            // [max_tasks] the projected stage's threshold (float bits)
    // round 0 (no best-so-far yet, k = 1): every task exactly scores the row its projected
    // codes rank nearest and prunes with that distance; qbest [Q] shares the best seed of
    // a query's tasks (float bits, atomicMin).  nullptr: no seeding.
    unsigned* qbest;
    int* xlist;                               // [cap] entries re-read exactly (k = 1 entry tail; s.cand16 set)
    int* xn;                                  // their count
};
int pq_scan_warps();                          // warps of one scan_pq_kernel launch
constexpr int PQ_OVER_CAP = 8 << 20;          // 8M entries (128 MB + lo8)
// after_scan (nullable): recorded right after the streaming scan kernel (round 0: the
// seed minima in ov.qbest are final there)
cudaError_t launch_scan_pq(const RoundState& s, const lf_index& idx, const float* q, const int8_t* qc,
                           const float4* qm, int* surv_cnt, const PQOverflow& ov, int64_t max_tasks,
                           cudaStream_t st, cudaEvent_t after_scan = nullptr);

}  // namespace lf
