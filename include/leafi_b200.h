/*
 * leafi_b200.h -- C-ABI of the B200-native LeaFi hot path (arXiv 2502.01836).
 *
 * The reference (`leafsearch`, pure Python/numpy) has no FFI: its seams are
 * Python functions.  Each entry point below replaces one of them and is bound
 * from Python with ctypes.  Conventions:
 *
 *   - every pointer named d_* is DEVICE memory owned by the caller (torch
 *     tensors in the Python host layer); h_* pointers are host memory;
 *   - `stream` is a cudaStream_t passed as void*; all work is stream-ordered;
 *   - functions return 0 on success, a nonzero LF_E* code otherwise; the
 *     message is available from lf_last_error() (thread-local);
 *   - no torch types, no C++ types cross this boundary.
 *
 * Series are stored fp32 (lossless: the reference keeps fp32-exact values,
 * series.py:48-50) in LEAF-CONTIGUOUS order: leaves in ascending node id,
 * members of a leaf in ascending series id (tree.py:102-106,152,184).
 */
#ifndef LEAFI_B200_H
#define LEAFI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LF_OK 0
#define LF_EINVAL 1     /* bad argument (maps to ValueError in Python) */
#define LF_ECUDA 2      /* CUDA runtime error (maps to RuntimeError) */
#define LF_ENOMEM 3
#define LF_EFORMAT 4    /* malformed LEAF file (maps to FormatError, series.py:25-31) */

#define LF_MAX_SEG 64
#define LF_N_STATS 6    /* visited, searched, lb_pruned, filter_pruned, inferences, series_scanned */

/* Device-resident index (the GPU image of reference tree.Index, tree.py:93-122). */
typedef struct lf_index {
    int64_t n_series;        /* rows in X */
    int32_t m;               /* series length */
    int32_t n_seg;           /* segments (summarize.py:15-37) */
    int32_t n_nodes;         /* all tree nodes, ids 0..n_nodes-1 */
    int32_t n_leaves;        /* leaves, slots 0..n_leaves-1 in ascending node id */
    int64_t max_leaf_rows;   /* largest leaf (rows) */
    int32_t seg_start[LF_MAX_SEG];
    int32_t seg_width[LF_MAX_SEG];
    const float* d_X;            /* [n_series][m] leaf-contiguous */
    const int64_t* d_row_id;     /* [n_series] original series id of each row */
    const int64_t* d_leaf_ptr;   /* [n_leaves+1] row offsets */
    const int32_t* d_node_leaf;  /* [n_nodes] leaf slot, -1 for internal nodes */
    const double* d_env_min;     /* [n_seg][n_nodes] SoA envelope minima */
    const double* d_env_max;     /* [n_seg][n_nodes] SoA envelope maxima */
    const int32_t* d_leaf_filter;/* [n_leaves] filter slot or -1 (may be NULL) */
    /* optional int8 shadow of X for the bounded scan (lf_quantize_rows); all NULL = unused */
    const int8_t* d_X8;          /* [n_series][roundup(m, 32)] round(x / scale), zero-padded */
    const float* d_qmeta;        /* [n_series][4] per row: scale = max|x| / 127, sum of squared
                                    codes (exact in fp32), ||scale * code - x||_2 rounded up, 0 */
    /* optional projected shadow for the two-stage scan (NULL = unused): an orthonormal
       basis P of pca_k directions (fp64, rows orthonormal), the mean mu, and per row the
       int8 codes of y = P (x - mu) and 8 bytes of fp16 metadata {scale (the exact
       quantisation step: codes = rint(y / scale)), ||scale*code - y|| rounded up,
       ||(x - mu) - P^T y|| rounded to nearest, 0}; ||scale * code||^2 is recomputed from
       the codes -- ||x - q||^2 = ||y - y_q||^2 + ||r - r_q||^2 */
    int32_t pca_k;               /* 32 or 64 (0 = no projected shadow) */
    const double* d_P;           /* [pca_k][m] */
    const double* d_mu;          /* [m] */
    const int8_t* d_Xp;          /* [n_series][pca_k] */
    const uint16_t* d_pmeta;     /* [n_series + 2][4] fp16 bits (two rows of padding) */
    /* optional EAPCA envelopes (NULL = the reference's mean-only bound): per node the
       [min, max] of its members' segment standard deviations, SoA [n_seg][n_nodes];
       with them the search bound is the EAPCA bound (lf_bounds_eapca) */
    const double* d_sd_min;
    const double* d_sd_max;
} lf_index;

/* Options of one batched search (tree.py:220-229 search_engine keyword args). */
typedef struct lf_search_opts {
    int32_t k;                   /* 1 <= k <= n_series */
    double bsf_factor;           /* tree.py:261,282; 1/(1+eps) for cli.py:57-65 */
    const float* d_pred;         /* [Q][n_filters] filter predictions, or NULL */
    const double* d_pred_f64;    /* same in fp64 (host predictor callables); used if non-NULL */
    const double* d_offset;      /* [n_filters] conformal offsets (enhanced.py:127-134) */
    int32_t n_filters;
    int32_t sequential;          /* 1: one scanned leaf per query per round (exact
                                    reference semantics, every counter identical);
                                    0: growing rounds 1,4,16,..,max_round_leaves leaves per
                                       query (x4 per round; LF_ROUND_GROWTH_LOG2 overrides) */
    int32_t max_round_leaves;    /* cap of the round schedule (>= 1; the Python API uses 256) */
    int32_t want_trace;          /* fill the trace buffers below */
    int32_t early_abandon;       /* 1: abandon a row once its partial distance exceeds the
                                    threshold (HBM bytes saved; results identical; off when
                                    tracing; needs m % 64 == 0) */
    double* h_profile;           /* optional host array[LF_N_PROF]: CUDA-event times (ms)
                                    accumulated per phase, see LF_PROF_* */
    /* In-search filter inference (used when d_pred and d_pred_f64 are NULL and d_W1T_h
       is set): the fp16 filter pack -- W1T_h [F][hidden][in] fp16 bits with per-filter
       power-of-two exponents d_wexp (lf_filter_predict_f16's operands), b1 [F][m],
       W2 [F][m], b2 [F]; m in {64, 128, 192, 256}, or (filter_m below) any m <= 256 with
       the pack zero-padded to filter_m = roundup(m, 64).  Round 0 needs no prediction (bsf is
       +inf); right after it ONE tensor-core pass predicts exactly the (query, filtered
       leaf) pairs with lb <= bsf0 * f -- every pair the walk can still reach, since bsf
       only decreases -- bit-identical to lf_filter_predict_f16's predictions.  (A query
       whose bsf is still +inf after round 0, k > first leaf's size, gets its pass when
       it asks for one.) */
    const uint16_t* d_W1T_h;
    const int32_t* d_wexp;
    const float* d_b1;
    const float* d_W2;
    const float* d_b2;
    int32_t filter_m;            /* width of the in-search filter operands: 0 = m; else
                                    roundup(m, 64) <= 256, the fp16 pack's W1T_h / b1 / W2
                                    zero-padded to it (query rows are padded on the device) */
} lf_search_opts;

#define LF_N_PROF 15
#define LF_PROF_BOUNDS_MS 0      /* segment means + node bounds + leaf visit orders (records) */
#define LF_PROF_PLAN_MS 1        /* plan + chunk offsets, all rounds */
#define LF_PROF_SCAN_MS 2        /* leaf-scan kernel, all rounds */
#define LF_PROF_MERGE_MS 3       /* top-k merge, all rounds */
#define LF_PROF_ROUNDS 4         /* rounds executed */
#define LF_PROF_KERNELS 5        /* kernels launched by the library (own kernels; CUB sort counted as 1) */
#define LF_PROF_TOTAL_MS 6       /* whole call, first to last event */
#define LF_PROF_REFILLS 7        /* reserved (0) */
#define LF_PROF_EA_ROWS 8        /* rows tested by the early-abandon scan */
#define LF_PROF_EA_SURVIVORS 9   /* rows that survived the first 64-dim test */
#define LF_PROF_PREDICT_MS 10    /* in-search filter inference (pair lists + tensor-core GEMM) */
#define LF_PROF_PAIRS 11         /* (query, leaf) predictions computed in the search */
#define LF_PROF_PREDICT_STEPS 12 /* in-search inference passes (one after round 0, then on request) */
#define LF_PROF_SCAN_STREAM_BYTES 13 /* bytes the scans streamed (codes + row metadata, or fp32 rows) */
#define LF_PROF_SCAN_EXACT_BYTES 14  /* fp32 bytes re-read for exact distances of surviving rows */

/* Optional per-query trace (tree.py:77-83 TraceEntry), capacity n_leaves per query. */
typedef struct lf_trace {
    int32_t* d_len;        /* [Q] entries written */
    int32_t* d_leaf;       /* [Q][n_leaves] node id of the visited leaf */
    double* d_lb;          /* [Q][n_leaves] its lower bound */
    int8_t* d_searched;    /* [Q][n_leaves] 1 if scanned */
    double* d_leaf_nn;     /* [Q][n_leaves] min distance in the leaf (NaN if not scanned) */
    double* d_bsf_before;  /* [Q][n_leaves] best-so-far used for the decision */
} lf_trace;

const char* lf_last_error(void);
int lf_version(void);
int lf_device_sm_count(int device);

/*
 * Struct layout as this library was compiled, for bindings that mirror the
 * structs above (ctypes, cgo, JNA): lf_abi_sizeof("lf_index") is sizeof, and
 * lf_abi_offsetof("lf_index", "d_X") the field's offsetof; -1 for an unknown
 * struct or field.  Types: "lf_index", "lf_search_opts", "lf_trace".
 */
int64_t lf_abi_sizeof(const char* type_name);
int64_t lf_abi_offsetof(const char* type_name, const char* field_name);

/*
 * Query segment means and node lower bounds.
 * Replaces summarize.summarize_series/matrix (summarize.py:44-56) and
 * lower_bound_from_summary / lower_bounds_batch (summarize.py:97-122).
 *   lb_mode 0: the search-path bound (np.dot: one FMA chain), tree.py:256,273
 *   lb_mode 1: the batched traingen bound (einsum order), traingen.py:167-169
 * Outputs d_qsumm [Q][n_seg] and d_lb [Q][n_nodes] (n_nodes of the SoA arrays).
 */
int lf_bounds(const float* d_queries, int64_t Q, const lf_index* idx,
              const double* d_env_min, const double* d_env_max, int32_t n_env,
              int32_t lb_mode, double* d_qsumm, double* d_lb, void* stream);

/*
 * EAPCA bound (DSTree's mean + standard deviation summary; no reference code --
 * the reference envelope keeps means only, summarize.py:59-107): per segment the
 * reference mean and sd = sqrt(sum (x_t - mean)^2 / w) (left-to-right fp64 sum),
 * lb = sqrt(sum_i w_i (gm_i^2 + gs_i^2)) with gm / gs the gaps of the query's
 * mean / sd to the node's [min, max] (summarize.py:97-107 shape).  d_qsumm
 * [Q][2 n_seg] receives the query means then sds; d_lb [Q][n_env].
 */
int lf_bounds_eapca(const float* d_queries, int64_t Q, const lf_index* idx, const double* d_env_min,
                    const double* d_env_max, const double* d_sd_min, const double* d_sd_max, int32_t n_env,
                    double* d_qsumm, double* d_lb, void* stream);
/* Per-row EAPCA summaries of device rows: d_out [n][2 n_seg] = means then sds. */
int lf_eapca_device(const float* d_values, int64_t n, int32_t m, int32_t n_seg, double* d_out, void* stream);

/*
 * Batched best-first search: bounds, per-query (lb, node id) visit order,
 * round-driven cascade lb -> filter -> leaf scan, top-k by (distance, id).
 * Replaces tree.search_engine (tree.py:220-297) for a batch of Q queries.
 * Outputs: d_out_ids [Q][k] (int64), d_out_dists [Q][k], d_out_stats [Q][6].
 * `trace` may be NULL.
 */
int lf_search(const lf_index* idx, const float* d_queries, int64_t Q,
              const lf_search_opts* opts, int64_t* d_out_ids, double* d_out_dists,
              int64_t* d_out_stats, const lf_trace* trace, void* stream);

/*
 * Search plans: the batched search above as ONE CUDA graph, built once for an
 * (index, Q, opts) and launched per query batch.  The plan owns its scratch; the
 * graph holds the prologue (bounds, visit orders, query codes), round 0, the
 * in-search prediction pass and a conditional WHILE node over the rounds (the round
 * counter and the "any walk active" test live on the device), so a search is a
 * query copy, one graph launch and the result copies -- no host round trips.
 * Results and counters are those of lf_search with the same opts (no traces or
 * profiles: want_trace and h_profile must be 0).  The index, predictions, offsets
 * and filter buffers named by idx / opts must stay allocated and unchanged for the
 * plan's life; d_queries [Q][m] may change per run.
 */
typedef struct lf_search_plan lf_search_plan;
lf_search_plan* lf_search_plan_create(const lf_index* idx, int64_t Q, const lf_search_opts* opts, void* stream);
int lf_search_plan_run(lf_search_plan* plan, const float* d_queries, int64_t* d_out_ids, double* d_out_dists,
                       int64_t* d_out_stats, void* stream);
void lf_search_plan_free(lf_search_plan* plan);

/*
 * The same search split into rounds, for callers that exchange the per-query
 * best-so-far between rounds (leaf-sharded multi-GPU: allreduce-min over NVLink).
 *   s = lf_search_begin(idx, q, Q, opts, trace, d_stats, stream)   bounds + order
 *   do lf_search_round(s, d_bound, d_bsf_out, &active)             one round
 *   while (global active > 0)
 *   lf_search_end(s, d_out_ids, d_out_dists); lf_search_free(s)
 * d_bound [Q] (nullable): external bound; the round prunes with
 * min(local k-th best, d_bound[q]).  d_bsf_out [Q] (nullable): local k-th best
 * after the round (inf while fewer than k found).  Counters accumulate into
 * d_stats [Q][6] (zeroed by begin).  The session is bound to `stream`.
 */
typedef struct lf_session lf_session;
lf_session* lf_search_begin(const lf_index* idx, const float* d_queries, int64_t Q,
                            const lf_search_opts* opts, const lf_trace* trace, int64_t* d_stats,
                            void* stream);
int lf_search_round(lf_session* s, const double* d_bound, double* d_bsf_out, int32_t* h_active);
/*
 * The same round without a host synchronisation, so a caller can keep one round
 * in flight while the bound exchange of the previous one runs (leaf-sharded
 * search: the ranks' MIN-allreduce of [bsf, -active] is stream-ordered after the
 * round and before the next).  lf_search_round_async enqueues the round and
 * writes its active-query count to the DEVICE int *d_active (nullable);
 * lf_search_round_wait waits for the OLDEST enqueued round and returns its count
 * in *h_active.  At most two rounds may be in flight; not for lazy inference.
 */
int lf_search_round_async(lf_session* s, const double* d_bound, double* d_bsf_out, int32_t* d_active);
int lf_search_round_wait(lf_session* s, int32_t* h_active);
int lf_search_end(lf_session* s, int64_t* d_out_ids, double* d_out_dists);
void lf_search_free(lf_session* s);

/*
 * Filter inference for every (query, filter) pair, batch-invariant fp32.
 * Replaces MlpModel.forward (mlp.py:90-95) as called per leaf at tree.py:281.
 *   W1 [F][m][m] (x @ W1 layout, mlp.py:94), b1 [F][m], W2 [F][m], b2 [F]
 * Output d_pred [Q][F].
 */
int lf_filter_predict(const float* d_queries, int64_t Q, int32_t m,
                      const float* d_W1, const float* d_b1, const float* d_W2,
                      const float* d_b2, int32_t F, float* d_pred, void* stream);

/*
 * Same on the 5th-gen tensor cores (tcgen05.mma kind::tf32, TMA-fed, TMEM
 * accumulators, fused bias/rectifier/W2 epilogue).  W1T is the TRANSPOSED
 * first layer, [F][hidden][in] (K-major B operand); m in {32, 64, ..., 256}.
 * Batch-invariant like lf_filter_predict; precision is tf32 products with
 * fp32 accumulation.
 */
int lf_filter_predict_tc(const float* d_queries, int64_t Q, int32_t m,
                         const float* d_W1T, const float* d_b1, const float* d_W2,
                         const float* d_b2, int32_t F, float* d_pred, void* stream);

/*
 * The same GEMM with fp16 operands (tcgen05.mma kind::f16, twice the tf32 rate).
 * Every operand row is stored scaled by a power of two so its max |value| lies in
 * [2^13, 2^14): fp16 then keeps tf32's 10-bit mantissa with no overflow, and the
 * epilogue undoes the scaling exactly.  d_W1T_h [F][hidden][in] fp16 bits with
 * per-filter exponents d_wexp [F] (lf_filter_rows_to_f16 over W1T viewed as F x m*m
 * rows); the queries are converted inside the call.  m in {64, 128, 192, 256}.
 */
int lf_filter_predict_f16(const float* d_queries, int64_t Q, int32_t m,
                          const uint16_t* d_W1T_h, const int32_t* d_wexp, const float* d_b1,
                          const float* d_W2, const float* d_b2, int32_t F, float* d_pred,
                          void* stream);
/* fp32 rows [rows][m] -> fp16 bits scaled by 2^-exps[r] (max |value| in [2^13, 2^14)). */
int lf_filter_rows_to_f16(const float* d_X, int64_t rows, int32_t m, uint16_t* d_out,
                          int32_t* d_exps, void* stream);

/*
 * Predictions for an explicit list of (query, filter) pairs on the tensor cores:
 * pairs are bucketed by filter, their query rows gathered, and one tcgen05 tile
 * list evaluates them -- bit-identical to the same pairs of lf_filter_predict_tc
 * (_tc) / lf_filter_predict_f16 (_f16: the fp16 pack, query rows gathered straight
 * from the fp16 query matrix with coalesced cp.async -- the kernel of lf_search's in-search
 * inference).  d_out [P] (fp64 of the fp32 prediction).
 */
int lf_filter_predict_pairs_f16(const float* d_queries, int64_t Q, int32_t m, const uint16_t* d_W1T_h,
                                const int32_t* d_wexp, const float* d_b1, const float* d_W2, const float* d_b2,
                                int32_t F, const int32_t* d_pair_q, const int32_t* d_pair_f, int64_t P,
                                double* d_out, void* stream);
int lf_filter_predict_pairs_tc(const float* d_queries, int32_t m, const float* d_W1T, const float* d_b1,
                               const float* d_W2, const float* d_b2, int32_t F, const int32_t* d_pair_q,
                               const int32_t* d_pair_f, int64_t P, double* d_out, void* stream);

/*
 * Exact query x leaf minimum distance (direct form, fp64 accumulation).
 * Replaces batch_distances(...).min(axis=1) (series.py:127-139) as used by
 * collect_targets (traingen.py:175-188) and collect_local_targets (:138).
 *   d_leaf_sel [S]: leaf slots; output d_dl [Q][S] (row stride ldd >= S).
 */
int lf_leaf_min_dist(const float* d_queries, int64_t Q, const lf_index* idx,
                     const int32_t* d_leaf_sel, int32_t S, double* d_dl, int64_t ldd,
                     void* stream);

/*
 * Same, but queries come in groups that are each compared with ONE leaf
 * (collect_local_targets, traingen.py:135-144): group g = queries
 * [h_qptr[g], h_qptr[g+1]) against leaf slot h_group_leaf[g].  h_* are host
 * arrays (n_groups+1 / n_groups entries).  Output d_dl [Q].
 */
int lf_local_min_dist(const float* d_queries, const lf_index* idx, const int64_t* h_qptr,
                      const int32_t* h_group_leaf, int32_t n_groups, double* d_dl,
                      void* stream);

/*
 * Tensor-core versions of the two calls above (m in {32, ..., 256}): tf32
 * tcgen05 GEMM for q . x with a rigorous per-pair error bound, then an exact fp64
 * re-check of the rows that can still be the minimum -- results are the exact
 * fp64 direct-form minima (same terms as lf_leaf_min_dist, another summation
 * order, so equal to ~1 ulp).  Leaf selection and
 * groups are HOST arrays here.
 */
int lf_leaf_min_dist_tc(const float* d_queries, int64_t Q, const lf_index* idx,
                        const int32_t* h_leaf_sel, int32_t S, double* d_dl, int64_t ldd,
                        void* stream);
int lf_local_min_dist_tc(const float* d_queries, const lf_index* idx, const int64_t* h_qptr,
                         const int32_t* h_group_leaf, int32_t n_groups, double* d_dl, void* stream);

/*
 * Same two calls on the INT8 tensor cores (tcgen05.mma.kind::i8) over the
 * collection's int8 shadow (lf_quantize_rows; m in {128, 256}): exact int32 code
 * dot products give a rigorous interval for every (query, row) distance, and only
 * rows that can still be a leaf minimum are re-checked EXACTLY in fp64 from the
 * fp32 rows -- results are the exact fp64 direct-form minima (same terms as
 * lf_leaf_min_dist, another summation order, so equal to ~1 ulp).
 */
int lf_leaf_min_dist_q8(const float* d_queries, int64_t Q, const lf_index* idx,
                        const int32_t* h_leaf_sel, int32_t S, double* d_dl, int64_t ldd,
                        void* stream);
int lf_local_min_dist_q8(const float* d_queries, const lf_index* idx, const int64_t* h_qptr,
                         const int32_t* h_group_leaf, int32_t n_groups, double* d_dl, void* stream);

/*
 * Full distance matrix between queries and an arbitrary row block
 * (series.batch_distances, series.py:127-139). d_block [B][m], out [Q][B].
 */
int lf_batch_distances(const float* d_queries, int64_t Q, const float* d_block, int64_t B,
                       int32_t m, double* d_out, void* stream);

/*
 * Native index build (tree.build_index, tree.py:164-189), bit-identical node
 * table.  Host memory.  Opaque handle protocol:
 *   h = lf_tree_build(values, n, m, n_seg, max_leaf_size, n_threads)
 *   lf_tree_info(h, &n_nodes, &n_leaves)
 *   lf_tree_export(h, ...)   (arrays sized by lf_tree_info; members sized n)
 *   lf_tree_free(h)
 */
typedef struct lf_tree lf_tree;
lf_tree* lf_tree_build(const float* h_values, int64_t n, int32_t m, int32_t n_seg,
                       int64_t max_leaf_size, int32_t n_threads);
int lf_tree_info(const lf_tree* t, int32_t* n_nodes, int32_t* n_leaves);
int lf_tree_export(const lf_tree* t, double* env_min /*[n_nodes][n_seg]*/,
                   double* env_max, int32_t* left, int32_t* right, int32_t* split_seg,
                   double* split_thr, int64_t* size, int8_t* oversized,
                   int64_t* member_ptr /*[n_nodes+1]*/, int64_t* members /*[n]*/);
void lf_tree_free(lf_tree* t);

/* Same build from precomputed segment means (host fp64 [n][n_seg], e.g. from
 * lf_paa_device): the collection itself never has to visit the host. */
lf_tree* lf_tree_build_from_summaries(const double* h_summs, int64_t n, int32_t n_seg,
                                      int64_t max_leaf_size);

/* Segment means of device rows (summarize_matrix, summarize.py:52-56), numpy order. */
int lf_paa_device(const float* d_values, int64_t n, int32_t m, int32_t n_seg, double* d_out,
                  void* stream);

/*
 * Memory-lean LEAF-format loader (series.py:190-215 _save_matrix / _load_matrix;
 * SURVEY §8(f)3).  The payload streams through a few pinned host buffers into HBM
 * (pread by n_threads host threads, H2D, per-chunk kernels); host memory stays
 * O(n_threads x 32 MB) instead of the reference's fp32 + fp64 copies (F7).
 *   lf_leaf_header   -- _load_matrix's header checks; LF_EFORMAT with the
 *                       reference's message and *err_offset (FormatError.offset)
 *   lf_leaf_paa_file -- pass 1: segment means [n][n_seg] (lf_paa_device order) into
 *                       d_summ; the rows are not kept
 *   lf_leaf_load     -- pass 2: row i -> d_X[d_pos[i]] (d_pos NULL = identity,
 *                       d_pos[i] < 0 = skipped: another rank's leaf), i.e. straight
 *                       into the leaf-contiguous layout of lf_index.d_X
 *   lf_leaf_save     -- write device rows [n][m] as a LEAF file (series.py:190-195)
 * The loaders reject non-finite values (series.py:65-66) with LF_EINVAL.
 */
int lf_leaf_header(const char* path, int64_t* n, int32_t* m, int64_t* err_offset);
int lf_leaf_paa_file(const char* path, int64_t n, int32_t m, int32_t n_seg, double* d_summ,
                     int32_t n_threads, void* stream);
int lf_leaf_load(const char* path, int64_t n, int32_t m, const int64_t* d_pos, float* d_X,
                 int32_t n_threads, void* stream);
int lf_leaf_save(const char* path, const float* d_X, int64_t n, int32_t m, void* stream);

/* Build the int8 shadow used by the bounded leaf scan: per row r, scale_r =
 * max|x| / 127, code = rint(x / scale_r), xx_r = sum code^2, and the exact
 * quantisation error norm qerr_r = ||scale_r * code - x||_2 (fp64, rounded up),
 * packed as d_qmeta[r] = {scale_r, xx_r, qerr_r, 0} (16 B per row, so one bulk
 * copy stages a block of rows).  Then for any query,
 * | ||x - q|| - ||scale*code - q|| | <= qerr_r. */
int lf_quantize_rows(const float* d_X, int64_t n, int32_t m, int8_t* d_X8, float* d_qmeta,
                     void* stream);


/*
 * Conformal auto-tuner fitting (conformal.py:171-198 simulate_search, for R offset
 * vectors at once): the calibration skeleton in visit order -- bounds, leaf minimum
 * distances, predictions (NaN: no filter), filter slots (-1: none), all [nq][L] --
 * and offsets [R][F]; out [R][nq] = the distance each calibration query's filtered
 * search reaches.  Bit-identical to the host replay (comparisons and minima only).
 */
int lf_replay_offsets(const double* d_lb, const double* d_dl, const double* d_pred, const int32_t* d_slot,
                      int64_t nq, int32_t L, const double* d_offsets, int64_t R, int32_t F, double* d_out,
                      void* stream);

/* Segment means for host rows (summarize_matrix, summarize.py:52-56), numpy order. */
int lf_paa_host(const float* h_values, int64_t n, int32_t m, int32_t n_seg, double* h_out,
                int32_t n_threads);

#ifdef __cplusplus
}
#endif
#endif /* LEAFI_B200_H */
