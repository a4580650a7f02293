// K1: query segment means + node lower bounds over SoA envelopes (HBM-bound).
//
// Reference: summarize.py:44-56 (segment means), summarize.py:97-107 (search
// bound, np.dot -> one fp64 FMA chain over segments), summarize.py:114-122
// (batched bound used by traingen, einsum -> sequential sum of (g*g)*w).
// Both orders are reproduced bit-for-bit so visit orders and counters match.
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "bounds.cuh"
#include "common.cuh"

namespace lf {

// One thread per (query, segment).  zero2 (nullable, [2 Q]): the leaf-bound range
// words lb_tile_kernel accumulates into, zeroed here (no memset node in the graphs).
__global__ void paa_kernel(const float* __restrict__ q, int64_t Q, lf_index idx,
                           double* __restrict__ qsumm, unsigned* __restrict__ zero2 = nullptr) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (zero2 != nullptr && t < 2 * Q) zero2[t] = 0u;
    if (t >= Q * idx.n_seg) return;
    int64_t qi = t / idx.n_seg;
    int s = (int)(t - qi * idx.n_seg);
    qsumm[t] = segment_mean(q + qi * idx.m, idx.seg_start[s], idx.seg_width[s]);
}

// One thread per (query, segment): EAPCA summary, means then sds ([Q][2 n_seg]).
__global__ void eapca_kernel(const float* __restrict__ q, int64_t Q, lf_index idx, double* __restrict__ out) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= Q * idx.n_seg) return;
    const int64_t qi = t / idx.n_seg;
    const int s = (int)(t - qi * idx.n_seg);
    const float* row = q + qi * idx.m;
    const double mu = segment_mean(row, idx.seg_start[s], idx.seg_width[s]);
    out[qi * 2 * idx.n_seg + s] = mu;
    out[qi * 2 * idx.n_seg + idx.n_seg + s] = segment_sd(row, idx.seg_start[s], idx.seg_width[s], mu);
}

// max(mn - q, q - mx, 0) (summarize.py:103-104): mn <= mx, so at most one of the
// two differences is positive -- selects instead of fmax, bit-identical.  The sign
// tests read the high words on the integer pipe (no DSETP on the fp64 pipe): hi > 0
// is x > 0 except for positive subnormals with a zero high word, whose square
// underflows to an exact 0 in every bound mode, so the bound is unchanged.
__device__ __forceinline__ double env_gap(double mn, double mx, double q) {
    const double a = mn - q, b = q - mx;
    return __double2hiint(a) > 0 ? a : (__double2hiint(b) > 0 ? b : 0.0);
}

// The per-segment term of each bound mode, folded into acc:
//   0: np.dot(widths * gap, gap) -- one FMA chain (search path, summarize.py:107)
//   1: einsum("qns,qns,s")        -- sequential (g * g) * w (traingen, summarize.py:114-122)
//   2: EAPCA                      -- acc + w * (gm^2 + gs^2), no FMA (oracle eapca definition)
template <int MODE>
__device__ __forceinline__ double bound_term(double acc, double w, double gm, double gs) {
    if (MODE == 0) return __fma_rn(__dmul_rn(w, gm), gm, acc);
    if (MODE == 1) return __dadd_rn(acc, __dmul_rn(__dmul_rn(gm, gm), w));
    return __dadd_rn(acc, __dmul_rn(w, __dadd_rn(__dmul_rn(gm, gm), __dmul_rn(gs, gs))));
}

// lb[q][node] for nodes of one query row; query summaries staged in smem
// (any n_seg; MODE 2 reads means then sds, [2 n_seg] per query).
template <int MODE>
__global__ void lb_kernel(const double* __restrict__ qsumm, int64_t Q, int n_seg, lf_index idx,
                          const double* __restrict__ env_min, const double* __restrict__ env_max,
                          const double* __restrict__ sd_min, const double* __restrict__ sd_max,
                          int n_env, double* __restrict__ lb) {
    __shared__ double qs[2 * LF_MAX_SEG];
    __shared__ double ws[LF_MAX_SEG];
    const int qw = MODE == 2 ? 2 * n_seg : n_seg;
    for (int64_t qi = blockIdx.y; qi < Q; qi += gridDim.y) {
        __syncthreads();
        if (threadIdx.x < qw) qs[threadIdx.x] = qsumm[qi * qw + threadIdx.x];
        if (threadIdx.x < n_seg) ws[threadIdx.x] = (double)idx.seg_width[threadIdx.x];
        __syncthreads();
        for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < n_env;
             node += gridDim.x * blockDim.x) {
            double acc = 0.0;
            for (int s = 0; s < n_seg; ++s) {
                const double gm = env_gap(env_min[(int64_t)s * n_env + node], env_max[(int64_t)s * n_env + node],
                                          qs[s]);
                const double gs = MODE == 2 ? env_gap(sd_min[(int64_t)s * n_env + node],
                                                      sd_max[(int64_t)s * n_env + node], qs[n_seg + s])
                                            : 0.0;
                acc = bound_term<MODE>(acc, ws[s], gm, gs);
            }
            lb[qi * n_env + node] = sqrt(acc);
        }
    }
}

// lb[q][node] for QT queries x 128 nodes per CTA: each thread holds its node's
// envelope (n_seg <= 8) in registers and reuses it for QT queries, so the
// envelopes are read from L2 once per QT queries instead of once per query.
// Same arithmetic as lb_kernel (bit-identical bounds).  With qmax / qmin set it
// also records, per query, the range of its leaf bounds as float bits (rounded:
// the leaf-order kernel only needs it to spread its buckets); qmin holds the
// complement of the minimum's bits.
constexpr int LBT_NODES = 128;
constexpr int LBT_Q = 16;
constexpr int LBT_SEG = 8;

// NS > 0: n_seg known at compile time (no per-segment guards; 246 -> fewer issued
// instructions per (query, node) at n_seg = 8), 0: any n_seg <= 8.
template <int MODE, int NS = 0>
__global__ void __launch_bounds__(LBT_NODES, MODE == 2 ? 2 : 4)
    lb_tile_kernel(const double* __restrict__ qsumm, int64_t Q, int ns_, lf_index idx,
                   const double* __restrict__ env_min, const double* __restrict__ env_max,
                   const double* __restrict__ sd_min, const double* __restrict__ sd_max, int n_env,
                   double* __restrict__ lb, unsigned* __restrict__ qmax, unsigned* __restrict__ qmin,
                   double* __restrict__ plb, int* __restrict__ pnode) {
    constexpr int QW = MODE == 2 ? 2 * LBT_SEG : LBT_SEG;
    const int ns = NS > 0 ? NS : ns_;
    __shared__ double qs[LBT_Q][QW];
    __shared__ double ws[LBT_SEG];
    const int node = blockIdx.x * LBT_NODES + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int64_t q0 = (int64_t)blockIdx.y * LBT_Q;
    const int qw = MODE == 2 ? 2 * ns : ns;
    for (int i = threadIdx.x; i < LBT_Q * qw; i += LBT_NODES) {
        const int qq = i / qw, sg = i - qq * qw;
        const int col = MODE == 2 && sg >= ns ? LBT_SEG + (sg - ns) : sg;
        qs[qq][col] = q0 + qq < Q ? qsumm[(q0 + qq) * qw + sg] : 0.0;
    }
    if (threadIdx.x < ns) ws[threadIdx.x] = (double)idx.seg_width[threadIdx.x];
    __syncthreads();
    const bool valid = node < n_env;
    const bool isl = qmax != nullptr && valid && __ldg(idx.d_node_leaf + node) >= 0;
    double mn[LBT_SEG], mx[LBT_SEG], smn[MODE == 2 ? LBT_SEG : 1], smx[MODE == 2 ? LBT_SEG : 1];
#pragma unroll
    for (int sg = 0; sg < LBT_SEG; ++sg) {
        mn[sg] = (valid && sg < ns) ? __ldg(env_min + (int64_t)sg * n_env + node) : 0.0;
        mx[sg] = (valid && sg < ns) ? __ldg(env_max + (int64_t)sg * n_env + node) : 0.0;
        if constexpr (MODE == 2) {
            smn[sg] = (valid && sg < ns) ? __ldg(sd_min + (int64_t)sg * n_env + node) : 0.0;
            smx[sg] = (valid && sg < ns) ? __ldg(sd_max + (int64_t)sg * n_env + node) : 0.0;
        }
    }
    const int qn = (int)min((int64_t)LBT_Q, Q - q0);
    for (int qq = 0; qq < qn; ++qq) {
        double acc = 0.0;
#pragma unroll
        for (int sg = 0; sg < LBT_SEG; ++sg) {
            if (sg < ns) {
                const double gm = env_gap(mn[sg], mx[sg], qs[qq][sg]);
                double gs = 0.0;
                if constexpr (MODE == 2) gs = env_gap(smn[sg], smx[sg], qs[qq][LBT_SEG + sg]);
                acc = bound_term<MODE>(acc, ws[sg], gm, gs);
            }
        }
        const double v = sqrt(acc);
        if (valid) lb[(q0 + qq) * n_env + node] = v;
        if (qmax != nullptr) {
            const unsigned fb = __float_as_uint((float)v);
            const unsigned hi = __reduce_max_sync(0xffffffffu, isl ? fb : 0u);
            const unsigned lo = __reduce_min_sync(0xffffffffu, isl ? fb : 0xffffffffu);
            if (lane == 0 && lo != 0xffffffffu) {
                atomicMax(qmax + q0 + qq, hi);
                atomicMax(qmin + q0 + qq, ~lo);     // complemented: both start at 0, one memset
            }
            if (plb != nullptr) {       // the warp's minimum (lb, node) over its leaves, exactly:
                // bound bits order like the non-negative values; three integer reductions
                const unsigned long long b = (unsigned long long)__double_as_longlong(v);
                const unsigned bh = (unsigned)(b >> 32), bl = (unsigned)b;
                const unsigned mh = __reduce_min_sync(0xffffffffu, isl ? bh : 0xffffffffu);
                const bool c1 = isl && bh == mh;
                const unsigned ml = __reduce_min_sync(0xffffffffu, c1 ? bl : 0xffffffffu);
                const bool c2 = c1 && bl == ml;
                const unsigned mn = __reduce_min_sync(0xffffffffu, c2 ? (unsigned)node : 0xffffffffu);
                if (lane == 0 && node < n_env) {                 // warps past the last node own no slot
                    const int W = (n_env + 31) >> 5;
                    const int64_t at = (q0 + qq) * W + (node >> 5);
                    plb[at] = mn == 0xffffffffu ? kInf : __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
                    pnode[at] = mn == 0xffffffffu ? -1 : (int)mn;
                }
            }
        }
    }
}

int launch_bounds(const float* d_q, int64_t Q, const lf_index& idx, const double* env_min,
                  const double* env_max, int n_env, int mode, double* d_qsumm, double* d_lb,
                  cudaStream_t st, unsigned* d_qmax, unsigned* d_qmin, const double* sd_min,
                  const double* sd_max, double* d_plb, int* d_pnode) {
    if (Q == 0) return LF_OK;
    const bool tiled = n_env > 0 && idx.n_seg <= LBT_SEG && (Q + LBT_Q - 1) / LBT_Q <= 65535;
    // the range words: zeroed by paa_kernel when contiguous ([qmax | qmin], the callers' layout)
    const bool zero_in_paa = tiled && d_qmax != nullptr && d_qmin == d_qmax + Q && mode != 2;
    {
        int64_t n = Q * idx.n_seg;
        if (zero_in_paa) n = std::max<int64_t>(n, 2 * Q);
        int thr = 256;
        if (mode == 2)
            eapca_kernel<<<(unsigned)((n + thr - 1) / thr), thr, 0, st>>>(d_q, Q, idx, d_qsumm);
        else
            paa_kernel<<<(unsigned)((n + thr - 1) / thr), thr, 0, st>>>(d_q, Q, idx, d_qsumm,
                                                                        zero_in_paa ? d_qmax : nullptr);
        LF_CUDA(cudaGetLastError());
    }
    if (n_env == 0) return LF_OK;
    if (tiled) {
        if (d_qmax != nullptr && !zero_in_paa) {
            LF_CUDA(cudaMemsetAsync(d_qmax, 0, sizeof(unsigned) * Q, st));
            LF_CUDA(cudaMemsetAsync(d_qmin, 0, sizeof(unsigned) * Q, st));
        }
        dim3 grid((unsigned)((n_env + LBT_NODES - 1) / LBT_NODES), (unsigned)((Q + LBT_Q - 1) / LBT_Q));
#define LF_TILE(M, N) lb_tile_kernel<M, N><<<grid, LBT_NODES, 0, st>>>(d_qsumm, Q, idx.n_seg, idx, env_min, env_max, \
                                                                      sd_min, sd_max, n_env, d_lb, d_qmax, d_qmin, \
                                                                      d_plb, d_pnode)
        if (mode == 0 && idx.n_seg == LBT_SEG) LF_TILE(0, LBT_SEG);
        else if (mode == 0) LF_TILE(0, 0);
        else if (mode == 1) LF_TILE(1, 0);
        else LF_TILE(2, 0);
#undef LF_TILE
        LF_CUDA(cudaGetLastError());
        return LF_OK;
    }
    LF_REQUIRE(d_qmax == nullptr, "leaf bound ranges need n_seg <= 8");
    dim3 block(256);
    dim3 grid((unsigned)((n_env + 255) / 256), (unsigned)(Q < 65535 ? Q : 65535));
#define LF_GEN(M) lb_kernel<M><<<grid, block, 0, st>>>(d_qsumm, Q, idx.n_seg, idx, env_min, env_max, sd_min, sd_max, \
                                                     n_env, d_lb)
    if (mode == 0) LF_GEN(0);
    else if (mode == 1) LF_GEN(1);
    else LF_GEN(2);
#undef LF_GEN
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

__global__ void iota_rows_kernel(int* __restrict__ v, int64_t Q, int n, int* __restrict__ offs) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < Q * n) v[t] = (int)(t % n);
    if (t <= Q) offs[t] = (int)(t * n);
}

// ------------------------------------------------------------ leaf order ----
// The record of visit position p of query q (bounds.cuh): its bound, the gap
// bound before it, leaf slot | filter flag, and pred - offset of the filter.
// ITEMS positions per thread, the dependent loads (node -> leaf -> filter ->
// prediction, offset) issued level by level so their latencies overlap.
template <int ITEMS>
__device__ __forceinline__ void put_records(const OrderArgs& o, const lf_index& idx, int64_t q, int Lr, int L,
                                            const int (&p)[ITEMS], const int (&node)[ITEMS],
                                            const double (&lbv)[ITEMS], const double (&gapv)[ITEMS]) {
    const bool filt = idx.d_leaf_filter != nullptr && (o.pred != nullptr || o.pred64 != nullptr || o.lazy);
    int leaf[ITEMS], fs[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) leaf[i] = p[i] < L ? __ldg(idx.d_node_leaf + node[i]) : -1;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) fs[i] = (filt && leaf[i] >= 0) ? __ldg(idx.d_leaf_filter + leaf[i]) : -1;
    double pv[ITEMS], off[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        pv[i] = 0.0;
        off[i] = 0.0;
        if (fs[i] >= 0 && !o.lazy) {
            pv[i] = o.pred64 != nullptr ? o.pred64[q * o.F + fs[i]] : (double)o.pred[q * o.F + fs[i]];
            off[i] = o.offset[fs[i]];
        }
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        if (p[i] >= L) continue;
        const int64_t at = q * Lr + p[i];
        int rec = leaf[i];
        double a = -kInf;
        if (fs[i] >= 0) {
            rec |= LF_REC_HASF;
            a = o.lazy ? __longlong_as_double(0x7ff8000000000000LL) : pv[i] - off[i];
        }
        o.lbs[at] = lbv[i];
        o.gap[at] = gapv[i];
        o.leafo[at] = rec;
        // in-search inference writes adj of every pair the walk can reach before the walk
        // reads it (plan reads adj only below pcount), so the lazy order leaves it unset
        if (!o.lazy) o.adj[at] = a;
        if (o.order != nullptr) o.order[at] = node[i];
    }
}

// One CTA per query (trees of <= 8192 nodes, <= 4096 leaf slots); the node
// bounds come from the L2-resident bound matrix and the range of the query's
// leaf bounds from lb_tile_kernel.  A counting sort:
//   1. every leaf is staged in shared memory (warp-aggregated slots, any order)
//      and counted in bucket floor((lb - lo) * (NB - 1) / (hi - lo)) -- a map
//      monotone in lb, so every leaf of a lower bucket precedes every leaf of a
//      higher one in (lb, id) order;
//   2. one scan of the counts, an atomic scatter into the buckets;
//   3. each bucket (about one leaf on average) is put in exact (lb, node id)
//      order: insertion sort, or -- buckets of more than LO_BIG leaves, bounds
//      clustered far below their spread -- a warp computes every element's rank
//      (pairs (lb, id) are distinct, so ranks are a permutation);
//   4. every non-leaf node finds the first leaf after it in (lb, id) order inside
//      its own bucket (or at the next bucket's start) and raises that leaf's gap
//      bound to its own bound (atomicMax on the bits: bounds are non-negative).
// Global round trips: one for the leaves' bounds, one for the non-leaves', and
// the record gathers.
// Two shapes of the same kernel (LoCfg):
//   small: <= 8192 nodes / 4096 leaf slots, 512 threads, everything in shared memory;
//   big:   <= 32768 nodes / 16384 leaf slots, 1024 threads, the bucket counts in
//          shared memory and the staged / sorted leaves and gap bits in a per-query
//          global scratch (L2) -- the trees of BASELINE config 5, without a library sort.
template <bool BIG>
struct LoCfg {
    static constexpr int THREADS = BIG ? 1024 : 512;
    static constexpr int WARPS = THREADS / 32;
    static constexpr int LEAF_ITEMS = BIG ? 16 : 8;
    static constexpr int MAX_LEAVES = THREADS * LEAF_ITEMS;
    static constexpr int MAX_NI = BIG ? 32 : 16;          // node items per thread (flags: 32 bits)
    static constexpr int NB = BIG ? 16384 : 4096;         // buckets of the counting sort
    static constexpr int BIG_LIST = MAX_LEAVES / 33 + 1;
    static constexpr int SMEM_LEAVES = BIG ? 1 : MAX_LEAVES;
};
constexpr int LO_THREADS = LoCfg<false>::THREADS;       // (the small shape's limits, used by callers)
constexpr int LO_MAX_LEAVES = LoCfg<false>::MAX_LEAVES;
constexpr int LO_MAX_NI = LoCfg<false>::MAX_NI;
constexpr int LO_BIG = 32;

template <bool BIG>
struct LoSmem {
    using C = LoCfg<BIG>;
    union {
        struct {
            double lb[C::SMEM_LEAVES];             // staged leaves (any order)
            int node[C::SMEM_LEAVES];
        } st;
        unsigned long long gap[C::SMEM_LEAVES];    // after the sort: gap bound bits per position
    } u;
    double lb[C::SMEM_LEAVES];                     // leaves in (lb, node id) order
    int node[C::SMEM_LEAVES];
    int bend[C::NB];                               // bucket counts -> starts -> ends
    int big[C::BIG_LIST];
    int nstage, nbig;
    double tlb_w[C::WARPS];                        // pruned orders: the first leaf past thr
    int tnode_w[C::WARPS];
    double tlb;
    int tnode;
    int wsum[C::WARPS];
};

// Global scratch of the big shape, [Q][n_leaves] each.
struct LoScratch {
    double* st_lb;
    int* st_node;
    double* lb;
    int* node;
    unsigned long long* gap;
};

template <int NB>
__device__ __forceinline__ int lo_bucket(double v, double lo, double scale) {
    const double k = floor((v - lo) * scale);
    return k <= 0.0 ? 0 : (k >= (double)(NB - 1) ? NB - 1 : (int)k);
}

__device__ __forceinline__ bool lo_less(double la, int na, double lb_, int nb) {
    return la < lb_ || (la == lb_ && na < nb);
}

template <int NI, bool BIG>
__global__ void __launch_bounds__(LoCfg<BIG>::THREADS, BIG ? 1 : 2)
    leaf_order_kernel(const double* __restrict__ lb, lf_index idx, const unsigned* __restrict__ qmax,
                      const unsigned* __restrict__ qmin, OrderArgs o, LoScratch gs) {
    using C = LoCfg<BIG>;
    constexpr int T = C::THREADS, NB = C::NB;
    extern __shared__ __align__(16) uint8_t lo_smem[];
    LoSmem<BIG>& sm = *reinterpret_cast<LoSmem<BIG>*>(lo_smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned below = (1u << lane) - 1u;
    const int64_t q = blockIdx.x;
    const int Nn = idx.n_nodes;
    const int Lr = idx.n_leaves;
    // staged / sorted leaves and gap bits: shared memory, or this query's global scratch
    double* st_lb = BIG ? gs.st_lb + q * Lr : sm.u.st.lb;
    int* st_node = BIG ? gs.st_node + q * Lr : sm.u.st.node;
    double* s_lb = BIG ? gs.lb + q * Lr : sm.lb;
    int* s_node = BIG ? gs.node + q * Lr : sm.node;
    unsigned long long* gapb = BIG ? gs.gap + q * Lr : sm.u.gap;
    const double* lbq = lb + q * Nn;
    double thr = kInf;                                   // pruned orders: leaves past thr are not records
    if (o.prune) {
        double b = o.seed != nullptr ? (double)__uint_as_float(o.seed[q])
                                     : (o.top_n[q] == o.k ? o.top_d[q * o.k + o.k - 1] : kInf);
        if (o.bound != nullptr) b = fmin(b, o.bound[q]);
        thr = b * o.f;
    }
    const double lo = (double)__uint_as_float(~qmin[q]);
    const double span = fmin((double)__uint_as_float(qmax[q]), thr) - lo;
    const double scale = (span > 0.0 && span < kInf) ? (double)(NB - 1) / span : 0.0;
    double tv = kInf;                                    // this thread's first leaf past thr
    int tn = 0x7fffffff;
    for (int b = tid; b < NB; b += T) sm.bend[b] = 0;
    if (tid == 0) {
        sm.nstage = 0;
        sm.nbig = 0;
    }
    __syncthreads();
    // 1. stage the leaves and count them per bucket (loads of 8 items in flight together)
    unsigned flags = 0;
#pragma unroll
    for (int h = 0; h < NI; h += 8) {
        int nl[8];
        double v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int node = (h + e) * T + tid;
            nl[e] = node < Nn ? __ldg(idx.d_node_leaf + node) : -1;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int node = (h + e) * T + tid;
            v[e] = nl[e] >= 0 ? lbq[node] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const bool isl = nl[e] >= 0;
            if (isl) flags |= 1u << (h + e);
            const bool stage = isl && v[e] <= thr;
            if (isl && !stage && lo_less(v[e], (h + e) * T + tid, tv, tn)) {
                tv = v[e];
                tn = (h + e) * T + tid;
            }
            const unsigned bm = __ballot_sync(0xffffffffu, stage);
            if (bm == 0) continue;
            int base = 0;
            if (lane == 0) base = atomicAdd(&sm.nstage, __popc(bm));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (stage) {
                const int pos = base + __popc(bm & below);
                st_lb[pos] = v[e];
                st_node[pos] = (h + e) * T + tid;
                atomicAdd(&sm.bend[lo_bucket<NB>(v[e], lo, scale)], 1);
            }
        }
    }
    if (o.prune) {                                       // the first leaf past thr: block minimum
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, tv, d);
            const int on = __shfl_xor_sync(0xffffffffu, tn, d);
            if (lo_less(ov, on, tv, tn)) { tv = ov; tn = on; }
        }
        if (lane == 0) { sm.tlb_w[warp] = tv; sm.tnode_w[warp] = tn; }
    }
    __syncthreads();
    const int L = sm.nstage;
    if (o.prune && tid == 0) {
        double bv = kInf;
        int bn = 0x7fffffff;
        for (int w = 0; w < C::WARPS; ++w)
            if (lo_less(sm.tlb_w[w], sm.tnode_w[w], bv, bn)) { bv = sm.tlb_w[w]; bn = sm.tnode_w[w]; }
        sm.tlb = bv;
        sm.tnode = bn == 0x7fffffff ? -1 : bn;
    }
    // 2. exclusive scan of the counts (PT consecutive buckets per thread), then scatter
    {
        constexpr int PT = NB / T;
        int c[PT], sum = 0;
#pragma unroll
        for (int j = 0; j < PT; ++j) {
            c[j] = sm.bend[tid * PT + j];
            sum += c[j];
        }
        int incl = sum;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
        }
        if (lane == 31) sm.wsum[warp] = incl;
        __syncthreads();
        int run = incl - sum;
        for (int w = 0; w < warp; ++w) run += sm.wsum[w];
#pragma unroll
        for (int j = 0; j < PT; ++j) {
            sm.bend[tid * PT + j] = run;
            run += c[j];
        }
    }
    __syncthreads();
    for (int p = tid; p < L; p += T) {
        const double v = st_lb[p];
        const int pos = atomicAdd(&sm.bend[lo_bucket<NB>(v, lo, scale)], 1);   // start -> end
        s_lb[pos] = v;
        s_node[pos] = st_node[p];
    }
    __syncthreads();
    // 3. exact (lb, node id) order inside each bucket
#pragma unroll
    for (int j = 0; j < NB / T; ++j) {
        const int b = j * T + tid;
        const int s0 = b == 0 ? 0 : sm.bend[b - 1], e0 = sm.bend[b];
        if (e0 - s0 > LO_BIG) {
            const int t = atomicAdd(&sm.nbig, 1);
            if (t < C::BIG_LIST) sm.big[t] = b;
            continue;
        }
        for (int a = s0 + 1; a < e0; ++a) {
            const double la = s_lb[a];
            const int na = s_node[a];
            int c = a - 1;
            while (c >= s0 && !lo_less(s_lb[c], s_node[c], la, na)) {
                s_lb[c + 1] = s_lb[c];
                s_node[c + 1] = s_node[c];
                --c;
            }
            s_lb[c + 1] = la;
            s_node[c + 1] = na;
        }
    }
    __syncthreads();
    if (sm.nbig > 0) {                                   // rare: a warp ranks each big bucket
        for (int t = warp; t < sm.nbig; t += C::WARPS) {
            const int b = sm.big[t];
            const int s0 = b == 0 ? 0 : sm.bend[b - 1], e0 = sm.bend[b];
            for (int i = s0 + lane; i < e0; i += 32) {
                const double li = s_lb[i];
                const int ni = s_node[i];
                int r = 0;
                for (int j2 = s0; j2 < e0; ++j2) r += lo_less(s_lb[j2], s_node[j2], li, ni);
                st_lb[s0 + r] = li;                      // the staging area is free now
                st_node[s0 + r] = ni;
            }
            __syncwarp();
            for (int i = s0 + lane; i < e0; i += 32) {
                s_lb[i] = st_lb[i];
                s_node[i] = st_node[i];
            }
        }
        __syncthreads();
    }
    const bool has_term = o.prune && sm.tnode >= 0;      // (visible: written before the last barriers)
    for (int p = tid; p < L + (has_term ? 1 : 0); p += T) gapb[p] = 0ull;
    __syncthreads();
    // 4. gap bounds of the non-leaf nodes
#pragma unroll
    for (int h = 0; h < NI; h += 8) {
        double v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int node = (h + e) * T + tid;
            v[e] = (node < Nn && !((flags >> (h + e)) & 1u)) ? lbq[node] : -1.0;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            if (v[e] < 0.0) continue;
            const int node = (h + e) * T + tid;
            if (v[e] > thr && !(has_term && lo_less(v[e], node, sm.tlb, sm.tnode))) continue;   // past the end
            const int b = lo_bucket<NB>(v[e], lo, scale);
            int p = b == 0 ? 0 : sm.bend[b - 1];
            const int e0 = sm.bend[b];
            while (p < e0 && lo_less(s_lb[p], s_node[p], v[e], node)) ++p;
            if (p < L || (p == L && has_term))
                atomicMax(&gapb[p], (unsigned long long)__double_as_longlong(v[e]));
        }
    }
    __syncthreads();
    // 5. records, 4 positions per thread at a time
#pragma unroll
    for (int h = 0; h < C::LEAF_ITEMS; h += 4) {
        int p[4], node[4];
        double lbv[4], gv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            p[e] = (h + e) * T + tid;
            const bool ok = p[e] < L;
            node[e] = ok ? s_node[p[e]] : 0;
            lbv[e] = ok ? s_lb[p[e]] : 0.0;
            gv[e] = ok ? __longlong_as_double((long long)gapb[p[e]]) : 0.0;
        }
        put_records<4>(o, idx, q, Lr, L, p, node, lbv, gv);
    }
    if (tid == 0) {
        if (has_term) {                                  // the terminal record
            const int p1[1] = {L}, n1[1] = {sm.tnode};
            const double l1[1] = {sm.tlb}, g1[1] = {__longlong_as_double((long long)gapb[L])};
            put_records<1>(o, idx, q, Lr, L + 1, p1, n1, l1, g1);
        }
        o.olen[q] = L + (has_term ? 1 : 0);
    }
}

// Any tree size: one warp per query walks the FULL sorted (lb, node id) order
// (CUB segmented sort of the bound matrix), keeps the local leaves in order and
// carries the largest non-leaf bound seen since the previous leaf.
__global__ void leaf_records_kernel(const double* __restrict__ slb, const int* __restrict__ sorder, lf_index idx,
                                    int64_t Q, OrderArgs o) {
    const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= Q) return;
    const unsigned below = (1u << lane) - 1u;
    const int Nn = idx.n_nodes, Lr = idx.n_leaves;
    const double* lbs = slb + q * Nn;
    const int* ord = sorder + q * Nn;
    double carry = 0.0;                                  // largest non-leaf bound after the last leaf
    int outp = 0;
    for (int base = 0; base < Nn; base += 32) {
        const int i = base + lane;
        const bool valid = i < Nn;
        const int node = valid ? ord[i] : 0;
        const double v = valid ? lbs[i] : 0.0;
        const int leaf = valid ? __ldg(idx.d_node_leaf + node) : -1;
        const bool isl = valid && leaf >= 0;
        const bool isn = valid && leaf < 0;
        const unsigned ml = __ballot_sync(0xffffffffu, isl);
        const unsigned mn = __ballot_sync(0xffffffffu, isn);
        const unsigned nl = mn & below, ll = ml & below;
        const int hn = nl ? 31 - __clz(nl) : -1;
        const int hl = ll ? 31 - __clz(ll) : -1;
        const double vn = __shfl_sync(0xffffffffu, v, hn >= 0 ? hn : 0);
        const double g = hn > hl ? vn : (hl >= 0 ? 0.0 : carry);
        const int lastn = mn ? 31 - __clz(mn) : -1;
        const int lastl = ml ? 31 - __clz(ml) : -1;
        const double vlast = __shfl_sync(0xffffffffu, v, lastn >= 0 ? lastn : 0);
        if (isl) {
            const int p1[1] = {outp + __popc(ll)};
            const int n1[1] = {node};
            const double l1[1] = {v}, g1[1] = {g};
            put_records<1>(o, idx, q, Lr, Lr, p1, n1, l1, g1);
        }
        outp += __popc(ml);
        if (lastn > lastl) carry = vlast;
        else if (lastl >= 0) carry = 0.0;
    }
    if (lane == 0) o.olen[q] = outp;
}

template <int NI, bool BIG>
static int launch_leaf_order(const double* d_lb, int64_t Q, const lf_index& idx, const unsigned* qmax,
                             const unsigned* qmin, const OrderArgs& oa, cudaStream_t st) {
    const int bytes = (int)sizeof(LoSmem<BIG>);
    LF_CUDA(smem_optin(leaf_order_kernel<NI, BIG>, bytes));
    Scratch g;                                           // big shape: per-query staging in L2
    LoScratch gs{};
    if (BIG) {
        const size_t per = (size_t)Q * idx.n_leaves;
        LF_CUDA(g.alloc(per * (8 + 4 + 8 + 4 + 8), st));
        gs.st_lb = g.as<double>();
        gs.lb = gs.st_lb + per;
        gs.gap = reinterpret_cast<unsigned long long*>(gs.lb + per);
        gs.st_node = reinterpret_cast<int*>(gs.gap + per);
        gs.node = gs.st_node + per;
    }
    leaf_order_kernel<NI, BIG><<<(unsigned)Q, LoCfg<BIG>::THREADS, bytes, st>>>(d_lb, idx, qmax, qmin, oa, gs);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

bool fused_order_ok(const lf_index& idx, int64_t Q) {
    using B = LoCfg<true>;
    return idx.n_nodes <= B::THREADS * B::MAX_NI && idx.n_leaves <= B::MAX_LEAVES && idx.n_seg <= LBT_SEG &&
           (Q + LBT_Q - 1) / LBT_Q <= 65535 && Q <= 0x7fffffff;
}

static bool small_order(const lf_index& idx) {
    using S = LoCfg<false>;
    return idx.n_nodes <= S::THREADS * S::MAX_NI && idx.n_leaves <= S::MAX_LEAVES;
}

int bounds_phase(const float* d_q, int64_t Q, const lf_index& idx, double* d_qsumm, double* d_lb, unsigned* qmax,
                 unsigned* qmin, double* plb, int* pnode, cudaStream_t st, int* kernels) {
    LF_REQUIRE(fused_order_ok(idx, Q), "bounds_phase: tree too large for the single-CTA leaf order");
    const bool eapca = idx.d_sd_min != nullptr && idx.d_sd_max != nullptr;
    int rc = launch_bounds(d_q, Q, idx, idx.d_env_min, idx.d_env_max, idx.n_nodes, eapca ? 2 : 0, d_qsumm, d_lb, st,
                           qmax, qmin, idx.d_sd_min, idx.d_sd_max, plb, pnode);
    if (rc == LF_OK && kernels) *kernels += 2;
    return rc;
}

int order_phase(const double* d_lb, int64_t Q, const lf_index& idx, const unsigned* qmax, const unsigned* qmin,
                const OrderArgs& oa, cudaStream_t st) {
    if (small_order(idx)) {
        if (idx.n_nodes <= LO_THREADS * 8) return launch_leaf_order<8, false>(d_lb, Q, idx, qmax, qmin, oa, st);
        return launch_leaf_order<16, false>(d_lb, Q, idx, qmax, qmin, oa, st);
    }
    if (idx.n_nodes <= LoCfg<true>::THREADS * 16) return launch_leaf_order<16, true>(d_lb, Q, idx, qmax, qmin, oa, st);
    return launch_leaf_order<32, true>(d_lb, Q, idx, qmax, qmin, oa, st);
}

// Segment means + node bounds + per-query leaf records: the bound matrix
// (lb_tile_kernel) feeds the per-query leaf sort when the tree fits one CTA
// (<= 8192 nodes, <= 4096 leaf slots), else CUB's segmented sort of all nodes
// and the warp-per-query record walk.
int bounds_and_order(const float* d_q, int64_t Q, const lf_index& idx, double* d_qsumm, double* d_lb,
                     const OrderArgs& oa, cudaStream_t st, int* kernels) {
    const int n = idx.n_nodes;
    if (Q == 0 || n == 0) return LF_OK;
    const bool fused = fused_order_ok(idx, Q);
    Scratch range;
    if (fused) LF_CUDA(range.alloc(sizeof(unsigned) * 2 * Q, st));
    unsigned* qmax = fused ? range.as<unsigned>() : nullptr;
    unsigned* qmin = fused ? qmax + Q : nullptr;
    const bool eapca = idx.d_sd_min != nullptr && idx.d_sd_max != nullptr;
    int rc = launch_bounds(d_q, Q, idx, idx.d_env_min, idx.d_env_max, n, eapca ? 2 : 0, d_qsumm, d_lb, st, qmax, qmin,
                           idx.d_sd_min, idx.d_sd_max);
    if (rc) return rc;
    if (kernels) *kernels += 2;
    if (fused) {
        if (kernels) *kernels += 1;
        return order_phase(d_lb, Q, idx, qmax, qmin, oa, st);
    }
    Scratch slb, sord;
    LF_CUDA(slb.alloc(sizeof(double) * Q * n, st));
    LF_CUDA(sord.alloc(sizeof(int) * Q * n, st));
    rc = sort_visit_order(d_lb, Q, n, slb.as<double>(), sord.as<int>(), st);
    if (rc) return rc;
    if (kernels) *kernels += 2;
    leaf_records_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(slb.as<double>(), sord.as<int>(), idx, Q,
                                                                          oa);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

// Per-query stable sort of (lb, node id): the heap pop order of tree.py:256-275
// (child lb >= parent lb and child id > parent id, so the heap is a sort).
int sort_visit_order(const double* d_lb, int64_t Q, int n, double* d_lb_sorted, int* d_order,
                     cudaStream_t st) {
    if (Q == 0 || n == 0) return LF_OK;
    LF_REQUIRE(Q * (int64_t)n < (int64_t)INT32_MAX, "query batch too large for one sort");
    Scratch ids, offs, tmp;
    LF_CUDA(ids.alloc(sizeof(int) * Q * n, st));
    LF_CUDA(offs.alloc(sizeof(int) * (Q + 1), st));
    int64_t cnt = Q * n > Q + 1 ? Q * n : Q + 1;
    iota_rows_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(ids.as<int>(), Q, n, offs.as<int>());
    LF_CUDA(cudaGetLastError());
    size_t bytes = 0;
    LF_CUDA(cub::DeviceSegmentedSort::StableSortPairs(
        nullptr, bytes, d_lb, d_lb_sorted, ids.as<int>(), d_order, (int)(Q * n), (int)Q,
        offs.as<int>(), offs.as<int>() + 1, st));
    LF_CUDA(tmp.alloc(bytes, st));
    LF_CUDA(cub::DeviceSegmentedSort::StableSortPairs(
        tmp.p, bytes, d_lb, d_lb_sorted, ids.as<int>(), d_order, (int)(Q * n), (int)Q,
        offs.as<int>(), offs.as<int>() + 1, st));
    return LF_OK;
}

}  // namespace lf

extern "C" int lf_bounds(const float* d_queries, int64_t Q, const lf_index* idx,
                         const double* d_env_min, const double* d_env_max, int32_t n_env,
                         int32_t lb_mode, double* d_qsumm, double* d_lb, void* stream) {
    LF_REQUIRE(idx != nullptr, "idx is NULL");
    LF_REQUIRE(idx->n_seg >= 1 && idx->n_seg <= LF_MAX_SEG, "bad segment count");
    LF_REQUIRE(lb_mode == 0 || lb_mode == 1, "lb_mode must be 0 or 1");
    return lf::launch_bounds(d_queries, Q, *idx, d_env_min, d_env_max, n_env, lb_mode, d_qsumm,
                             d_lb, lf::as_stream(stream));
}

extern "C" int lf_bounds_eapca(const float* d_queries, int64_t Q, const lf_index* idx, const double* d_env_min,
                               const double* d_env_max, const double* d_sd_min, const double* d_sd_max,
                               int32_t n_env, double* d_qsumm, double* d_lb, void* stream) {
    LF_REQUIRE(idx != nullptr && d_sd_min != nullptr && d_sd_max != nullptr, "NULL argument");
    LF_REQUIRE(idx->n_seg >= 1 && idx->n_seg <= LF_MAX_SEG, "bad segment count");
    return lf::launch_bounds(d_queries, Q, *idx, d_env_min, d_env_max, n_env, 2, d_qsumm, d_lb,
                             lf::as_stream(stream), nullptr, nullptr, d_sd_min, d_sd_max);
}

extern "C" int lf_eapca_device(const float* d_values, int64_t n, int32_t m, int32_t n_seg, double* d_out,
                               void* stream) {
    LF_REQUIRE(n_seg >= 1 && n_seg <= m && n_seg <= LF_MAX_SEG, "num_segments must be in [1, length]");
    if (n == 0) return LF_OK;
    lf_index idx{};
    idx.m = m;
    idx.n_seg = n_seg;
    const int base = m / n_seg, rem = m % n_seg;
    for (int i = 0, s = 0; i < n_seg; ++i) {
        idx.seg_width[i] = base + (i < rem ? 1 : 0);
        idx.seg_start[i] = s;
        s += idx.seg_width[i];
    }
    lf::eapca_kernel<<<(unsigned)((n * n_seg + 255) / 256), 256, 0, lf::as_stream(stream)>>>(d_values, n, idx, d_out);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

extern "C" int lf_paa_device(const float* d_values, int64_t n, int32_t m, int32_t n_seg, double* d_out,
                             void* stream) {
    LF_REQUIRE(n_seg >= 1 && n_seg <= m && n_seg <= LF_MAX_SEG, "num_segments must be in [1, length]");
    if (n == 0) return LF_OK;
    lf_index idx{};
    idx.m = m;
    idx.n_seg = n_seg;
    const int base = m / n_seg, rem = m % n_seg;
    for (int i = 0, s = 0; i < n_seg; ++i) {
        idx.seg_width[i] = base + (i < rem ? 1 : 0);
        idx.seg_start[i] = s;
        s += idx.seg_width[i];
    }
    const int64_t total = n * n_seg;
    lf::paa_kernel<<<(unsigned)((total + 255) / 256), 256, 0, lf::as_stream(stream)>>>(d_values, n, idx, d_out);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
