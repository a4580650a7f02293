// K1: query segment means + node lower bounds over SoA envelopes (HBM-bound).
//
// Reference: summarize.py:44-56 (segment means), summarize.py:97-107 (search
// bound, np.dot -> one fp64 FMA chain over segments), summarize.py:114-122
// (batched bound used by traingen, einsum -> sequential sum of (g*g)*w).
// Both orders are reproduced bit-for-bit so visit orders and counters match.
#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>

#include "bounds.cuh"
#include "common.cuh"

namespace lf {

// One thread per (query, segment).
__global__ void paa_kernel(const float* __restrict__ q, int64_t Q, lf_index idx,
                           double* __restrict__ qsumm) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= Q * idx.n_seg) return;
    int64_t qi = t / idx.n_seg;
    int s = (int)(t - qi * idx.n_seg);
    qsumm[t] = segment_mean(q + qi * idx.m, idx.seg_start[s], idx.seg_width[s]);
}

// lb[q][node] for nodes of one query row; segment means staged in smem.
template <int MODE>
__global__ void lb_kernel(const double* __restrict__ qsumm, int64_t Q, int n_seg, lf_index idx,
                          const double* __restrict__ env_min, const double* __restrict__ env_max,
                          int n_env, double* __restrict__ lb) {
    __shared__ double qs[LF_MAX_SEG];
    __shared__ double ws[LF_MAX_SEG];
    for (int64_t qi = blockIdx.y; qi < Q; qi += gridDim.y) {
        __syncthreads();
        if (threadIdx.x < n_seg) {
            qs[threadIdx.x] = qsumm[qi * n_seg + threadIdx.x];
            ws[threadIdx.x] = (double)idx.seg_width[threadIdx.x];
        }
        __syncthreads();
        for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < n_env;
             node += gridDim.x * blockDim.x) {
            double acc = 0.0;
            for (int s = 0; s < n_seg; ++s) {
                double mn = env_min[(int64_t)s * n_env + node];
                double mx = env_max[(int64_t)s * n_env + node];
                double g = fmax(mn - qs[s], qs[s] - mx);
                g = fmax(g, 0.0);
                if (MODE == 0) {
                    acc = __fma_rn(__dmul_rn(ws[s], g), g, acc);          // np.dot(widths*gap, gap)
                } else {
                    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(g, g), ws[s]));  // einsum qns,qns,s
                }
            }
            lb[qi * n_env + node] = sqrt(acc);
        }
    }
}

int launch_bounds(const float* d_q, int64_t Q, const lf_index& idx, const double* env_min,
                  const double* env_max, int n_env, int mode, double* d_qsumm, double* d_lb,
                  cudaStream_t st) {
    if (Q == 0) return LF_OK;
    {
        int64_t n = Q * idx.n_seg;
        int thr = 256;
        paa_kernel<<<(unsigned)((n + thr - 1) / thr), thr, 0, st>>>(d_q, Q, idx, d_qsumm);
        LF_CUDA(cudaGetLastError());
    }
    if (n_env == 0) return LF_OK;
    dim3 block(256);
    dim3 grid((unsigned)((n_env + 255) / 256), (unsigned)(Q < 65535 ? Q : 65535));
    if (mode == 0)
        lb_kernel<0><<<grid, block, 0, st>>>(d_qsumm, Q, idx.n_seg, idx, env_min, env_max,
                                             n_env, d_lb);
    else
        lb_kernel<1><<<grid, block, 0, st>>>(d_qsumm, Q, idx.n_seg, idx, env_min, env_max,
                                             n_env, d_lb);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

__global__ void iota_rows_kernel(int* __restrict__ v, int64_t Q, int n, int* __restrict__ offs) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < Q * n) v[t] = (int)(t % n);
    if (t <= Q) offs[t] = (int)(t * n);
}

// One visit-order record: node, its bound, its leaf slot (+ filter flag) and the
// filter operand pred - offset (tree.py:277-286), exactly as the plan evaluates it.
__device__ inline void put_record(const OrderArgs& o, const lf_index& idx, int64_t q, int Nn, int p, double lb,
                                  int node) {
    const int64_t at = q * Nn + p;
    o.lbs[at] = lb;
    o.order[at] = node;
    const int leaf = idx.d_node_leaf[node];
    int rec = leaf;
    double a = -kInf;
    if (leaf >= 0 && idx.d_leaf_filter != nullptr && (o.pred != nullptr || o.pred64 != nullptr || o.lazy)) {
        const int fs = idx.d_leaf_filter[leaf];
        if (fs >= 0) {
            rec |= LF_REC_HASF;
            if (o.lazy) {
                a = __longlong_as_double(0x7ff8000000000000LL);    // filled by the lazy inference
            } else {
                const double pv = o.pred64 != nullptr ? o.pred64[q * o.F + fs] : (double)o.pred[q * o.F + fs];
                a = pv - o.offset[fs];
            }
        }
    }
    o.leafo[at] = rec;
    o.adj[at] = a;
}

__device__ inline double node_bound(const double* qs, const double* ws, int ns, const double* env_min,
                                    const double* env_max, int n_env, int node) {
    double acc = 0.0;
    for (int sg = 0; sg < ns; ++sg) {                  // lb_kernel<0>: np.dot(widths*gap, gap)
        const double mn = env_min[(int64_t)sg * n_env + node];
        const double mx = env_max[(int64_t)sg * n_env + node];
        double g = fmax(mn - qs[sg], qs[sg] - mx);
        g = fmax(g, 0.0);
        acc = __fma_rn(__dmul_rn(ws[sg], g), g, acc);
    }
    return sqrt(acc);
}

// ITEMS bounds per thread for nodes first, first + stride, ... (striped, so each
// warp load is 256 contiguous bytes of one segment's envelope row).  Segments
// are the OUTER loop: all 2 x ITEMS loads of a segment are in flight together
// instead of one dependent L2 round trip per (node, segment).  Each node's FMA
// chain still runs over segments in order -- bit-identical to node_bound.
template <int ITEMS>
__device__ __forceinline__ void node_bounds_striped(const double* qs, const double* ws, int ns,
                                                    const double* __restrict__ env_min,
                                                    const double* __restrict__ env_max, int n_env, int first,
                                                    int stride, double (&lb)[ITEMS]) {
    double acc[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) acc[i] = 0.0;
    for (int sg = 0; sg < ns; ++sg) {
        const double qv = qs[sg], wv = ws[sg];
        const double* mnp = env_min + (int64_t)sg * n_env;
        const double* mxp = env_max + (int64_t)sg * n_env;
        double mn[ITEMS], mx[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int node = first + i * stride;
            mn[i] = node < n_env ? __ldg(mnp + node) : 0.0;
            mx[i] = node < n_env ? __ldg(mxp + node) : 0.0;
        }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            double g = fmax(mn[i] - qv, qv - mx[i]);
            g = fmax(g, 0.0);
            acc[i] = __fma_rn(__dmul_rn(wv, g), g, acc[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) lb[i] = sqrt(acc[i]);
}

// put_record for ITEMS visit positions per thread (p = first + i * stride), the
// dependent loads (node -> leaf -> filter -> prediction, offset) issued level by
// level across all ITEMS positions so their latencies overlap.
template <int ITEMS>
__device__ __forceinline__ void put_records_striped(const OrderArgs& o, const lf_index& idx, int64_t q, int Nn,
                                                    int first, int stride, const unsigned* key_hi,
                                                    const int* node_at, const unsigned* lo_by_node) {
    int node[ITEMS], leaf[ITEMS], fs[ITEMS];
    const bool filt = idx.d_leaf_filter != nullptr && (o.pred != nullptr || o.pred64 != nullptr || o.lazy);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int p = first + i * stride;
        node[i] = p < Nn ? node_at[p] : -1;
    }
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) leaf[i] = node[i] >= 0 ? __ldg(idx.d_node_leaf + node[i]) : -1;
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
        const int p = first + i * stride;
        if (p >= Nn) continue;
        const int64_t at = q * Nn + p;
        o.lbs[at] = __hiloint2double((int)key_hi[p], (int)lo_by_node[node[i]]);
        o.order[at] = node[i];
        int rec = leaf[i];
        double a = -kInf;
        if (fs[i] >= 0) {
            rec |= LF_REC_HASF;
            a = o.lazy ? __longlong_as_double(0x7ff8000000000000LL) : pv[i] - off[i];
        }
        o.leafo[at] = rec;
        o.adj[at] = a;
    }
}

// Fused K1 + K2 for trees of up to 8192 nodes, FULL order: one CTA per query
// computes every node's search bound straight into registers and sorts the
// nodes in shared memory -- the bound matrix never round-trips through HBM.
// The sort key is the HIGH 32 bits of the non-negative fp64 bound (they order
// like the doubles): a stable 4-pass 8-bit block radix sort instead of a 16-pass
// sort of 64-bit keys.  Equal high words are then put in exact (lb, node id)
// order by sorting each run on the low words (runs are rare and short; equal
// bounds keep ascending ids from the stable sort), so the result is the exact
// (lb, id) order of tree.py:256-275.
constexpr int FS_THREADS = 512;

template <int ITEMS, int RB>
struct FsSmem {
    using Sort = cub::BlockRadixSort<unsigned, FS_THREADS, ITEMS, int, RB>;
    unsigned lo[FS_THREADS * ITEMS];                   // low word of each node's bound, by node id
    union {
        typename Sort::TempStorage sort;
        struct {
            unsigned key[FS_THREADS * ITEMS];          // sorted high words
            int node[FS_THREADS * ITEMS];              // sorted node ids
        } out;
    } u;
};

template <int ITEMS, int RB>
__global__ void __launch_bounds__(FS_THREADS, 1) bounds_sort_kernel(const double* __restrict__ qsumm, lf_index idx,
                                                                 int n_env, OrderArgs o) {
    using Sm = FsSmem<ITEMS, RB>;
    extern __shared__ __align__(16) uint8_t fs_smem[];
    Sm& sm = *reinterpret_cast<Sm*>(fs_smem);
    __shared__ double qs[LF_MAX_SEG];
    __shared__ double ws[LF_MAX_SEG];
    const int64_t q = blockIdx.x;
    if (o.only != nullptr && o.only[q] == 0) return;
    const int ns = idx.n_seg;
    if (threadIdx.x < ns) {
        qs[threadIdx.x] = qsumm[q * ns + threadIdx.x];
        ws[threadIdx.x] = (double)idx.seg_width[threadIdx.x];
    }
    __syncthreads();
    {
        double lb[ITEMS];
        node_bounds_striped<ITEMS>(qs, ws, ns, idx.d_env_min, idx.d_env_max, n_env, threadIdx.x, FS_THREADS, lb);
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const int node = i * FS_THREADS + threadIdx.x;
            if (node < n_env) {
                sm.u.out.key[node] = (unsigned)__double2hiint(lb[i]);
                sm.lo[node] = (unsigned)__double2loint(lb[i]);
            }
        }
    }
    __syncthreads();
    unsigned keys[ITEMS];
    int vals[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int node = threadIdx.x * ITEMS + i;          // blocked arrangement: stable sort keeps id order
        if (node < n_env) {
            keys[i] = sm.u.out.key[node];
            vals[i] = node;
        } else {
            keys[i] = 0xFFFFFFFFu;                         // padding sorts last (real keys <= +inf's 0x7FF00000)
            vals[i] = INT_MAX;
        }
    }
    __syncthreads();                                       // the sort's temp storage overlays out.key
    // Bit 31 (the sign of a non-negative bound) is always 0 -- padding's 0x7FFFFFFF in
    // the low 31 bits still sorts after +inf's 0x7FF00000.  Striped output: conflict-free stores.
    typename Sm::Sort(sm.u.sort).SortBlockedToStriped(keys, vals, 0, 31);
    __syncthreads();                                       // temp storage is reused below
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        sm.u.out.key[i * FS_THREADS + threadIdx.x] = keys[i];
        sm.u.out.node[i * FS_THREADS + threadIdx.x] = vals[i];
    }
    __syncthreads();
    for (int p = threadIdx.x; p < n_env; p += FS_THREADS) {   // exact order inside runs of equal high words
        const unsigned kp = sm.u.out.key[p];
        if ((p == 0 || sm.u.out.key[p - 1] != kp) && p + 1 < n_env && sm.u.out.key[p + 1] == kp) {
            int e = p + 1;
            while (e < n_env && sm.u.out.key[e] == kp) ++e;
            for (int a = p + 1; a < e; ++a) {              // insertion sort by (low word, id)
                const int na = sm.u.out.node[a];
                const unsigned la = sm.lo[na];
                int b = a - 1;
                while (b >= p) {
                    const int nb = sm.u.out.node[b];
                    const unsigned lbw = sm.lo[nb];
                    if (lbw < la || (lbw == la && nb < na)) break;
                    sm.u.out.node[b + 1] = nb;
                    --b;
                }
                sm.u.out.node[b + 1] = na;
            }
        }
    }
    __syncthreads();
    put_records_striped<ITEMS>(o, idx, q, n_env, threadIdx.x, FS_THREADS, sm.u.out.key, sm.u.out.node, sm.lo);
    if (threadIdx.x == 0) {
        o.olen[q] = n_env;
        if (o.only != nullptr) o.only[q] = 0;
    }
}

// Fused K1 + K2, PREFIX of the order (trees of up to 8192 nodes).  A search
// only ever walks the head of its visit order (it stops at the first node with
// lb > bsf * f), so sorting all n_nodes pairs per query is mostly wasted work.
// One CTA per query: bounds into registers; radix-select (4 byte passes over
// the high 32 bits of the non-negative fp64 bound, which order like the
// doubles) the key T of the PF_K-th smallest; compact every node with key <= T
// (or < T if that overflows PF_CAP) -- exactly the head of the (lb, id) order --
// and bitonic-sort it by (lb, id) in shared memory.  A query whose walk reaches
// the end of its prefix is refilled with the full order (refill_order).
constexpr int PF_THREADS = 512;
constexpr int PF_ITEMS = 16;
constexpr int PF_K = 1024;
constexpr int PF_CAP = 2048;

__global__ void __launch_bounds__(PF_THREADS, 1) prefix_order_kernel(const double* __restrict__ qsumm, lf_index idx,
                                                                  int Nn, OrderArgs o) {
    __shared__ double qs[LF_MAX_SEG];
    __shared__ double ws[LF_MAX_SEG];
    __shared__ double sk[PF_CAP];
    __shared__ int sv[PF_CAP];
    __shared__ int hist[256];
    __shared__ unsigned s_prefix;
    __shared__ int s_rem, s_lt, s_le, s_cnt;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t q = blockIdx.x;
    const int ns = idx.n_seg;
    if (tid < ns) {
        qs[tid] = qsumm[q * ns + tid];
        ws[tid] = (double)idx.seg_width[tid];
    }
    if (tid == 0) { s_lt = 0; s_le = 0; s_cnt = 0; }
    __syncthreads();
    double key[PF_ITEMS];
    unsigned k32[PF_ITEMS];
    node_bounds_striped<PF_ITEMS>(qs, ws, ns, idx.d_env_min, idx.d_env_max, Nn, tid, PF_THREADS, key);
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i) {
        const int node = i * PF_THREADS + tid;             // striped; the bitonic sort orders by (lb, id)
        if (node < Nn) {
            k32[i] = (unsigned)__double2hiint(key[i]);     // lb >= 0: monotone in lb
        } else {
            key[i] = kInf;
            k32[i] = 0xFFFFFFFFu;                          // never selected
        }
    }
    unsigned T = 0xFFFFFFFEu;                              // Nn <= PF_CAP: everything
    bool take = true;
    if (Nn > PF_CAP) {
        unsigned prefix = 0, mask = 0;
        int rem = PF_K;
        for (int shift = 24; shift >= 0; shift -= 8) {
            if (tid < 256) hist[tid] = 0;
            __syncthreads();
#pragma unroll
            for (int i = 0; i < PF_ITEMS; ++i)
                if (k32[i] != 0xFFFFFFFFu && (k32[i] & mask) == prefix) atomicAdd(&hist[(k32[i] >> shift) & 255], 1);
            __syncthreads();
            if (warp == 0) {
                int c[8], sum = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) { c[j] = hist[lane * 8 + j]; sum += c[j]; }
                int incl = sum;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += v;
                }
                const int excl = incl - sum;
                if (excl < rem && rem <= incl) {
                    int acc = excl, b = 7;
                    for (int j = 0; j < 8; ++j) {
                        if (acc + c[j] >= rem) { b = j; break; }
                        acc += c[j];
                    }
                    s_prefix = prefix | ((unsigned)(lane * 8 + b) << shift);
                    s_rem = rem - acc;
                }
            }
            __syncthreads();
            prefix = s_prefix;
            rem = s_rem;
            mask |= 255u << shift;
        }
        T = prefix;                                        // key of the PF_K-th smallest bound
        int lt = 0, le = 0;
#pragma unroll
        for (int i = 0; i < PF_ITEMS; ++i) {
            lt += k32[i] < T;
            le += k32[i] <= T;
        }
        atomicAdd(&s_lt, lt);
        atomicAdd(&s_le, le);
        __syncthreads();
        if (s_le > PF_CAP) {                               // take only keys < T (count < PF_K); none
            if (s_lt == 0) take = false;                   // at all -> the plan refills at once
            else T -= 1;
        }
    }
#pragma unroll
    for (int i = 0; i < PF_ITEMS; ++i)
        if (take && k32[i] <= T) {
            const int pos = atomicAdd(&s_cnt, 1);
            sk[pos] = key[i];
            sv[pos] = i * PF_THREADS + tid;
        }
    __syncthreads();
    const int cnt = s_cnt;
    int N = 64;
    while (N < cnt) N <<= 1;
    for (int i = cnt + tid; i < N; i += PF_THREADS) { sk[i] = kInf; sv[i] = INT_MAX; }
    __syncthreads();
    for (int k = 2; k <= N; k <<= 1) {                     // bitonic sort by (lb, node id)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < N; i += PF_THREADS) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const double a = sk[i], b = sk[ixj];
                    const int va = sv[i], vb = sv[ixj];
                    const bool gt = a > b || (a == b && va > vb);
                    if (gt == ((i & k) == 0)) { sk[i] = b; sk[ixj] = a; sv[i] = vb; sv[ixj] = va; }
                }
            }
            __syncthreads();
        }
    }
    for (int p = tid; p < cnt; p += PF_THREADS) put_record(o, idx, q, Nn, p, sk[p], sv[p]);
    if (tid == 0) o.olen[q] = cnt;
}

__global__ void records_kernel(const double* __restrict__ lb_sorted, const int* __restrict__ order, lf_index idx,
                               int64_t Q, int Nn, OrderArgs o) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < Q * Nn) {
        const int64_t q = t / Nn;
        put_record(o, idx, q, Nn, (int)(t - q * Nn), lb_sorted[t], order[t]);
    }
    if (t < Q) o.olen[t] = Nn;
}

template <int ITEMS, int RB = 4>
static int launch_fused(const double* d_qsumm, int64_t Q, const lf_index& idx, int n, const OrderArgs& oa,
                        cudaStream_t st) {
    const int bytes = (int)sizeof(FsSmem<ITEMS, RB>);
    LF_CUDA(smem_optin(bounds_sort_kernel<ITEMS, RB>, bytes));
    bounds_sort_kernel<ITEMS, RB><<<(unsigned)Q, FS_THREADS, bytes, st>>>(d_qsumm, idx, n, oa);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

static int sort_radix_bits() {                         // LF_SORT_RB: digit width of the block sort (4..7)
    const char* e = std::getenv("LF_SORT_RB");
    const int rb = e != nullptr ? std::atoi(e) : 5;
    return rb >= 4 && rb <= 7 ? rb : 5;
}

template <int ITEMS>
static int launch_fused_rb(const double* d_qsumm, int64_t Q, const lf_index& idx, int n, const OrderArgs& oa,
                           cudaStream_t st) {
    switch (sort_radix_bits()) {
        case 5: return launch_fused<ITEMS, 5>(d_qsumm, Q, idx, n, oa, st);
        case 6: return launch_fused<ITEMS, 6>(d_qsumm, Q, idx, n, oa, st);
        case 7: return launch_fused<ITEMS, 7>(d_qsumm, Q, idx, n, oa, st);
        default: return launch_fused<ITEMS, 4>(d_qsumm, Q, idx, n, oa, st);
    }
}

static int launch_full_fused(const double* d_qsumm, int64_t Q, const lf_index& idx, int n, const OrderArgs& oa,
                             cudaStream_t st) {
    if (n <= FS_THREADS * 4) return launch_fused_rb<4>(d_qsumm, Q, idx, n, oa, st);
    if (n <= FS_THREADS * 8) return launch_fused_rb<8>(d_qsumm, Q, idx, n, oa, st);
    return launch_fused_rb<16>(d_qsumm, Q, idx, n, oa, st);
}

// Segment means + bounds + per-query visit-order records in as few passes as the
// tree size allows: fused prefix / block sort up to 8192 nodes, else bounds
// kernel + CUB segmented sort + record gather.
int bounds_and_order(const float* d_q, int64_t Q, const lf_index& idx, double* d_qsumm, double* d_lb_scratch,
                     const OrderArgs& oa, bool prefix, cudaStream_t st, int* kernels) {
    const int n = idx.n_nodes;
    if (Q == 0 || n == 0) return LF_OK;
    if (n <= FS_THREADS * 16 && Q <= 0x7fffffff) {
        {
            int64_t tot = Q * idx.n_seg;
            paa_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(d_q, Q, idx, d_qsumm);
            LF_CUDA(cudaGetLastError());
        }
        if (kernels) *kernels += 2;
        if (prefix && n > PF_CAP) {
            prefix_order_kernel<<<(unsigned)Q, PF_THREADS, 0, st>>>(d_qsumm, idx, n, oa);
            LF_CUDA(cudaGetLastError());
            return LF_OK;
        }
        OrderArgs all = oa;
        all.only = nullptr;
        return launch_full_fused(d_qsumm, Q, idx, n, all, st);
    }
    int rc = launch_bounds(d_q, Q, idx, idx.d_env_min, idx.d_env_max, n, 0, d_qsumm, d_lb_scratch, st);
    if (rc) return rc;
    if (kernels) *kernels += 5;
    rc = sort_visit_order(d_lb_scratch, Q, n, oa.lbs, oa.order, st);
    if (rc) return rc;
    const int64_t tot = std::max<int64_t>(Q * n, Q);
    records_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(oa.lbs, oa.order, idx, Q, n, oa);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

int refill_order(const float* d_q, int64_t Q, const lf_index& idx, const double* d_qsumm, double* d_lb_scratch,
                 const OrderArgs& oa, cudaStream_t st, int* kernels) {
    (void)d_q;
    (void)d_lb_scratch;
    const int n = idx.n_nodes;
    LF_REQUIRE(n <= FS_THREADS * 16, "refill is only needed for prefix orders (<= 8192 nodes)");
    if (kernels) *kernels += 1;
    return launch_full_fused(d_qsumm, Q, idx, n, oa, st);
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
