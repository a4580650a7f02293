// K5 on the INT8 tensor cores: exact query x leaf minimum distances for
// training-data generation (collect_targets / collect_local_targets,
// traingen.py:135-220; series.py:127-139 direct-form fp64 distances).
//
// The collection's int8 shadow (lf_quantize_rows: per-row scale s_x, codes c_x,
// sum of squared codes xx, quantisation error e_x = ||s_x c_x - x||) and the
// queries' codes (same scheme: s_q, c_q, qq, e_q) turn the O(Q N m) part into
// an exact int32 GEMM on tcgen05.mma.kind::i8:
//     D = c_q . c_x                                (exact, s32 accumulators in TMEM)
//     d^2(x^, q^) = s_x^2 xx + s_q^2 qq - 2 s_x s_q D   (fp32, rounding <= tol)
// and by the triangle inequality the true distance lies in
//     [sqrt(d^2 - tol) - e_x - e_q, sqrt(d^2 + tol) + e_x + e_q].
// Per (query, leaf) only rows whose lower end can reach the running minimum are
// re-checked EXACTLY in fp64 direct form from the fp32 rows (warp-cooperative),
// so the result is the exact fp64 minimum (same terms as lf_leaf_min_dist,
// another summation order: agreement to ~1 ulp).  The running minimum U is the
// exact best of the leaf's earlier chunks, or -- in a query's first chunk of a
// leaf -- min over the chunk of the upper ends.
//
// Tiles: 128 queries (UMMA M) x 256 rows (N) x m (K, 128-byte SW128 k-blocks, 4
// K=32 MMAs each).  The row chunk is double-buffered and resident while every
// query block streams past it; two TMEM accumulators of 256 columns.
// Warp roles (320 threads, one persistent CTA per SM):
//   warp 0: TMA producer (+ the chunk's per-row bound terms into smem)
//   warp 1: TMEM owner + MMA issuer
//   warps 2..9: epilogue, two groups of 4 (TMEM columns 0-127 / 128-255)
#include <vector>

#include "common.cuh"
#include "tc.cuh"

namespace lf {
namespace q8k {

using namespace ptx;

constexpr int BM = 128;                         // queries per tile
constexpr int BN = 256;                         // rows per chunk
constexpr int KBB = 128;                        // bytes (int8 elements) per k-block
constexpr int MAX_KB = 2;                       // m <= 256
constexpr int STAGES = 4;
constexpr int THREADS = 320;
constexpr int EPI_WARPS = 8;
constexpr int A_BYTES = BM * KBB;               // 16 KiB per query stage
constexpr int B_KB_BYTES = BN * KBB;            // 32 KiB per chunk k-block
constexpr int B_BYTES = MAX_KB * B_KB_BYTES;    // 64 KiB per chunk buffer
constexpr int TMEM_COLS = 512;                  // 2 accumulators x 256 columns
constexpr int OFF_B = 0;
constexpr int OFF_A = OFF_B + 2 * B_BYTES;
constexpr int OFF_META = OFF_A + STAGES * A_BYTES;
constexpr int OFF_EMAX = OFF_META + 2 * BN * 16;
constexpr int OFF_BAR = OFF_EMAX + 16;
constexpr int N_BAR = 2 * STAGES + 2 + 2 + 2 + 2;
constexpr int OFF_TMEM = OFF_BAR + N_BAR * 8;
constexpr int OFF_LIST = OFF_TMEM + 16;
constexpr int OFF_SBEST = OFF_LIST + EPI_WARPS * 64 * 4;
constexpr int SMEM_BYTES = OFF_SBEST + EPI_WARPS * 32 * 8 + 1024;

struct Item {                      // one leaf against one query range
    int leaf;                      // leaf slot
    int col;                       // output column
    long long q0, q1;              // query rows [q0, q1)
};

// Exact fp64 direct-form re-check of a warp's candidate list (series.py:142-146):
// 8 lanes per candidate, each summing 1/8 of the dimensions with all its loads in
// flight at once (one L2 round trip per group of 4 candidates, not one per
// dimension block), then a fixed 3-step shuffle tree.  Folds the result into the
// owner's smem best and the global output (bit patterns of non-negative doubles
// order like the values).
template <int M>
__device__ __forceinline__ void recheck8(const int* list, int cnt, int lane, const float* __restrict__ Qf,
                                         long long qbase, const float* __restrict__ X, long long row0,
                                         unsigned long long* sbest, unsigned long long* __restrict__ out,
                                         long long ldo, int col) {
    constexpr int PER = M / 32;                       // float4 per lane
    const int sub = lane & 7;
    for (int base = 0; base < cnt; base += 4) {
        const int e = base + (lane >> 3);
        const bool valid = e < cnt;
        const int ent = valid ? list[e] : 0;
        const int owner = ent >> 8, rr = ent & 255;
        const float4* qrow = reinterpret_cast<const float4*>(Qf + (qbase + owner) * M);
        const float4* xrow = reinterpret_cast<const float4*>(X + (row0 + rr) * M);
        float4 xv[PER], qv[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            xv[i] = valid ? __ldg(xrow + sub + 8 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
            qv[i] = valid ? __ldg(qrow + sub + 8 * i) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        double part = 0.0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const double e0 = (double)xv[i].x - (double)qv[i].x, e1 = (double)xv[i].y - (double)qv[i].y;
            const double e2 = (double)xv[i].z - (double)qv[i].z, e3 = (double)xv[i].w - (double)qv[i].w;
            part = __fma_rn(e0, e0, part); part = __fma_rn(e1, e1, part);
            part = __fma_rn(e2, e2, part); part = __fma_rn(e3, e3, part);
        }
        part += __shfl_xor_sync(0xffffffffu, part, 4);
        part += __shfl_xor_sync(0xffffffffu, part, 2);
        part += __shfl_xor_sync(0xffffffffu, part, 1);
        if (valid && sub == 0) {
            const unsigned long long bits = (unsigned long long)__double_as_longlong(part);
            atomicMin(&sbest[owner], bits);
            atomicMin(out + (qbase + owner) * ldo + col, bits);
        }
    }
}

__global__ void __launch_bounds__(THREADS, 1)
mindist_q8_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_x,
                  const Item* __restrict__ items, int n_items, lf_index idx, const float* __restrict__ Qf,
                  const float4* __restrict__ qmeta, unsigned long long* __restrict__ out, long long ldo) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-B alignment for the SW128 tiles, by offsetting the __shared__ array itself so the
    // compiler keeps the shared address space (LDS, not generic loads)
    uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
    uint8_t* Bs = smem + OFF_B;
    uint8_t* As = smem + OFF_A;
    float4* meta = reinterpret_cast<float4*>(smem + OFF_META);        // [2][BN] {s^2 xx, s, e, alpha}
    float* emax_s = reinterpret_cast<float*>(smem + OFF_EMAX);        // [2]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* empty = full + STAGES;
    uint64_t* bfull = empty + STAGES;
    uint64_t* bempty = bfull + 2;
    uint64_t* tfull = bempty + 2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
    int* cand_all = reinterpret_cast<int*>(smem + OFF_LIST);
    unsigned long long* sbest_all = reinterpret_cast<unsigned long long*>(smem + OFF_SBEST);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = idx.m;
    const int n_kb = m / KBB;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) {
            // every writer / reader lane arrives itself (the producer's 32 lanes write the
            // chunk's bound terms; all epilogue lanes read them), so the happens-before
            // edges are per thread (compute-sanitizer racecheck models them that way)
            mbar_init(&bfull[s], 32);
            mbar_init(&bempty[s], 1 + EPI_WARPS * 32);
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], EPI_WARPS);
        }
        mbar_fence_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {                                            // ---- producer
        const float4* rmeta = reinterpret_cast<const float4*>(idx.d_qmeta);
        int stage = 0;
        uint32_t phase = 0;
        long long chunk = 0;
        for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
            const Item item = items[it];
            const long long lb = idx.d_leaf_ptr[item.leaf], le = idx.d_leaf_ptr[item.leaf + 1];
            const int n_qb = (int)((item.q1 - item.q0 + BM - 1) / BM);
            for (long long r0 = lb; r0 < le; r0 += BN, ++chunk) {
                const int bb = (int)(chunk & 1);
                __syncwarp();                       // lanes 1-31 wait for lane 0's TMA issue loop
                mbar_wait(&bempty[bb], (uint32_t)((chunk >> 1) & 1) ^ 1u);
                float em = 0.f;
                for (int i = lane; i < BN; i += 32) {
                    const long long r = r0 + i;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (r < le) {
                        const float4 mr = __ldg(rmeta + r);
                        const float a = mr.x * mr.x * mr.y;
                        v = make_float4(a, mr.x, mr.z, fmaf(-(1.f + 3e-5f) * mr.z, mr.z, (1.f - 2e-5f) * a));
                        em = fmaxf(em, mr.z);
                    }
                    meta[bb * BN + i] = v;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) em = fmaxf(em, __shfl_xor_sync(0xffffffffu, em, o));
                if (lane == 0) emax_s[bb] = em;
                __syncwarp();
                if (lane == 0) {
                    mbar_expect_tx(&bfull[bb], (uint32_t)(n_kb * B_KB_BYTES));
                    for (int kb = 0; kb < n_kb; ++kb)
                        tma_2d(&map_x, &bfull[bb], Bs + bb * B_BYTES + kb * B_KB_BYTES, kb * KBB, (int)r0);
                } else {
                    mbar_arrive(&bfull[bb]);
                }
                for (int qb = 0; qb < n_qb; ++qb) {
                    for (int kb = 0; kb < n_kb; ++kb) {
                        if (lane == 0) {
                            mbar_wait(&empty[stage], phase ^ 1);
                            mbar_expect_tx(&full[stage], A_BYTES);
                            tma_2d(&map_q, &full[stage], As + stage * A_BYTES, kb * KBB, (int)(item.q0 + qb * BM));
                        }
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {                                     // ---- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_s8(BM, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            long long chunk = 0;
            for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
                const Item item = items[it];
                const long long lb = idx.d_leaf_ptr[item.leaf], le = idx.d_leaf_ptr[item.leaf + 1];
                const int n_qb = (int)((item.q1 - item.q0 + BM - 1) / BM);
                for (long long r0 = lb; r0 < le; r0 += BN, ++chunk) {
                    const int bb = (int)(chunk & 1);
                    mbar_wait(&bfull[bb], (uint32_t)((chunk >> 1) & 1));
                    tc_after();
                    const uint32_t bs = su32(Bs + bb * B_BYTES);
                    for (int qb = 0; qb < n_qb; ++qb) {
                        mbar_wait(&tempty[acc], acc_phase ^ 1);
                        tc_after();
                        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
                        for (int kb = 0; kb < n_kb; ++kb) {
                            mbar_wait(&full[stage], phase);
                            tc_after();
                            const uint32_t as = su32(As + stage * A_BYTES);
#pragma unroll
                            for (int kk = 0; kk < KBB / 32; ++kk)         // K = 32 int8 = 32 bytes per MMA
                                mma_i8(d, sw128_desc(as + kk * 32), sw128_desc(bs + kb * B_KB_BYTES + kk * 32), idesc,
                                       (kb | kk) != 0 ? 1u : 0u);
                            mma_commit(&empty[stage]);
                            if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        }
                        mma_commit(&tfull[acc]);
                        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                    }
                    mma_commit(&bempty[bb]);                            // chunk no longer read by MMAs
                }
            }
        }
    } else {                                                    // ---- epilogue (warps 2..9)
        const int quarter = warp & 3;
        const int grp = (warp - 2) >> 2;                        // column half
        const int row = quarter * 32 + lane;
        int* list = cand_all + (warp - 2) * 64;
        unsigned long long* sbest = sbest_all + (warp - 2) * 32;     // this warp's queries' best (bits)
        int acc = 0;
        uint32_t acc_phase = 0;
        long long chunk = 0;
        for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
            const Item item = items[it];
            const long long lb = idx.d_leaf_ptr[item.leaf], le = idx.d_leaf_ptr[item.leaf + 1];
            const int n_qb = (int)((item.q1 - item.q0 + BM - 1) / BM);
            for (long long r0 = lb; r0 < le; r0 += BN, ++chunk) {
                const int bb = (int)(chunk & 1);
                const int nrows = (int)min((long long)BN, le - r0);
                mbar_wait(&bfull[bb], (uint32_t)((chunk >> 1) & 1));       // chunk bound terms visible
                const float4* mt = meta + bb * BN + grp * 128;
                const int ncols = max(0, min(128, nrows - grp * 128));
                const float emax_rows = emax_s[bb];
                // per-tile query state, prefetched one query block ahead (global loads off the
                // critical path: a stale best only loosens the test)
                auto load_q = [&](int qb_, double& b_, float4& m_) {
                    const long long q_ = item.q0 + (long long)qb_ * BM + row;
                    const bool v_ = q_ < item.q1;
                    b_ = v_ ? __longlong_as_double((long long)*(volatile unsigned long long*)(out + q_ * ldo + item.col))
                            : 0.0;
                    m_ = v_ ? __ldg(qmeta + q_) : make_float4(1.f, 0.f, 0.f, 0.f);
                };
                double best_n;
                float4 qm_n;
                load_q(0, best_n, qm_n);
                for (int qb = 0; qb < n_qb; ++qb) {
                    const long long q = item.q0 + (long long)qb * BM + row;
                    const bool qv = q < item.q1;
                    double best = best_n;
                    const float4 qm = qm_n;
                    if (qb + 1 < n_qb) load_q(qb + 1, best_n, qm_n);
                    const float Cq = qm.x * qm.x * qm.y, cq2 = 2.f * qm.x;
                    const float emax = emax_rows + qm.z;
                    mbar_wait(&tfull[acc], acc_phase);
                    tc_after();
                    const uint32_t taddr =
                        tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN + grp * 128);
                    float U = best < kInf ? __fsqrt_ru(__double2float_ru(best)) : __int_as_float(0x7f800000);
                    // a query's first chunk of the leaf: min over my columns of the upper ends (the
                    // TMEM loads are warp-collective, so the whole warp runs the pass if any lane needs it)
                    if (__any_sync(0xffffffffu, !(best < kInf))) {
                        float v = __int_as_float(0x7f800000);
                        for (int c0 = 0; c0 < ncols; c0 += 32) {
                            uint32_t r[32];
                            LF_TMEM_LD32X(taddr + (uint32_t)c0, r);
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                if (c0 + j < ncols) {
                                    const float4 mr = mt[c0 + j];
                                    const float c1 = mr.x + Cq;
                                    const float d2 = fmaf(-(cq2 * mr.y), (float)(int)r[j], c1);
                                    v = fminf(v, fmaf(1e-5f, c1, d2));
                                }
                            }
                        }
                        if (!(best < kInf)) U = (sqrtf(fmaxf(v, 0.f)) + emax) * (1.f + 1e-6f);
                    }
                    // candidates: sqrt(d^2 - tol) - e_r - e_q <= U  <=>  d^2 - tol <= (U + e_q + e_r)^2
                    const float V = (U + qm.z) * (1.f + 1e-6f);
                    const long long qbase = item.q0 + (long long)qb * BM + quarter * 32;
                    sbest[lane] = (unsigned long long)__double_as_longlong(best);
                    int cnt = 0;
                    // exact fp64 re-check, one candidate per lane (rows come from L2: the chunk's
                    // fp32 rows are shared by every query block that streams past it)
                    auto flush = [&]() {
                        __syncwarp();
                        if (m == 256)
                            recheck8<256>(list, cnt, lane, Qf, qbase, idx.d_X, r0 + grp * 128, sbest, out, ldo, item.col);
                        else
                            recheck8<128>(list, cnt, lane, Qf, qbase, idx.d_X, r0 + grp * 128, sbest, out, ldo, item.col);
                        __syncwarp();
                        best = __longlong_as_double((long long)sbest[lane]);
                        cnt = 0;
                    };
                    for (int c0 = 0; c0 < ncols; c0 += 32) {
                        uint32_t r[32];
                        LF_TMEM_LD32X(taddr + (uint32_t)c0, r);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        // d^2 - tol <= (V + e_r)^2, expanded so each element costs ~8 fp32 ops:
                        //   alpha_r + beta - gamma e_r <= (cq2 D) s_r   with
                        //   alpha_r = (1-2e-5) s_r^2 xx_r - (1+3e-5) e_r^2  (per row, in smem),
                        //   beta = (1-2e-5) Cq - (1+3e-5) V^2, gamma = 2 (1+3e-5) V  (per query);
                        // the widened constants cover the 1e-5 tolerance and fp32 rounding.
                        const bool vf = V < __int_as_float(0x7f800000);   // V = inf: every row qualifies
                        const float beta = vf ? fmaf(-(1.f + 3e-5f) * V, V, (1.f - 2e-5f) * Cq)
                                              : -__int_as_float(0x7f800000);
                        const float gamma = vf ? 2.f * (1.f + 3e-5f) * V : 0.f;
                        unsigned bits = 0;
                        if (qv) {
                            if (c0 + 32 <= ncols) {
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    const float4 mr = mt[c0 + j];
                                    const float lhs = fmaf(-gamma, mr.z, mr.w + beta);
                                    bits |= (lhs <= (cq2 * (float)(int)r[j]) * mr.y ? 1u : 0u) << j;
                                }
                            } else {
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    if (c0 + j < ncols) {
                                        const float4 mr = mt[c0 + j];
                                        const float lhs = fmaf(-gamma, mr.z, mr.w + beta);
                                        bits |= (lhs <= (cq2 * (float)(int)r[j]) * mr.y ? 1u : 0u) << j;
                                    }
                                }
                            }
                        }
                        while (__any_sync(0xffffffffu, bits != 0)) {     // append <= 32 entries per pass
                            if (cnt > 32) flush();
                            const bool has = bits != 0;
                            const unsigned mask = __ballot_sync(0xffffffffu, has);
                            if (has) {
                                const int j = __ffs(bits) - 1;
                                bits &= bits - 1;
                                list[cnt + __popc(mask & ((1u << lane) - 1u))] = (lane << 8) | (c0 + j);
                            }
                            cnt += __popc(mask);
                        }
                    }
                    if (cnt) flush();
                    tc_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
                }
                __syncwarp();
                mbar_arrive(&bempty[bb]);                                // bound terms may be replaced
            }
        }
    }
    tc_before();
    __syncthreads();
    if (warp == 1) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

__global__ void fill_bits_kernel(unsigned long long* p, int64_t rows, int64_t cols, int64_t ld, unsigned long long v) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < rows * cols) p[(t / cols) * ld + (t % cols)] = v;
}

__global__ void sqrt_bits_kernel(double* p, int64_t rows, int64_t cols, int64_t ld) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < rows * cols) {
        double* e = p + (t / cols) * ld + (t % cols);
        *e = sqrt(*e);
    }
}

static int run(const float* d_q, int64_t Q, const lf_index& idx, const std::vector<Item>& items, double* d_out,
               int64_t out_rows, int64_t out_cols, int64_t ldo, cudaStream_t st) {
    LF_REQUIRE(idx.d_X8 != nullptr && idx.d_qmeta != nullptr, "int8 min-distance needs the int8 shadow (X8)");
    LF_REQUIRE(idx.m == 128 || idx.m == 256, "int8 tensor-core min-distance needs m in {128, 256}");
    LF_REQUIRE(((uintptr_t)d_q & 15) == 0 && ((uintptr_t)idx.d_X & 15) == 0, "operands must be 16-byte aligned");
    if (items.empty() || Q == 0) return LF_OK;
    Scratch d_items, qc, qm;
    LF_CUDA(d_items.alloc(sizeof(Item) * items.size(), st));
    LF_CUDA(cudaMemcpyAsync(d_items.p, items.data(), sizeof(Item) * items.size(), cudaMemcpyHostToDevice, st));
    const int mp = (idx.m + 255) / 256 * 256;
    LF_CUDA(qc.alloc((size_t)Q * mp, st));
    LF_CUDA(qm.alloc(sizeof(float4) * Q, st));
    int rc = quantize_queries(d_q, Q, idx.m, mp, qc.as<int8_t>(), qm.as<float4>(), st);
    if (rc) return rc;
    fill_bits_kernel<<<(unsigned)((out_rows * out_cols + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<unsigned long long*>(d_out), out_rows, out_cols, ldo, 0x7ff0000000000000ULL);
    LF_CUDA(cudaGetLastError());
    CUtensorMap mq, mx;
    rc = encode_map_2d(&mq, CU_TENSOR_MAP_DATA_TYPE_UINT8, qc.p, Q, idx.m, mp, KBB, BM);
    if (rc) return rc;
    rc = encode_map_2d(&mx, CU_TENSOR_MAP_DATA_TYPE_UINT8, idx.d_X8, idx.n_series, idx.m, idx.m, KBB, BN);
    if (rc) return rc;
    LF_CUDA(smem_optin(mindist_q8_kernel, SMEM_BYTES));
    const int grid = (int)std::min<size_t>(items.size(), (size_t)sm_count());
    mindist_q8_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(mq, mx, d_items.as<Item>(), (int)items.size(), idx, d_q,
                                                         qm.as<float4>(),
                                                         reinterpret_cast<unsigned long long*>(d_out), ldo);
    LF_CUDA(cudaGetLastError());
    sqrt_bits_kernel<<<(unsigned)((out_rows * out_cols + 255) / 256), 256, 0, st>>>(d_out, out_rows, out_cols, ldo);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

}  // namespace q8k
}  // namespace lf

extern "C" int lf_leaf_min_dist_q8(const float* d_queries, int64_t Q, const lf_index* idx, const int32_t* h_leaf_sel,
                                   int32_t S, double* d_dl, int64_t ldd, void* stream) {
    using namespace lf;
    LF_REQUIRE(idx != nullptr && Q >= 0 && S >= 0 && ldd >= S, "bad arguments");
    std::vector<q8k::Item> items;
    items.reserve(S);
    for (int s = 0; s < S; ++s) items.push_back(q8k::Item{h_leaf_sel[s], s, 0, Q});
    return q8k::run(d_queries, Q, *idx, items, d_dl, Q, S, ldd, as_stream(stream));
}

extern "C" int lf_local_min_dist_q8(const float* d_queries, const lf_index* idx, const int64_t* h_qptr,
                                    const int32_t* h_group_leaf, int32_t n_groups, double* d_dl, void* stream) {
    using namespace lf;
    LF_REQUIRE(idx != nullptr && n_groups >= 0, "bad arguments");
    if (n_groups == 0) return LF_OK;
    const int64_t Q = h_qptr[n_groups];
    std::vector<q8k::Item> items;
    items.reserve(n_groups);
    for (int g = 0; g < n_groups; ++g)
        if (h_qptr[g + 1] > h_qptr[g]) items.push_back(q8k::Item{h_group_leaf[g], 0, h_qptr[g], h_qptr[g + 1]});
    return q8k::run(d_queries, Q, *idx, items, d_dl, Q, 1, 1, as_stream(stream));
}
