// K5 on the tensor cores: exact query x leaf minimum distances for training-data
// generation (collect_targets / collect_local_targets, traingen.py:135-220).
//
// For every (query q, leaf) pair the reference computes min over the leaf's rows
// of ||q - x|| in fp64 direct form (series.py:127-139).  Here:
//
//  1. tcgen05.mma.kind::tf32 computes dot = q . x for a 128-query x 128-row tile
//     (A = queries, B = a 128-row chunk of the leaf, both K-major, TMA SWIZZLE_128B;
//     the B chunk stays resident in smem while every query block streams past it;
//     4 TMEM accumulator buffers of 128 columns);
//  2. the epilogue forms a = |q|^2 + |x|^2 - 2 dot with a rigorous error bound
//     E = 2^-6 |q| |x| (tf32 operands carry <= 2^-10 relative error each, so
//     |2 dot error| <= 2^-8 |q||x| plus fp32 accumulation; 4x margin), so the exact
//     squared distance lies in [a - E, a + E];
//  3. a row can only be the leaf minimum if its lower end a - E does not exceed
//     U = min(best exact so far, min over the tile of a + E); those few rows are
//     re-checked EXACTLY in fp64 direct form by the whole warp (lane-strided
//     partial sums + a fixed shuffle tree), reading x from the resident smem
//     tile, and folded with a 64-bit atomicMin on the bit pattern.
//
// The result is therefore the exact fp64 direct-form minimum (same terms as
// lf_leaf_min_dist, summed in another order: agreement to ~1 ulp), with the
// O(Q N m) work on the tensor cores and only
// O(Q L) exact re-checks (about one per (query, leaf) on random walks).
//
// Warp roles (192 threads, one persistent CTA per SM):
//   warp 0: TMA producer   warp 1: TMEM owner + MMA issuer   warps 2-5: epilogue
#include <cuda.h>
#include <cudaTypedefs.h>

#include <vector>

#include "common.cuh"

namespace lf {
namespace tk {

constexpr int BM = 128;            // queries per tile
constexpr int BN = 128;            // rows per chunk (resident B tile)
constexpr int BK = 32;             // fp32 per 128-byte swizzle row
constexpr int STAGES = 4;
constexpr int THREADS = 192;
constexpr int A_BYTES = BM * BK * 4;           // 16 KiB per stage
constexpr int KB_BYTES = BN * BK * 4;          // 16 KiB per B k-block
constexpr int MAX_KB = 8;                      // m <= 256
constexpr int TMEM_COLS = 512;                 // 4 accumulators x 128 columns
constexpr int NACC = 4;
constexpr int SMEM_BYTES = MAX_KB * KB_BYTES + STAGES * A_BYTES + 1024 + 4096;

struct Item {                      // one leaf against one query range
    int leaf;                      // leaf slot
    int col;                       // output column
    long long q0, q1;              // query rows [q0, q1)
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "LF_W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LF_W_%=;\n}" ::"r"(su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            su32(dst)),
        "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

#define LF_TMEM_LD32(taddr, r)                                                                                 \
    asm volatile(                                                                                              \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"      \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                            \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),    \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),            \
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),          \
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),          \
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                               \
        : "r"(taddr))

// element (row r, dim k) of a resident K-major SWIZZLE_128B tile made of 128-row k-blocks
__device__ __forceinline__ float b_elem(const uint8_t* B, int r, int k) {
    const int kb = k >> 5, kk = k & 31;
    const int chunk = (kk >> 2) ^ (r & 7);
    return *reinterpret_cast<const float*>(B + kb * KB_BYTES + r * 128 + (chunk << 4) + ((kk & 3) << 2));
}

__global__ void __launch_bounds__(THREADS, 1)
mindist_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_x,
                  const Item* __restrict__ items, int n_items, lf_index idx, const float* __restrict__ Qm,
                  const double* __restrict__ qnorm, const double* __restrict__ xnorm,
                  unsigned long long* __restrict__ out, long long ldo) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    uint8_t* Bt = smem;                                         // resident row chunk
    uint8_t* As = smem + MAX_KB * KB_BYTES;                     // query stages
    double* xn_s = reinterpret_cast<double*>(As + STAGES * A_BYTES);      // |x|^2 of the chunk rows
    double* xr_s = xn_s + BN;                                              // |x|
    uint64_t* full = reinterpret_cast<uint64_t*>(xr_s + BN);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + NACC;
    uint64_t* bfull = tempty + NACC;
    uint64_t* bempty = bfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + 1);
    int* cand_list = reinterpret_cast<int*>(tmem_slot + 4);             // 4 epilogue warps x 64 entries

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = idx.m;
    const int n_kb = m / BK;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < NACC; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 4); }
        mbar_init(bfull, 1);
        mbar_init(bempty, 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {                                            // ---- producer (whole warp; lane 0 issues TMA)
        int stage = 0;
        uint32_t phase = 0, bphase = 0;
        for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
            const Item item = items[it];
            const long long lb = idx.d_leaf_ptr[item.leaf], le = idx.d_leaf_ptr[item.leaf + 1];
            const int n_qb = (int)((item.q1 - item.q0 + BM - 1) / BM);
            for (long long r0 = lb; r0 < le; r0 += BN) {
                mbar_wait(bempty, bphase ^ 1);                  // epilogue done with the previous chunk
                for (int i = lane; i < BN; i += 32) {
                    const long long r = r0 + i;
                    const double v = r < le ? xnorm[r] : 0.0;
                    xn_s[i] = v;
                    xr_s[i] = sqrt(v);
                }
                __syncwarp();
                if (lane == 0) {
                    mbar_expect_tx(bfull, (uint32_t)(n_kb * KB_BYTES));
                    for (int kb = 0; kb < n_kb; ++kb) tma_2d(&map_x, bfull, Bt + kb * KB_BYTES, kb * BK, (int)r0);
                }
                bphase ^= 1;
                for (int qb = 0; qb < n_qb; ++qb) {
                    for (int kb = 0; kb < n_kb; ++kb) {
                        if (lane == 0) {
                            mbar_wait(&empty[stage], phase ^ 1);
                            mbar_expect_tx(&full[stage], A_BYTES);
                            tma_2d(&map_q, &full[stage], As + stage * A_BYTES, kb * BK, (int)(item.q0 + qb * BM));
                        }
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {                                     // ---- MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_tf32(BM, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0, bphase = 0;
            for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
                const Item item = items[it];
                const long long lb = idx.d_leaf_ptr[item.leaf], le = idx.d_leaf_ptr[item.leaf + 1];
                const int n_qb = (int)((item.q1 - item.q0 + BM - 1) / BM);
                for (long long r0 = lb; r0 < le; r0 += BN) {
                    mbar_wait(bfull, bphase);
                    bphase ^= 1;
                    fence_after();
                    const uint32_t bs = su32(Bt);
                    for (int qb = 0; qb < n_qb; ++qb) {
                        mbar_wait(&tempty[acc], acc_phase ^ 1);
                        fence_after();
                        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
                        for (int kb = 0; kb < n_kb; ++kb) {
                            mbar_wait(&full[stage], phase);
                            fence_after();
                            const uint32_t as = su32(As + stage * A_BYTES);
#pragma unroll
                            for (int kk = 0; kk < BK / 8; ++kk)
                                mma_tf32(d, sw128_desc(as + kk * 32), sw128_desc(bs + kb * KB_BYTES + kk * 32), idesc,
                                         (kb | kk) != 0 ? 1u : 0u);
                            mma_commit(&empty[stage]);
                            if (++stage == STAGES) { stage = 0; phase ^= 1; }
                        }
                        mma_commit(&tfull[acc]);
                        if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
                    }
                }
            }
        }
    } else {                                                    // ---- epilogue (warps 2..5)
        const int quarter = warp & 3;
        const int row = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0, bphase = 0;
        constexpr double kErr = 1.0 / 64.0;                     // 2^-6 (4x margin)
        for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
            const Item item = items[it];
            const long long lb = idx.d_leaf_ptr[item.leaf], le = idx.d_leaf_ptr[item.leaf + 1];
            const int n_qb = (int)((item.q1 - item.q0 + BM - 1) / BM);
            for (long long r0 = lb; r0 < le; r0 += BN) {
                const int nrows = (int)min((long long)BN, le - r0);
                mbar_wait(bfull, bphase);                       // B tile + norms visible
                bphase ^= 1;
                for (int qb = 0; qb < n_qb; ++qb) {
                    mbar_wait(&tfull[acc], acc_phase);
                    fence_after();
                    const long long q = item.q0 + (long long)qb * BM + row;
                    const bool qv = q < item.q1;
                    const double qn = qv ? qnorm[q] : 0.0;
                    const double qr = sqrt(qn);
                    unsigned long long* dst = out + (qv ? q : 0) * ldo + item.col;
                    double best = qv ? __longlong_as_double((long long)*(volatile unsigned long long*)dst) : 0.0;
                    const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * BN);
                    // pass 1: U = min(best, min_r (a_r + E_r))
                    double U = best;
                    for (int c0 = 0; c0 < BN; c0 += 32) {
                        uint32_t r[32];
                        LF_TMEM_LD32(taddr + (uint32_t)c0, r);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int rr = c0 + j;
                            if (rr < nrows) {
                                const double a = qn + xn_s[rr] - 2.0 * (double)__uint_as_float(r[j]);
                                U = fmin(U, a + kErr * qr * xr_s[rr]);
                            }
                        }
                    }
                    // pass 2: rows whose interval reaches below U are re-checked EXACTLY,
                    // cooperatively: the warp gathers (lane, row) candidates and all 32
                    // lanes sum one candidate at a time (k = lane + 32 i, then a
                    // fixed shuffle tree) -- no 256-long dependent FMA chains.
                    int* list = cand_list + (warp - 2) * 64;
                    int cnt = 0;
                    const long long qbase = item.q0 + (long long)qb * BM + quarter * 32;
                    auto flush = [&]() {
                        for (int e = 0; e < cnt; ++e) {
                            const int ent = list[e];
                            const int owner = ent >> 8, rr = ent & 255;
                            const long long qe = qbase + owner;
                            const float* qrow = Qm + qe * m;
                            double part = 0.0;
                            for (int k = lane; k < m; k += 32) {
                                const double dd = (double)b_elem(Bt, rr, k) - (double)__ldg(qrow + k);
                                part = __fma_rn(dd, dd, part);
                            }
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
                            if (lane == owner && part < best) {
                                best = part;
                                atomicMin(dst, (unsigned long long)__double_as_longlong(part));
                            }
                        }
                        __syncwarp();
                        cnt = 0;
                    };
                    for (int c0 = 0; c0 < BN; c0 += 32) {
                        uint32_t r[32];
                        LF_TMEM_LD32(taddr + (uint32_t)c0, r);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int rr = c0 + j;
                            bool cand = false;
                            if (qv && rr < nrows) {
                                const double a = qn + xn_s[rr] - 2.0 * (double)__uint_as_float(r[j]);
                                cand = a - kErr * qr * xr_s[rr] <= U;
                            }
                            const unsigned mask = __ballot_sync(0xffffffffu, cand);
                            if (mask) {
                                if (cnt + 32 > 64) flush();
                                if (cand) list[cnt + __popc(mask & ((1u << lane) - 1u))] = (lane << 8) | rr;
                                __syncwarp();
                                cnt += __popc(mask);
                            }
                        }
                    }
                    if (cnt) flush();
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[acc]);
                    if (++acc == NACC) { acc = 0; acc_phase ^= 1; }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(bempty);             // chunk's B tile may be replaced
            }
        }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

__global__ void row_norms_kernel(const float* __restrict__ X, int64_t n, int m, double* __restrict__ out) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= n) return;
    double acc = 0.0;
    for (int k = lane; k < m; k += 32) {
        const double v = (double)X[r * m + k];
        acc = __fma_rn(v, v, acc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[r] = acc;
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

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

static int make_map(CUtensorMap* map, const float* base, int64_t rows, int cols, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return fail(LF_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(LF_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return LF_OK;
}

// items -> device, norms, fill, kernel, sqrt
static int run(const float* d_q, int64_t Q, const lf_index& idx, const std::vector<Item>& items,
               double* d_out, int64_t out_rows, int64_t out_cols, int64_t ldo, cudaStream_t st) {
    LF_REQUIRE(idx.m >= 32 && idx.m <= 256 && idx.m % 32 == 0, "tensor-core min-distance needs m in {32,...,256}");
    LF_REQUIRE(((uintptr_t)d_q & 15) == 0 && ((uintptr_t)idx.d_X & 15) == 0, "operands must be 16-byte aligned");
    if (items.empty() || Q == 0) return LF_OK;
    Scratch d_items, qn, xn;
    LF_CUDA(d_items.alloc(sizeof(Item) * items.size(), st));
    LF_CUDA(cudaMemcpyAsync(d_items.p, items.data(), sizeof(Item) * items.size(), cudaMemcpyHostToDevice, st));
    LF_CUDA(qn.alloc(sizeof(double) * Q, st));
    LF_CUDA(xn.alloc(sizeof(double) * idx.n_series, st));
    row_norms_kernel<<<(unsigned)((Q * 32 + 255) / 256), 256, 0, st>>>(d_q, Q, idx.m, qn.as<double>());
    row_norms_kernel<<<(unsigned)((idx.n_series * 32 + 255) / 256), 256, 0, st>>>(idx.d_X, idx.n_series, idx.m,
                                                                                   xn.as<double>());
    fill_bits_kernel<<<(unsigned)((out_rows * out_cols + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<unsigned long long*>(d_out), out_rows, out_cols, ldo, 0x7ff0000000000000ULL);
    LF_CUDA(cudaGetLastError());
    CUtensorMap mq, mx;
    int rc = make_map(&mq, d_q, Q, idx.m, BM);
    if (rc) return rc;
    rc = make_map(&mx, idx.d_X, idx.n_series, idx.m, BN);
    if (rc) return rc;
    LF_CUDA(smem_optin(mindist_tc_kernel, SMEM_BYTES));
    const int grid = (int)std::min<size_t>(items.size(), (size_t)sm_count());
    mindist_tc_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(mq, mx, d_items.as<Item>(), (int)items.size(), idx, d_q,
                                                         qn.as<double>(), xn.as<double>(),
                                                         reinterpret_cast<unsigned long long*>(d_out), ldo);
    LF_CUDA(cudaGetLastError());
    sqrt_bits_kernel<<<(unsigned)((out_rows * out_cols + 255) / 256), 256, 0, st>>>(d_out, out_rows, out_cols, ldo);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

}  // namespace tk
}  // namespace lf

extern "C" int lf_leaf_min_dist_tc(const float* d_queries, int64_t Q, const lf_index* idx,
                                   const int32_t* h_leaf_sel, int32_t S, double* d_dl, int64_t ldd,
                                   void* stream) {
    using namespace lf;
    LF_REQUIRE(idx != nullptr && Q >= 0 && S >= 0 && ldd >= S, "bad arguments");
    std::vector<tk::Item> items;
    items.reserve(S);
    for (int s = 0; s < S; ++s) items.push_back(tk::Item{h_leaf_sel[s], s, 0, Q});
    return tk::run(d_queries, Q, *idx, items, d_dl, Q, S, ldd, as_stream(stream));
}

extern "C" int lf_local_min_dist_tc(const float* d_queries, const lf_index* idx, const int64_t* h_qptr,
                                    const int32_t* h_group_leaf, int32_t n_groups, double* d_dl, void* stream) {
    using namespace lf;
    LF_REQUIRE(idx != nullptr && n_groups >= 0, "bad arguments");
    if (n_groups == 0) return LF_OK;
    const int64_t Q = h_qptr[n_groups];
    std::vector<tk::Item> items;
    items.reserve(n_groups);
    for (int g = 0; g < n_groups; ++g)
        if (h_qptr[g + 1] > h_qptr[g]) items.push_back(tk::Item{h_group_leaf[g], 0, h_qptr[g], h_qptr[g + 1]});
    return tk::run(d_queries, Q, *idx, items, d_dl, Q, 1, 1, as_stream(stream));
}
