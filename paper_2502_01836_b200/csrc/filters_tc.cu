// K3 on the 5th-generation tensor cores: grouped filter GEMM with a fused
// bias / rectifier / W2-dot epilogue.
//
//   pred[q, f] = b2[f] + sum_j W2[f, j] * relu(b1[f, j] + sum_i X[q, i] * W1[f, i, j])
//   (mlp.py:90-95, evaluated for every (query, filter) pair; tree.py:278-286)
//
// Per tile (filter f, 128 queries): D[128 x m] = X_tile[128 x m] . W1_f[m x m]
// with tcgen05.mma.kind::tf32 (M=128, N=m<=256, K=8 per instruction), operands
// staged by TMA (SWIZZLE_128B, K-major: W1 is pre-transposed to [F][hidden][in])
// through a 4-stage mbarrier pipeline, fp32 accumulators in TMEM (two 256-column
// buffers so the epilogue of tile i overlaps the MMAs of tile i+1).  The
// epilogue warps read their accumulator row with tcgen05.ld and fold bias,
// rectifier and the W2 dot product in registers -- H never leaves the SM.
//
// Warp roles (320 threads, one persistent CTA per SM):
//   warp 0: TMA producer    warp 1: TMEM owner + MMA issuer    warps 2-9: epilogue
//
// Batch invariance: an output's K order (k-blocks, then the four
// K=8 MMAs inside a block) and its j order in the epilogue depend only on m,
// never on Q or on the tile a query falls in.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"

namespace lf {
namespace tc {

constexpr int BM = 128;          // queries per tile (UMMA M)
constexpr int BK = 32;           // fp32 elements per 128-byte swizzle row (fp16: 64)
constexpr int STAGES = 4;
constexpr int THREADS = 320;          // producer, MMA issuer, 8 epilogue warps
constexpr int A_BYTES = BM * BK * 4;          // 16 KiB
constexpr int B_BYTES_MAX = 256 * 128;        // 32 KiB (N = m <= 256, 128-byte rows)
constexpr int STAGE_BYTES = A_BYTES + B_BYTES_MAX;
constexpr int TMEM_COLS = 512;                // 2 accumulator buffers x 256 columns
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + 4096 /*b1, W2 x 2*/ +
                           1024 /*half-row partials x 2*/;

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
        "LF_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LF_WAIT_%=;\n}" ::"r"(su32(b)),
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
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
                 : "memory");
}

// K-major, SWIZZLE_128B UMMA shared-memory descriptor (cute::UMMA::SmemDescriptor):
// start>>4 | LBO(16 B, unused for swizzled K-major)>>4 <<16 | SBO(1024 B: 8 rows x 128 B)>>4 <<32
// | version 1 <<46 | layout SWIZZLE_128B (2) <<61.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// Instruction descriptor: D f32, A/B f16, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
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

// PAIRS = false: every (query, filter) pair, tiles (f, 128-query block), dense pred [Q][F].
// PAIRS = true : a device tile list (f, first row, rows) over GATHERED query rows
//                (one row per (query, visit-order position) pair, grouped by filter);
//                the epilogue writes adj[q][pos] = pred - offset[f] straight into the
//                search's visit-order records.  Same MMA K order and epilogue order
//                as the dense kernel, so every prediction is bit-identical to it.
struct PairArgs {
    const int4* tiles;           // (filter, first gathered row, rows, 0)
    const int* n_tiles;          // device count
    const int2* dst;             // per gathered row: (query, visit-order position)
    const double* offset;        // [F]
    double* adj;                 // [Q][Nn]
    int Nn;
    int dbg;                     // LF_REACH_DBG (measurement only): 1 fixed gather rows, 2 no W1 load, 4 no W1 prefetch
};

// fp16 operands (F16 = true): each X row and each filter's W1 is stored scaled by a
// power of two (max |value| in [2^13, 2^14), exact), so fp16 keeps tf32's 10-bit
// mantissa without overflow; the epilogue multiplies the accumulator back by
// 2^(xexp[row] + wexp[f]) -- exact -- before the bias.
struct F16Args {
    const int* xexp;             // per X row (dense: query; pairs: gathered row; GATHER: query)
    const int* wexp;             // per filter
    const uint8_t* xrows;        // GATHER: fp16 query rows [Q][m]
};

// GATHER (with PAIRS and F16): the A operand is not a materialised row list but the
// batch's fp16 query matrix (F16Args.xrows, L2-resident); the producer warp copies each
// tile's 128 query rows straight into the SW128 K-major stage layout with cp.async
// (16-byte chunk c of row r at r * 128 + ((c ^ (r & 7)) * 16)), and each lane's copies
// arrive on the stage's full barrier when they land (cp.async.mbarrier.arrive.noinc).
// TMA tile::gather4 (4 rows per instruction) did the same at ~7 us per tile against
// ~2 us with cp.async: the TMA unit serialises the 128 row fetches of a tile.
template <bool PAIRS, bool F16, bool GATHER = false>
__global__ void __launch_bounds__(THREADS, 1)
filter_tc_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                 int64_t Q, int m, int F, const float* __restrict__ b1, const float* __restrict__ W2,
                 const float* __restrict__ b2, float* __restrict__ pred, PairArgs pa, F16Args fa) {
    constexpr int BKE = F16 ? 64 : BK;               // elements per 128-byte K block
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);   // stays in the shared window
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_mb = (int)((Q + BM - 1) / BM);
    const int64_t n_tiles = PAIRS ? (int64_t)*pa.n_tiles : (int64_t)F * n_mb;
    const int n_kb = m / BKE;
    const uint32_t b_bytes = (uint32_t)m * 128;

    if (warp == 0 && lane == 0) {
        // GATHER: the stage's W1 TMA (lane 0's expect_tx arrive) + one cp.async arrive per lane
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], GATHER ? 33 : 1); mbar_init(&empty[s], 1); }
        for (int s = 0; s < 2; ++s) { mbar_init(&tfull[s], 1); mbar_init(&tempty[s], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (!GATHER) asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (GATHER && warp == 0) {                               // ---- producer, gathered A
        // Each tile is (usually) a new filter whose W1 (m x m fp16, 128 KiB) comes from
        // DRAM: the next tiles' W1 is prefetched into L2 one and two tiles ahead, and the
        // next tile's rows are looked up while this tile's stages are issued.
        int stage = 0;
        uint32_t phase = 0;
        const int row_bytes = m * 2;
        const int64_t g = gridDim.x;
        // tile descriptors three tiles deep in registers: no load feeds a use in the
        // same tile (a dependent global load per tile cost ~1 us of producer time)
        auto tile_at = [&](int64_t tt) { return tt < n_tiles ? pa.tiles[tt] : make_int4(0, 0, 1, 0); };
        auto prefetch_w = [&](int64_t tt, int ff) {
            if (lane == 0 && tt < n_tiles && !(pa.dbg & 4))
                for (int kb = 0; kb < n_kb; ++kb)
                    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&map_w),
                                 "r"(kb * BKE), "r"(ff * m)
                                 : "memory");
        };
        auto rows_of = [&](int64_t tt, const int4& tl, int* q4) {   // lane owns tile rows lane + 32 j
            if (tt < n_tiles) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    q4[j] = (pa.dbg & 1) ? lane + 32 * j : pa.dst[tl.y + min(lane + 32 * j, tl.z - 1)].x;
            }
        };
        int4 T0 = tile_at(blockIdx.x), T1 = tile_at(blockIdx.x + g), T2 = tile_at(blockIdx.x + 2 * g);
        int qi[4] = {0, 0, 0, 0}, qn[4] = {0, 0, 0, 0};
        prefetch_w(blockIdx.x, T0.x);
        prefetch_w(blockIdx.x + g, T1.x);
        rows_of(blockIdx.x, T0, qi);
        for (int64_t t = blockIdx.x; t < n_tiles; t += g) {
            const int f = T0.x;
            const int4 T3 = tile_at(t + 3 * g);                  // used two tiles from now
            prefetch_w(t + 2 * g, T2.x);
            rows_of(t + g, T1, qn);                              // in flight while this tile is issued
            for (int kb = 0; kb < n_kb; ++kb) {
                if (lane == 0) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], (pa.dbg & 2) ? 0u : b_bytes);
                    if (!(pa.dbg & 2)) tma_2d(&map_w, &full[stage], smem + stage * STAGE_BYTES + A_BYTES, kb * BKE, f * m);
                }
                __syncwarp();
                const uint32_t sa = su32(smem + stage * STAGE_BYTES);
                // 8 lanes per row, 4 rows (four whole 128-byte lines) per instruction; the row's
                // query comes from the lane that owns it (rows lane + 32 j)
                const int c = lane & 7;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int r = 4 * j + (lane >> 3);
                    const int qr = __shfl_sync(0xffffffffu, qi[j >> 3], r & 31);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa + r * 128 + ((c ^ (r & 7)) << 4)),
                                 "l"(fa.xrows + (int64_t)qr * row_bytes + kb * 128 + c * 16)
                                 : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[stage])) : "memory");
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) qi[j] = qn[j];
            T0 = T1;
            T1 = T2;
            T2 = T3;
        }
    } else if (warp == 0) {
        if (lane == 0) {                                     // ---- TMA producer
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                int f, row0;
                if (PAIRS) {
                    const int4 tl = pa.tiles[t];
                    f = tl.x;
                    row0 = tl.y;
                } else {
                    f = (int)(t / n_mb);
                    row0 = (int)(t % n_mb) * BM;
                }
                for (int kb = 0; kb < n_kb; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + stage * STAGE_BYTES;
                    uint8_t* sb = sa + A_BYTES;
                    mbar_expect_tx(&full[stage], A_BYTES + b_bytes);
                    tma_2d(&map_x, &full[stage], sa, kb * BKE, row0);
                    tma_2d(&map_w, &full[stage], sb, kb * BKE, f * m);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {                                     // ---- MMA issuer (single thread)
            const uint32_t idesc = F16 ? idesc_f16(BM, m) : idesc_tf32(BM, m);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);      // epilogue drained this buffer
                tc_fence_after();
                const uint32_t d = tmem_base + (uint32_t)(acc * 256);
                for (int kb = 0; kb < n_kb; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    // GATHER: A was written by cp.async (generic proxy), read by the MMA (async proxy)
                    if (GATHER) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const uint32_t sa = su32(smem + stage * STAGE_BYTES);
                    const uint32_t sb = sa + A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {             // K = 8 tf32 / 16 f16 = 32 bytes per MMA
                        if (F16)
                            mma_f16(d, sw128_desc(sa + kk * 32), sw128_desc(sb + kk * 32), idesc,
                                    (kb | kk) != 0 ? 1u : 0u);
                        else
                            mma_tf32(d, sw128_desc(sa + kk * 32), sw128_desc(sb + kk * 32), idesc,
                                     (kb | kk) != 0 ? 1u : 0u);
                    }
                    mma_commit(&empty[stage]);                  // smem slot free once these MMAs retire
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[acc]);                        // accumulator ready for the epilogue
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {                                                 // ---- epilogue (warps 2..9)
        // b1[f] / W2[f] (2 x m floats) are staged in shared memory one tile ahead with
        // cp.async by the epilogue threads: each tile is a new filter for this CTA,
        // so reading them with per-column global loads paid an L2 round trip per chunk.
        // Two warps per TMEM lane quarter: half 0 (warps 2-5) folds columns [0, hc),
        // half 1 (warps 6-9) columns [hc, m); half 1 hands its partial to half 0 through
        // shared memory (double-buffered by tile parity, one named barrier per pair).
        const int et = threadIdx.x - 64;                     // 0..255
        const int quarter = warp & 3;                        // TMEM lanes [32*quarter, +32)
        const int half = (warp - 2) >> 2;
        const int row = quarter * 32 + lane;
        const int hc = ((m >> 1) + 31) & ~31;                // half 0's columns
        const int c_begin = half ? hc : 0, c_end = half ? m : hc;
        float* pbuf = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);   // [2][2][256]
        float* xbuf = pbuf + 2 * 512;                                               // [2][128]
        // Every per-tile scalar is fetched ahead so no global round trip sits between
        // two tiles: the tile descriptor two tiles ahead, the next tile's per-row pair
        // (query, position), b2, offset and filter exponent at the start of this tile,
        // and its query exponent (dependent on the pair) after this tile's columns.
        struct Tile { int f, row0, nrows; };
        auto tile_of = [&](int64_t t) -> Tile {
            if (t >= n_tiles) return Tile{0, 0, 0};
            if (PAIRS) {
                const int4 tl = pa.tiles[t];
                return Tile{tl.x, tl.y, tl.z};
            }
            return Tile{(int)(t / n_mb), (int)(t % n_mb) * BM, BM};
        };
        struct RowVals { int2 d; float b2v; double off; int wex; int ex; bool valid; };
        auto row_vals = [&](const Tile& T, int64_t t) -> RowVals {     // independent loads only
            RowVals v{make_int2(0, 0), 0.f, 0.0, 0, 0, false};
            if (t >= n_tiles) return v;
            const int64_t xr = (int64_t)T.row0 + row;
            v.valid = PAIRS ? row < T.nrows : xr < Q;
            if (PAIRS && v.valid) v.d = pa.dst[xr];
            v.b2v = b2[T.f];
            if (PAIRS && pa.offset != nullptr) v.off = pa.offset[T.f];
            if (F16) v.wex = fa.wexp[T.f];
            return v;
        };
        auto row_exp = [&](RowVals& v, const Tile& T) {                   // the dependent level
            if (F16 && v.valid) v.ex = GATHER ? fa.xexp[v.d.x] : fa.xexp[(int64_t)T.row0 + row];
        };
        auto stage_params = [&](const Tile& T, int64_t t, int slot) {
            if (t < n_tiles) {
                const int chunks = m >> 2;                   // 16-byte chunks per vector
                if (et < 2 * chunks) {
                    const float* src = (et < chunks ? b1 + (int64_t)T.f * m + et * 4
                                                    : W2 + (int64_t)T.f * m + (et - chunks) * 4);
                    float* dst = pbuf + slot * 512 + (et < chunks ? et * 4 : 256 + (et - chunks) * 4);
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(su32(dst)), "l"(src) : "memory");
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        int acc = 0;
        uint32_t acc_phase = 0;
        int slot = 0;
        const int64_t g = gridDim.x;
        Tile cur = tile_of(blockIdx.x), nxt = tile_of(blockIdx.x + g), nn = tile_of(blockIdx.x + 2 * g);
        stage_params(cur, blockIdx.x, 0);
        RowVals rv = row_vals(cur, blockIdx.x);
        row_exp(rv, cur);
        for (int64_t t = blockIdx.x; t < n_tiles; t += g) {
            const int f = cur.f, nrows = cur.nrows;
            (void)nrows;
            stage_params(nxt, t + g, slot ^ 1);
            RowVals rn = row_vals(nxt, t + g);               // lands while this tile is folded
            const Tile n3 = tile_of(t + 3 * g);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            asm volatile("bar.sync 1, 256;" ::: "memory");   // this tile's parameters visible
            const float4* b1s = reinterpret_cast<const float4*>(pbuf + slot * 512);
            const float4* w2s = reinterpret_cast<const float4*>(pbuf + slot * 512 + 256);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            float part = 0.f;
            // F16: undo the operands' scaling (exact power of two)
            const float sc = F16 ? scalbnf(1.f, rv.valid ? rv.ex + rv.wex : rv.wex) : 1.f;
            const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(acc * 256);
            for (int c0 = c_begin; c0 < c_end; c0 += 64) {     // two 32-column loads per wait
                uint32_t r[2][32];
                const bool two = c0 + 32 < c_end;                 // warp-uniform
                LF_TMEM_LD32(taddr + (uint32_t)c0, r[0]);
                if (two) LF_TMEM_LD32(taddr + (uint32_t)(c0 + 32), r[1]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    if (hh == 1 && !two) break;
                    const int cb = c0 + hh * 32;
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        const float4 bb = b1s[(cb >> 2) + j4];
                        const float4 ww = w2s[(cb >> 2) + j4];
                        const float bv[4] = {bb.x, bb.y, bb.z, bb.w};
                        const float wv[4] = {ww.x, ww.y, ww.z, ww.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            // F16: acc * 2^e is exact, so one FFMA rounds exactly like FMUL + FADD
                            const float a = __uint_as_float(r[hh][j4 * 4 + u]);
                            const float h = F16 ? fmaxf(__fmaf_rn(a, sc, bv[u]), 0.f) : fmaxf(__fadd_rn(a, bv[u]), 0.f);
                            part = __fmaf_rn(h, wv[u], part);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            row_exp(rn, nxt);                                // rn.d has landed by now
            if (half) xbuf[slot * 128 + row] = part;
            asm volatile("bar.sync %0, 64;" ::"r"(2 + quarter) : "memory");   // the quarter's two warps
            if (half == 0 && rv.valid) {
                part = __fadd_rn(part, xbuf[slot * 128 + row]);
                if (PAIRS) {
                    const double pv = (double)__fadd_rn(part, rv.b2v);
                    pa.adj[(int64_t)rv.d.x * pa.Nn + rv.d.y] = pa.offset != nullptr ? pv - rv.off : pv;
                } else {
                    pred[((int64_t)cur.row0 + row) * F + f] = __fadd_rn(part, rv.b2v);
                }
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");   // slot free for the tile after next
            slot ^= 1;
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            cur = nxt;
            nxt = nn;
            nn = n3;
            rv = rn;
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
    }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link).
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

static int make_map(CUtensorMap* map, const void* base, int64_t rows, int cols, int box_rows, bool f16 = false) {
    auto fn = encode_fn();
    if (!fn) return fail(LF_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const int esize = f16 ? 2 : 4;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * esize};
    cuuint32_t box[2] = {(cuuint32_t)(128 / esize), (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                    const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(LF_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return LF_OK;
}

}  // namespace tc
}  // namespace lf

extern "C" int lf_filter_predict_tc(const float* d_queries, int64_t Q, int32_t m, const float* d_W1T,
                                    const float* d_b1, const float* d_W2, const float* d_b2, int32_t F,
                                    float* d_pred, void* stream) {
    using namespace lf;
    LF_REQUIRE(Q >= 0 && F >= 0, "bad sizes");
    LF_REQUIRE(m >= 32 && m <= 256 && m % 32 == 0, "tensor-core filter path needs m in {32, 64, ..., 256}");
    LF_REQUIRE(((uintptr_t)d_queries & 15) == 0 && ((uintptr_t)d_W1T & 15) == 0 && ((uintptr_t)d_b1 & 15) == 0 &&
                   ((uintptr_t)d_W2 & 15) == 0,
               "operands must be 16-byte aligned");
    if (Q == 0 || F == 0) return LF_OK;
    CUtensorMap mx, mw;
    int rc = tc::make_map(&mx, d_queries, Q, m, tc::BM);
    if (rc) return rc;
    rc = tc::make_map(&mw, d_W1T, (int64_t)F * m, m, m);
    if (rc) return rc;
    const int n_mb = (int)((Q + tc::BM - 1) / tc::BM);
    LF_CUDA(smem_optin(tc::filter_tc_kernel<false, false>, tc::SMEM_BYTES));
    const int64_t tiles = (int64_t)F * n_mb;
    const int grid = (int)std::min<int64_t>(tiles, sm_count());
    tc::filter_tc_kernel<false, false><<<grid, tc::THREADS, tc::SMEM_BYTES, as_stream(stream)>>>(
        mx, mw, Q, m, F, d_b1, d_W2, d_b2, d_pred, tc::PairArgs{}, tc::F16Args{});
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

namespace lf {
// Predictions for gathered (query, position) rows grouped by filter (lazy inference
// inside lf_search): d_rows [P][m], tile list and count on the device.
int filter_pairs_tc(const float* d_rows, int64_t P, int m, const float* d_W1T, const float* d_b1,
                    const float* d_W2, const float* d_b2, int F, const int4* d_tiles, const int* d_ntiles,
                    const int2* d_dst, const double* d_offset, double* d_adj, int Nn, cudaStream_t st) {
    if (P == 0 || F == 0) return LF_OK;
    CUtensorMap mx, mw;
    int rc = tc::make_map(&mx, d_rows, P, m, tc::BM);
    if (rc) return rc;
    rc = tc::make_map(&mw, d_W1T, (int64_t)F * m, m, m);
    if (rc) return rc;
    LF_CUDA(smem_optin(tc::filter_tc_kernel<true, false>, tc::SMEM_BYTES));
    tc::PairArgs pa{d_tiles, d_ntiles, d_dst, d_offset, d_adj, Nn};
    tc::filter_tc_kernel<true, false><<<sm_count(), tc::THREADS, tc::SMEM_BYTES, st>>>(mx, mw, P, m, F, d_b1, d_W2,
                                                                                      d_b2, nullptr, pa,
                                                                                      tc::F16Args{});
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
}  // namespace lf

// ---------------------------------------------------------------------------
// Explicit (query, filter) pair list: bucket by filter, gather, pair GEMM.
namespace lf {
namespace tc {
__global__ void pair_hist_kernel(const int32_t* __restrict__ pf, int64_t P, int* __restrict__ hist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P) atomicAdd(&hist[pf[i]], 1);
}
__global__ void pair_bucket_q_kernel(const int32_t* __restrict__ pq, const int32_t* __restrict__ pf, int64_t P,
                                     int* __restrict__ fcur, int2* __restrict__ dst) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P) dst[atomicAdd(&fcur[pf[i]], 1)] = make_int2(pq[i], (int)i);
}
__global__ void pair_bucket_kernel(const float* __restrict__ queries, int m, const int32_t* __restrict__ pq,
                                   const int32_t* __restrict__ pf, int64_t P, int* __restrict__ fcur,
                                   int2* __restrict__ dst, float* __restrict__ rows) {
    const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= P) return;
    int slot = 0;
    if (lane == 0) {
        slot = atomicAdd(&fcur[pf[i]], 1);
        dst[slot] = make_int2((int)i, 0);
    }
    slot = __shfl_sync(0xffffffffu, slot, 0);
    const float* src = queries + (int64_t)pq[i] * m;
    for (int c = lane; c < m; c += 32) rows[(int64_t)slot * m + c] = src[c];
}
}  // namespace tc
int pair_tiles(const int* d_hist, int F, int* d_fcur, int4* d_tiles, int* d_ntiles, cudaStream_t st, int stride = 0);
}  // namespace lf

extern "C" int lf_filter_predict_pairs_tc(const float* d_queries, int32_t m, const float* d_W1T, const float* d_b1,
                                          const float* d_W2, const float* d_b2, int32_t F, const int32_t* d_pair_q,
                                          const int32_t* d_pair_f, int64_t P, double* d_out, void* stream) {
    using namespace lf;
    LF_REQUIRE(m >= 32 && m <= 256 && m % 32 == 0, "tensor-core filter path needs m in {32, 64, ..., 256}");
    LF_REQUIRE(P >= 0 && F >= 1, "bad sizes");
    LF_REQUIRE(((uintptr_t)d_b1 & 15) == 0 && ((uintptr_t)d_W2 & 15) == 0, "b1 / W2 must be 16-byte aligned");
    if (P == 0) return LF_OK;
    cudaStream_t st = as_stream(stream);
    Scratch hist, fcur, tiles, ntiles, dst, rows;
    LF_CUDA(hist.alloc(sizeof(int) * F, st));
    LF_CUDA(fcur.alloc(sizeof(int) * F, st));
    LF_CUDA(tiles.alloc(sizeof(int4) * (size_t)(P / 128 + F + 1), st));
    LF_CUDA(ntiles.alloc(sizeof(int), st));
    LF_CUDA(dst.alloc(sizeof(int2) * (size_t)P, st));
    LF_CUDA(rows.alloc(sizeof(float) * (size_t)P * m, st));
    LF_CUDA(cudaMemsetAsync(hist.p, 0, sizeof(int) * F, st));
    tc::pair_hist_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(d_pair_f, P, hist.as<int>());
    LF_CUDA(cudaGetLastError());
    int rc = pair_tiles(hist.as<int>(), F, fcur.as<int>(), tiles.as<int4>(), ntiles.as<int>(), st);
    if (rc) return rc;
    tc::pair_bucket_kernel<<<(unsigned)((P * 32 + 255) / 256), 256, 0, st>>>(d_queries, m, d_pair_q, d_pair_f, P,
                                                                            fcur.as<int>(), dst.as<int2>(),
                                                                            rows.as<float>());
    LF_CUDA(cudaGetLastError());
    return filter_pairs_tc(rows.as<float>(), P, m, d_W1T, d_b1, d_W2, d_b2, F, tiles.as<int4>(), ntiles.as<int>(),
                           dst.as<int2>(), nullptr, d_out, 1, st);
}

// ---------------------------------------------------------------------------
// fp16 operands: rows scaled by a power of two into fp16 (exact scaling, RN to
// fp16's 10-bit mantissa -- tf32's precision), kind::f16 MMAs at twice the tf32 rate.
namespace lf {
namespace tc {
__global__ void rows_to_f16_kernel(const float* __restrict__ X, int64_t rows, int m, __half* __restrict__ out,
                                   int* __restrict__ exps, int mo) {
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const float* x = X + r * m;
    float amax = 0.f;
    for (int c = lane; c < m; c += 32) amax = fmaxf(amax, fabsf(x[c]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    const int e = amax > 0.f ? ilogbf(amax) - 13 : 0;    // max |x| 2^-e in [2^13, 2^14)
    for (int c = lane; c < m; c += 32) out[r * mo + c] = __float2half_rn(scalbnf(x[c], -e));
    for (int c = m + lane; c < mo; c += 32) out[r * mo + c] = __float2half_rn(0.f);   // zero padding
    if (lane == 0) exps[r] = e;
}
}  // namespace tc

int rows_to_f16(const float* d_X, int64_t rows, int m, __half* d_out, int* d_exps, cudaStream_t st, int mo) {
    if (rows == 0) return LF_OK;
    tc::rows_to_f16_kernel<<<(unsigned)((rows * 32 + 255) / 256), 256, 0, st>>>(d_X, rows, m, d_out, d_exps,
                                                                                 mo > 0 ? mo : m);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
}  // namespace lf

extern "C" int lf_filter_rows_to_f16(const float* d_X, int64_t rows, int32_t m, uint16_t* d_out, int32_t* d_exps,
                                     void* stream) {
    using namespace lf;
    LF_REQUIRE(rows >= 0 && m >= 1, "bad sizes");
    return rows_to_f16(d_X, rows, m, reinterpret_cast<__half*>(d_out), d_exps, as_stream(stream));
}

extern "C" int lf_filter_predict_f16(const float* d_queries, int64_t Q, int32_t m, const uint16_t* d_W1T_h,
                                     const int32_t* d_wexp, const float* d_b1, const float* d_W2, const float* d_b2,
                                     int32_t F, float* d_pred, void* stream) {
    using namespace lf;
    LF_REQUIRE(Q >= 0 && F >= 0, "bad sizes");
    LF_REQUIRE(m >= 64 && m <= 256 && m % 64 == 0, "fp16 filter path needs m in {64, 128, 192, 256}");
    LF_REQUIRE(((uintptr_t)d_W1T_h & 15) == 0 && ((uintptr_t)d_b1 & 15) == 0 && ((uintptr_t)d_W2 & 15) == 0,
               "operands must be 16-byte aligned");
    if (Q == 0 || F == 0) return LF_OK;
    cudaStream_t st = as_stream(stream);
    Scratch xh, xe;
    LF_CUDA(xh.alloc(sizeof(__half) * (size_t)Q * m, st));
    LF_CUDA(xe.alloc(sizeof(int) * (size_t)Q, st));
    int rc = rows_to_f16(d_queries, Q, m, xh.as<__half>(), xe.as<int>(), st);
    if (rc) return rc;
    CUtensorMap mx, mw;
    rc = tc::make_map(&mx, xh.p, Q, m, tc::BM, true);
    if (rc) return rc;
    rc = tc::make_map(&mw, d_W1T_h, (int64_t)F * m, m, m, true);
    if (rc) return rc;
    const int n_mb = (int)((Q + tc::BM - 1) / tc::BM);
    LF_CUDA(smem_optin(tc::filter_tc_kernel<false, true>, tc::SMEM_BYTES));
    const int64_t tiles = (int64_t)F * n_mb;
    const int grid = (int)std::min<int64_t>(tiles, sm_count());
    tc::filter_tc_kernel<false, true><<<grid, tc::THREADS, tc::SMEM_BYTES, st>>>(
        mx, mw, Q, m, F, d_b1, d_W2, d_b2, d_pred, tc::PairArgs{}, tc::F16Args{xe.as<int>(), d_wexp});
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}

namespace lf {
// In-search filter inference over gathered query rows (lf_search with d_W1T_h): tile
// list (filter, first pair, pairs) and per-pair (query, visit-order position) on the
// device; adj[q][pos] = pred - offset.  Bit-identical to lf_filter_predict_f16.
int filter_reach_f16(const __half* d_xh, const int* d_xexp, int64_t Q, int m, const uint16_t* d_W1T_h,
                     const int* d_wexp, const float* d_b1, const float* d_W2, const float* d_b2, int F,
                     const int4* d_tiles, const int* d_ntiles, const int2* d_dst, const double* d_offset,
                     double* d_adj, int Nn, cudaStream_t st) {
    if (Q == 0 || F == 0) return LF_OK;
    CUtensorMap mw;
    CUtensorMap mx{};                                            // unused: A is gathered with cp.async
    int rc = tc::make_map(&mw, d_W1T_h, (int64_t)F * m, m, m, true);
    if (rc) return rc;
    LF_CUDA(smem_optin(tc::filter_tc_kernel<true, true, true>, tc::SMEM_BYTES));
    static const int dbg = getenv("LF_REACH_DBG") ? atoi(getenv("LF_REACH_DBG")) : 0;
    tc::PairArgs pa{d_tiles, d_ntiles, d_dst, d_offset, d_adj, Nn, dbg};
    tc::filter_tc_kernel<true, true, true><<<sm_count(), tc::THREADS, tc::SMEM_BYTES, st>>>(
        mx, mw, Q, m, F, d_b1, d_W2, d_b2, nullptr, pa,
        tc::F16Args{d_xexp, d_wexp, reinterpret_cast<const uint8_t*>(d_xh)});
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
}  // namespace lf

extern "C" int lf_filter_predict_pairs_f16(const float* d_queries, int64_t Q, int32_t m, const uint16_t* d_W1T_h,
                                           const int32_t* d_wexp, const float* d_b1, const float* d_W2,
                                           const float* d_b2, int32_t F, const int32_t* d_pair_q,
                                           const int32_t* d_pair_f, int64_t P, double* d_out, void* stream) {
    using namespace lf;
    LF_REQUIRE(m >= 64 && m <= 256 && m % 64 == 0, "fp16 filter path needs m in {64, 128, 192, 256}");
    LF_REQUIRE(P >= 0 && F >= 1 && Q >= 1, "bad sizes");
    LF_REQUIRE(((uintptr_t)d_W1T_h & 15) == 0 && ((uintptr_t)d_b1 & 15) == 0 && ((uintptr_t)d_W2 & 15) == 0,
               "operands must be 16-byte aligned");
    if (P == 0) return LF_OK;
    cudaStream_t st = as_stream(stream);
    Scratch hist, fcur, tiles, ntiles, dst, xh, xe;
    LF_CUDA(hist.alloc(sizeof(int) * F, st));
    LF_CUDA(fcur.alloc(sizeof(int) * F, st));
    LF_CUDA(tiles.alloc(sizeof(int4) * (size_t)(P / 128 + F + 1), st));
    LF_CUDA(ntiles.alloc(sizeof(int), st));
    LF_CUDA(dst.alloc(sizeof(int2) * (size_t)P, st));
    LF_CUDA(xh.alloc(sizeof(__half) * (size_t)Q * m, st));
    LF_CUDA(xe.alloc(sizeof(int) * (size_t)Q, st));
    int rc = rows_to_f16(d_queries, Q, m, xh.as<__half>(), xe.as<int>(), st);
    if (rc) return rc;
    LF_CUDA(cudaMemsetAsync(hist.p, 0, sizeof(int) * F, st));
    tc::pair_hist_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(d_pair_f, P, hist.as<int>());
    LF_CUDA(cudaGetLastError());
    rc = pair_tiles(hist.as<int>(), F, fcur.as<int>(), tiles.as<int4>(), ntiles.as<int>(), st);
    if (rc) return rc;
    tc::pair_bucket_q_kernel<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(d_pair_q, d_pair_f, P, fcur.as<int>(),
                                                                          dst.as<int2>());
    LF_CUDA(cudaGetLastError());
    // Nn = 0: adj[q * 0 + i] is out[i]
    return filter_reach_f16(xh.as<__half>(), xe.as<int>(), Q, m, d_W1T_h, d_wexp, d_b1, d_W2, d_b2, F,
                            tiles.as<int4>(), ntiles.as<int>(), dst.as<int2>(), nullptr, d_out, 0, st);
}
