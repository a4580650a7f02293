// Conformal auto-tuner fitting on the GPU: the replay of the
// filtered search over the calibration skeleton (conformal.py:171-198) for R
// offset vectors at once -- one thread per (offset vector, calibration query),
// threads of a warp share a query so the skeleton reads broadcast.  Along a
// query's visit order the bound only grows and the best-so-far only shrinks, so a
// thread stops at the first position whose bound exceeds its best-so-far (the
// reference stops when no query is alive; same result per query).  Comparisons and
// minima only: bit-identical to calibration.replay_many.
#include "common.cuh"

namespace lf {

__global__ void replay_kernel(const double* __restrict__ lb, const double* __restrict__ dl,
                              const double* __restrict__ pred, const int32_t* __restrict__ slot, int64_t nq, int L,
                              const double* __restrict__ off, int64_t R, int F, double* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= R * nq) return;
    const int64_t q = t / R, r = t - q * R;         // consecutive threads: same query, other offset vectors
    const double* lbq = lb + q * L;
    const double* dlq = dl + q * L;
    const double* pq = pred + q * L;
    const int32_t* sq = slot + q * L;
    const double* offr = off + r * F;
    double bsf = kInf;
    for (int p = 0; p < L; ++p) {
        if (!(lbq[p] <= bsf)) break;                // conformal.py:180 (alive = lb <= bsf)
        const double pr = pq[p];
        const int s = sq[p];
        const double o = (s >= 0 && F > 0) ? offr[s] : 0.0;
        const bool filt = !isnan(pr) && (pr - o) > bsf;
        if (!filt) bsf = fmin(bsf, dlq[p]);
    }
    out[r * nq + q] = bsf;
}

}  // namespace lf

extern "C" int lf_replay_offsets(const double* d_lb, const double* d_dl, const double* d_pred, const int32_t* d_slot,
                                 int64_t nq, int32_t L, const double* d_offsets, int64_t R, int32_t F, double* d_out,
                                 void* stream) {
    LF_REQUIRE(nq >= 0 && L >= 0 && R >= 0 && F >= 0, "bad sizes");
    if (nq == 0 || R == 0) return LF_OK;
    const int64_t n = nq * R;
    lf::replay_kernel<<<(unsigned)((n + 255) / 256), 256, 0, lf::as_stream(stream)>>>(d_lb, d_dl, d_pred, d_slot, nq,
                                                                                    L, d_offsets, R, F, d_out);
    LF_CUDA(cudaGetLastError());
    return LF_OK;
}
