#pragma once
#include <cuda_runtime.h>

#include "../../include/leafi_b200.h"

namespace lf {
int launch_bounds(const float* d_q, int64_t Q, const lf_index& idx, const double* env_min,
                  const double* env_max, int n_env, int mode, double* d_qsumm, double* d_lb,
                  cudaStream_t st);
int bounds_and_order(const float* d_q, int64_t Q, const lf_index& idx, double* d_qsumm, double* d_lb_scratch,
                     double* d_lbs, int* d_order, cudaStream_t st, int* kernels);
int sort_visit_order(const double* d_lb, int64_t Q, int n, double* d_lb_sorted, int* d_order,
                     cudaStream_t st);
}  // namespace lf
