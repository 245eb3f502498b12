// transform.h — host interface of the Step II transform kernels (transform.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace dopinf_b200 {
namespace transform {

// Per-row mean (when center) and per-variable max |x - mean| (MAX-combined
// into var_max, which the caller zeroes first).
cudaError_t launch_stats(const double* q, size_t ld, long long rows, int K, long long nx_i,
                         int n_vars, bool center, double* means, double* var_max, int num_sms,
                         cudaStream_t stream);

// q <- (q - means[row]) / scales[row / nx_i]; means/scales may be null;
// skip_zero_scale leaves rows of a zero-scale variable untouched.
cudaError_t launch_apply(double* q, size_t ld, long long rows, int K, long long nx_i,
                         const double* means, const double* scales, int num_sms,
                         cudaStream_t stream, bool skip_zero_scale = false);

}  // namespace transform
}  // namespace dopinf_b200
