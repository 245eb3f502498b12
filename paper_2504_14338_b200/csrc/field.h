// field.h — host interface of the field reconstruction kernel (field.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace dopinf_b200 {
namespace field {

// Largest contraction extent one launch takes (Φ tile resident in smem).
int max_r_pad();

// out (rows × nt_p, pitch ldo) = fma(s_row, phi · qtᵀ, mean_row) over the
// first k_ext columns (a multiple of 4, ≤ max_r_pad()) of phi (rows, pitch
// ldphi) and qt (nt_p rows, pitch ldq), both zero beyond r;
// s_row = scales[(row_base + row) / nx_i] (1 when scales is null), mean_row = means[row]
// (0 when null). accumulate != 0 adds the values already in `out` to the
// product before the epilogue (k-slabs of r > max_r_pad()).
cudaError_t launch_field(const double* phi, size_t ldphi, const double* qt, size_t ldq, long long rows, int nt_p,
                         int k_ext, const double* means, const double* scales, long long nx_i, long long row_base,
                         double* out, size_t ldo, int accumulate, int num_sms, cudaStream_t stream);

}  // namespace field
}  // namespace dopinf_b200
