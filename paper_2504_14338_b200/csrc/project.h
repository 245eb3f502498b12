// project.h — host interface of the projection / basis kernels (project.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace dopinf_b200 {
namespace project {

// Padded Φ_r column count (multiple of 16, or of 128 beyond 128).
int basis_cols_pad(int r);

// qhat (r x K) = tr(K x r)ᵀ d(K x K), reference FMA order.
cudaError_t launch_project(const double* tr, const double* d, int K, int r, double* qhat,
                           cudaStream_t stream);

// out (nsel x r) = q[rows] tr, reference (unfused) order.
cudaError_t launch_basis_rows(const double* q, size_t ld, int K, const double* tr, int r,
                              const long long* rows, int nsel, double* out, cudaStream_t stream);

// out (nsel x nt_p) = fma(s_row, dot(basis[k], qt[t]), means[row]) for the
// probe rows rows[k] (reconstruct_probes, reference dot order; scales null: s = 1).
cudaError_t launch_probe_series(const double* basis, int r, const double* qt, int nt_p, const long long* rows,
                                const double* means, const double* scales, long long nx_i, int nsel, double* out,
                                cudaStream_t stream);

// phi (rows x r_pad, pitch r_pad) = q (rows x K, pitch ld) · trtᵀ, with trt = T_rᵀ
// (r_pad x K, pitch ldt, rows >= r zero).
cudaError_t launch_basis(const double* q, size_t ld, long long rows, int K, const double* trt,
                         size_t ldt, int r_pad, double* phi, int num_sms, cudaStream_t stream);

}  // namespace project
}  // namespace dopinf_b200
