// rom.h — host interface of the OpInf grid-search kernels (rom.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace dopinf_b200 {
namespace rom {

// Per-pair score record: finite (0/1), train_err, growth, first zero-norm
// reference row (−1: none), constant-training-data flag (0/1).
constexpr int kScoreFields = 5;

// Dhat (nt−1 × d, pitch ldd ≥ d) and Qhat2ᵀ (nt−1 × r) from the r × nt Q̂.
cudaError_t launch_assemble(const double* qhat, int r, int nt, double* dhat, size_t ldd, double* q2t,
                            cudaStream_t stream);
// G (d × d) = DhatᵀDhat in the reference's FMA order (bit-identical).
cudaError_t launch_gram_exact(const double* dhat, size_t ldd, int K, int d, double* g, cudaStream_t stream);
// rhs (d × r, column-major) = Dhatᵀ Qhat2ᵀ, reference FMA order.
cudaError_t launch_rhs(const double* dhat, size_t ldd, const double* q2t, int K, int d, int r, double* rhs_cm,
                       cudaStream_t stream);
// lhs_p = G + diag(γ(β1[p], β2[p])) (d × d) and rhs_p = rhs for p < n_pairs.
cudaError_t launch_systems(const double* g, int d, int r, const double* beta1, const double* beta2, int n_pairs,
                           const double* rhs_cm, double* lhs, double* rhs_batch, cudaStream_t stream);
// b_p ← L_p⁻ᵀ L_p⁻¹ b_p for batch Cholesky factors (column-major lower d × d)
// and r right-hand sides each (column-major d × r); d ≤ 1760.
cudaError_t launch_chol_solve(const double* l, int d, int batch, double* b, int r, cudaStream_t stream);
// n_pairs ROMs (operators column-major d × r each) from q0 for n_steps rows.
cudaError_t launch_integrate(const double* ops, int r, const double* q0, int n_steps, int n_pairs, double* traj,
                             cudaStream_t stream);
// Scores (kScoreFields per pair) against the training rows qrows (nt × r).
cudaError_t launch_score(const double* traj, int n_steps, int r, const double* qrows, int nt, int n_pairs,
                         double* out, cudaStream_t stream);
// t (cols × rows) = aᵀ for a rows × cols.
cudaError_t launch_transpose(const double* a, int rows, int cols, double* t, cudaStream_t stream);

}  // namespace rom
}  // namespace dopinf_b200
