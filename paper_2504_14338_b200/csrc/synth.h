// synth.h — seeded device generators for the BASELINE.json configs (synth.cu).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace dopinf_b200 {
namespace synth {

// var0: global index of the first variable generated (mode draws and noise
// streams are keyed by the global variable index).
cudaError_t oscillator(double* q, size_t ld, long long rows, int K, long long nx_i,
                       long long row_begin, int n_vars, uint64_t seed, int n_modes, double dt,
                       double noise, const double* amps_host, int num_sms, cudaStream_t stream,
                       int var0 = 0);

cudaError_t lowrank(double* q, size_t ld, long long rows, int K, long long nx_i,
                    long long row_begin, uint64_t seed, int rank, double amplitude, int num_sms,
                    cudaStream_t stream);

}  // namespace synth
}  // namespace dopinf_b200
