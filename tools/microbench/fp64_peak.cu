// FP64 throughput probe for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64) vs
// DFMA vs both pipes at once. Sets the denominator for the Gram roofline.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); std::exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int ACC>
__global__ void k_dmma(double* out, int iters, double seed) {
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  double a = seed * (threadIdx.x + 1), b = seed * 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int ACC>
__global__ void k_dfma(double* out, int iters, double seed) {
  double c[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i] = seed * i;
  const double a = 1.0000001, b = seed * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

// Even warps DMMA, odd warps DFMA (iters_f scaled so both finish together).
template <int ACC>
__global__ void k_mixed(double* out, int iters, int iters_f, double seed) {
  const int warp = threadIdx.x / 32;
  double s = 0.0;
  if (warp % 2 == 0) {
    double c[ACC][2];
#pragma unroll
    for (int i = 0; i < ACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
    double a = seed * (threadIdx.x + 1), b = seed * 0.5;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < ACC; ++i) dmma(c[i][0], c[i][1], a, b);
    }
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  } else {
    double c[ACC];
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = seed * i;
    const double a = 1.0000001, b = seed * 1e-9;
    for (int it = 0; it < iters_f; ++it) {
#pragma unroll
      for (int i = 0; i < ACC; ++i) c[i] = fma(c[i], a, b);
    }
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i];
  }
  if (s == 12345.678) out[0] = s;
}

template <class F>
float time_it(F launch) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch(); launch();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 8));
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int ctas_per_sm : {1, 2}) {
      const int grid = sms * ctas_per_sm, block = warps * 32;
      const double n_mma = double(grid) * warps * iters * 8;
      float ms = time_it([&] { k_dmma<8><<<grid, block>>>(out, iters, 1.0); });
      std::printf("DMMA  warps/cta=%2d ctas/sm=%d  %.3f ms  %.2f TFLOP/s\n", warps, ctas_per_sm,
                  ms, n_mma * 512 / (ms * 1e-3) / 1e12);
      const double n_fma = double(grid) * block * iters * 8;
      ms = time_it([&] { k_dfma<8><<<grid, block>>>(out, iters, 1.0); });
      std::printf("DFMA  warps/cta=%2d ctas/sm=%d  %.3f ms  %.2f TFLOP/s\n", warps, ctas_per_sm,
                  ms, n_fma * 2 / (ms * 1e-3) / 1e12);
    }
  }
  for (int ratio : {1, 2, 4, 8}) {
    const int grid = sms, warps = 16, block = warps * 32;
    const int iters_f = iters * ratio;
    const double flops = double(grid) * (warps / 2) * iters * 8 * 512 +
                         double(grid) * (warps / 2) * 32 * iters_f * 8 * 2;
    float ms = time_it([&] { k_mixed<8><<<grid, block>>>(out, iters, iters_f, 1.0); });
    std::printf("MIXED dfma_iter_ratio=%d  %.3f ms  %.2f TFLOP/s combined\n", ratio, ms,
                flops / (ms * 1e-3) / 1e12);
  }
  CK(cudaFree(out));
  return 0;
}
