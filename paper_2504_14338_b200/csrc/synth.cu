// synth.cu — seeded synthetic snapshot generators for the BASELINE.json
// configs (plumbing for bench.py and the tests; not part of the snapshot
// pass). Every value is a pure function of (seed, variable, GLOBAL spatial
// index, snapshot index), so a row-sharded dataset is the same bytes however
// it is partitioned over ranks.
//
//   oscillator (configs 1, 2, 4):
//     Q[v,p,k] = amp_v Σ_{j=1..m} sin(jπ x_p + θ_vj) e^{−γ_vj t_k} cos(ω_vj t_k + φ_vj)
//                + noise · N(0,1),   t_k = k·dt,  x_p ~ U[0,1) per global point p,
//     θ, φ ~ U[0,2π), ω ~ U[1,50), γ ~ U[0,0.5) drawn per variable on the host.
//   lowrank (config 3):
//     Q[v,p,k] = N(0,1) + amp Σ_{j<m} U[p,j] V[j,k],  U ~ N(0,1)/√m, V ~ N(0,1).
#include <cmath>
#include <random>
#include <vector>

#include "common.cuh"
#include "synth.h"

namespace dopinf_b200 {
namespace synth {

namespace {

constexpr int kMaxModes = 128;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t key4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
    return mix64(mix64(mix64(seed ^ mix64(a)) ^ b) ^ c);
}

__device__ __forceinline__ double u01(uint64_t h) {  // [0, 1)
    return static_cast<double>(h >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double normal(uint64_t h) {  // Box-Muller on one hashed pair
    const double u1 = 1.0 - u01(h);
    const double u2 = u01(mix64(h ^ 0x5851F42D4C957F2DULL));
    return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// Column table B[v][j][k].
__global__ void osc_table_kernel(const double* __restrict__ modes, int n_vars, int m, int K,
                                 double dt, double* __restrict__ table) {
    const long long total = static_cast<long long>(n_vars) * m * K;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int k = static_cast<int>(e % K);
        const long long vj = e / K;
        const double* md = modes + vj * 4;  // theta, omega, gamma, phi
        const double t = k * dt;
        table[e] = exp(-md[2] * t) * cos(md[1] * t + md[3]);
    }
}

__global__ void lowrank_table_kernel(uint64_t seed, int m, int K, double* __restrict__ table) {
    const long long total = static_cast<long long>(m) * K;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        table[e] = normal(key4(seed, 0x5EED0002ULL, e / K, e % K));
    }
}

// Warp per group of kGroupRows rows of one variable: the rows' factors in
// shared memory, lanes stride over snapshots, and each column-table entry
// (L2-resident) is loaded once for the group's rows — a warp per single row
// re-read the table m times per element (≈ 24 TB of L2 traffic at config 4).
// Per element the arithmetic is unchanged: acc = fma(fac[j], tab[j][k], acc)
// over j ascending, then + noise·N(0,1).
constexpr int kGroupRows = 4;

template <bool kOsc>
__global__ void __launch_bounds__(256)
    fill_kernel(double* __restrict__ q, size_t ld, long long rows, int K, long long nx_i,
                long long row_begin, int m, const double* __restrict__ modes,
                const double* __restrict__ amps, const double* __restrict__ table, uint64_t seed,
                double noise, double amp, int var0) {
    __shared__ double fac[8][kGroupRows][kMaxModes];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const long long n_vars = (rows + nx_i - 1) / nx_i;
    const long long gpv = (nx_i + kGroupRows - 1) / kGroupRows;  // groups per variable
    const long long n_groups = n_vars * gpv;
    const long long nwarps = static_cast<long long>(gridDim.x) * 8;
    for (long long grp = static_cast<long long>(blockIdx.x) * 8 + warp; grp < n_groups; grp += nwarps) {
        const int v = static_cast<int>(grp / gpv);
        const long long l0 = (grp % gpv) * kGroupRows;                  // first local point of the group
        const int nr = nx_i - l0 < kGroupRows ? static_cast<int>(nx_i - l0) : kGroupRows;
        const int nv_tab = kOsc ? v : 0;
        for (int i = 0; i < nr; ++i) {
            const long long p = row_begin + l0 + i;  // global spatial index
            for (int j = lane; j < m; j += 32) {
                if (kOsc) {
                    const double x = u01(key4(seed, 0x5EED0001ULL, p, 0));
                    const double theta = modes[(static_cast<size_t>(v) * m + j) * 4 + 0];
                    fac[warp][i][j] = (amps ? amps[v] : 1.0) * sin((j + 1) * M_PI * x + theta);
                } else {
                    fac[warp][i][j] = amp * normal(key4(seed, 0x5EED0003ULL, p, j)) * rsqrt(static_cast<double>(m));
                }
            }
        }
        __syncwarp();
        const double* tab = table + static_cast<size_t>(nv_tab) * m * K;
        const long long row0 = static_cast<long long>(v) * nx_i + l0;
        for (int k = lane; k < K; k += 32) {
            double acc[kGroupRows];
#pragma unroll
            for (int i = 0; i < kGroupRows; ++i) acc[i] = 0.0;
            for (int j = 0; j < m; ++j) {
                const double t = tab[static_cast<size_t>(j) * K + k];
#pragma unroll
                for (int i = 0; i < kGroupRows; ++i) acc[i] = fma(fac[warp][i][j], t, acc[i]);
            }
#pragma unroll
            for (int i = 0; i < kGroupRows; ++i) {
                if (i < nr) {
                    const long long p = row_begin + l0 + i;
                    double a = acc[i];
                    if (noise != 0.0) a += noise * normal(key4(seed, 0x5EED0004ULL + var0 + v, p, k));
                    q[static_cast<size_t>(row0 + i) * ld + k] = a;
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace

cudaError_t oscillator(double* q, size_t ld, long long rows, int K, long long nx_i,
                       long long row_begin, int n_vars, uint64_t seed, int n_modes, double dt,
                       double noise, const double* amps_host, int num_sms, cudaStream_t stream, int var0) {
    if (n_modes < 1 || n_modes > kMaxModes) return cudaErrorInvalidValue;
    std::vector<double> modes(static_cast<size_t>(n_vars) * n_modes * 4);
    for (int v = 0; v < n_vars; ++v) {
        std::mt19937_64 gen(seed * 1000003ULL + static_cast<uint64_t>(var0 + v));
        auto uni = [&](double lo, double hi) {
            return lo + (hi - lo) * (static_cast<double>(gen() >> 11) * 0x1.0p-53);
        };
        for (int j = 0; j < n_modes; ++j) {
            double* md = &modes[(static_cast<size_t>(v) * n_modes + j) * 4];
            md[0] = uni(0.0, 2.0 * M_PI);  // theta
            md[1] = uni(1.0, 50.0);        // omega
            md[2] = uni(0.0, 0.5);         // gamma
            md[3] = uni(0.0, 2.0 * M_PI);  // phi
        }
    }
    double *d_modes = nullptr, *d_table = nullptr, *d_amps = nullptr;
    const size_t table_n = static_cast<size_t>(n_vars) * n_modes * K;
    cudaError_t e = cudaMallocAsync(&d_modes, modes.size() * sizeof(double), stream);
    if (e == cudaSuccess) e = cudaMallocAsync(&d_table, table_n * sizeof(double), stream);
    if (e == cudaSuccess && amps_host) e = cudaMallocAsync(&d_amps, n_vars * sizeof(double), stream);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(d_modes, modes.data(), modes.size() * sizeof(double),
                            cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess && amps_host)
        e = cudaMemcpyAsync(d_amps, amps_host, n_vars * sizeof(double), cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) {
        osc_table_kernel<<<num_sms * 4, 256, 0, stream>>>(d_modes, n_vars, n_modes, K, dt, d_table);
        note_launch();
        fill_kernel<true><<<num_sms * 8, 256, 0, stream>>>(q, ld, rows, K, nx_i, row_begin, n_modes,
                                                          d_modes, d_amps, d_table, seed, noise, 1.0, var0);
        note_launch();
        e = cudaGetLastError();
        // Host vectors must outlive the async copies.
        if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    }
    cudaFreeAsync(d_modes, stream);
    cudaFreeAsync(d_table, stream);
    if (d_amps) cudaFreeAsync(d_amps, stream);
    return e;
}

cudaError_t lowrank(double* q, size_t ld, long long rows, int K, long long nx_i,
                    long long row_begin, uint64_t seed, int rank, double amplitude, int num_sms,
                    cudaStream_t stream) {
    if (rank < 1 || rank > kMaxModes) return cudaErrorInvalidValue;
    double* d_table = nullptr;
    cudaError_t e = cudaMallocAsync(&d_table, static_cast<size_t>(rank) * K * sizeof(double), stream);
    if (e == cudaSuccess) {
        lowrank_table_kernel<<<num_sms * 4, 256, 0, stream>>>(seed, rank, K, d_table);
        note_launch();
        fill_kernel<false><<<num_sms * 8, 256, 0, stream>>>(q, ld, rows, K, nx_i, row_begin, rank,
                                                           nullptr, nullptr, d_table, seed, 1.0,
                                                           amplitude, 0);
        note_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(d_table, stream);
    return e;
}

}  // namespace synth
}  // namespace dopinf_b200
