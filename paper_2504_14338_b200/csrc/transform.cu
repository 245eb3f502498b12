// transform.cu — Step II snapshot transform (reference proj/src/transform.cpp).
//
// Two HBM passes instead of the reference's five (center: read + write,
// max-abs: read, scale: read + write):
//   stats pass  (read 8·n·K B): per row the temporal mean, computed in EXACTLY
//               the reference's floating-point order — the AVX2 sum of
//               kernels_avx2.cpp:48-55 (4 lane accumulators over i ≡ j mod 4,
//               hsum (l0+l2)+(l1+l3), sequential scalar tail), then / K — and
//               the row's max |x − mean|, which equals max(|fl(max−mean)|,
//               |fl(min−mean)|) because rounding is monotone. Row maxima are
//               max-reduced per variable (order independent → exact).
//   apply pass  (read + write 16·n·K B): x ← (x − mean) / s with IEEE
//               division, i.e. fl(fl(x + (−mean)) / s) as transform.cpp:16
//               then :47 compute it. Centering alone is s = 1 (no division).
// So the transformed block, the means and the scales are bit-identical to
// the reference's on the same input bytes.
#include <algorithm>

#include "common.cuh"
#include "transform.h"

namespace dopinf_b200 {
namespace transform {

namespace {

constexpr int kStatsWarps = 8;           // warps per block
constexpr int kRowsPerWarp = 8;          // one 4-lane group per row
constexpr int kColsPerIter = 64;         // 8 rows × 64 columns = 4 KiB per warp per chunk
constexpr int kPad = kColsPerIter + 4;   // row pitch in smem: 68 doubles (conflict-free reads)
constexpr int kLoads = kRowsPerWarp * kColsPerIter / 64;  // 16-byte loads per lane per chunk
constexpr int kMaxSmemVars = 64;

// Lane's share of one chunk: rows r0 + 2(u/2) + lane/16, columns c0 + 32(u%2) + 2(lane%16).
__device__ __forceinline__ void load_chunk(double2 (&v)[kLoads], const double* __restrict__ q, size_t ld,
                                           long long rows, int K, long long r0, int c0, int lane) {
#pragma unroll
    for (int u = 0; u < kLoads; ++u) {
        const long long lr = r0 + (u >> 1) * 2 + (lane >> 4);
        const int col = c0 + (u & 1) * 32 + (lane & 15) * 2;
        v[u] = make_double2(0.0, 0.0);
        if (lr < rows) {
            const double* src = q + static_cast<size_t>(lr) * ld + col;
            if (col + 1 < K) {
                v[u] = __ldcs(reinterpret_cast<const double2*>(src));
            } else if (col < K) {
                v[u].x = __ldcs(src);
            }
        }
    }
}

__global__ void __launch_bounds__(kStatsWarps * 32)
    stats_kernel(const double* __restrict__ q, size_t ld, long long rows, int K, long long nx_i,
                 int n_vars, int center, double* __restrict__ means, double* __restrict__ var_max) {
    __shared__ __align__(16) double buf[kStatsWarps][kRowsPerWarp][kPad];
    __shared__ double smax[kMaxSmemVars];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int g = lane >> 2, j = lane & 3;
    const bool smem_vars = n_vars <= kMaxSmemVars;
    for (int v = threadIdx.x; v < kMaxSmemVars; v += blockDim.x) smax[v] = 0.0;
    __syncthreads();

    const int K4 = K - (K & 3);
    const long long n_groups = (rows + kRowsPerWarp - 1) / kRowsPerWarp;
    const long long warp_stride = static_cast<long long>(gridDim.x) * kStatsWarps;
    double(*wb)[kPad] = buf[warp];

    for (long long grp = static_cast<long long>(blockIdx.x) * kStatsWarps + warp; grp < n_groups;
         grp += warp_stride) {
        const long long r0 = grp * kRowsPerWarp;
        const long long row = r0 + g;
        const bool row_ok = row < rows;
        double lacc = 0.0;
        double mx = -__longlong_as_double(0x7ff0000000000000LL);
        double mn = __longlong_as_double(0x7ff0000000000000LL);
        double2 v[kLoads];
        load_chunk(v, q, ld, rows, K, r0, 0, lane);
        for (int c0 = 0; c0 < K; c0 += kColsPerIter) {
            // Coalesced chunk (half-warp per 256 B row segment) → padded smem, then
            // prefetch the next chunk into registers while this one is reduced.
#pragma unroll
            for (int u = 0; u < kLoads; ++u) {
                *reinterpret_cast<double2*>(&wb[(u >> 1) * 2 + (lane >> 4)][(u & 1) * 32 + (lane & 15) * 2]) = v[u];
            }
            __syncwarp();
            if (c0 + kColsPerIter < K) load_chunk(v, q, ld, rows, K, r0, c0 + kColsPerIter, lane);
            if (row_ok) {
#pragma unroll
                for (int s = 0; s < kColsPerIter / 4; ++s) {
                    const int col = c0 + 4 * s + j;
                    if (col < K) {
                        const double x = wb[g][4 * s + j];
                        if (col < K4) lacc += x;  // lane j of the AVX2 accumulator, in order
                        mx = fmax(mx, x);
                        mn = fmin(mn, x);
                    }
                }
            }
            __syncwarp();
        }
        // hsum of the 4 lanes: (l0 + l2) + (l1 + l3)  (kernels_avx2.cpp:16-22)
        const double l1 = __shfl_down_sync(0xffffffffu, lacc, 1, 4);
        const double l2 = __shfl_down_sync(0xffffffffu, lacc, 2, 4);
        const double l3 = __shfl_down_sync(0xffffffffu, lacc, 3, 4);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, 1));
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, 2));
        if (j == 0 && row_ok) {
            double mean = 0.0;
            if (center) {
                double sum = (lacc + l2) + (l1 + l3);
                const double* tail = q + static_cast<size_t>(row) * ld;
                for (int c = K4; c < K; ++c) sum += tail[c];  // scalar tail, in order
                mean = sum / static_cast<double>(K);
                means[row] = mean;
            }
            const double m = fmax(fabs(mx - mean), fabs(mn - mean));
            const int var = static_cast<int>(row / nx_i);
            if (smem_vars) {
                atomic_max_nonneg(&smax[var], m);
            } else {
                atomic_max_nonneg(&var_max[var], m);
            }
        }
    }
    __syncthreads();
    if (smem_vars) {
        for (int v = threadIdx.x; v < n_vars; v += blockDim.x) {
            if (smax[v] > 0.0) atomic_max_nonneg(&var_max[v], smax[v]);
        }
    }
}

// x ← (x − mean[row]) / scale[var]  (or x − mean when scales == nullptr);
// a zero scale divides like the reference's div_scalar (±inf / NaN), unless
// skip_zero (the streamed pass: a degenerate variable stays centered, as the
// reference leaves it when compute_global_scales throws before scaling).
// Warp per row; each lane issues kApplyBatch (8) independent 16-byte loads before
// any store (streaming hints: the block is touched once per pass).
constexpr int kApplyBatch = 8;

template <bool kScale>
__global__ void __launch_bounds__(256)
    apply_kernel(double* __restrict__ q, size_t ld, long long rows, int K, long long nx_i,
                 const double* __restrict__ means, const double* __restrict__ scales, int skip_zero) {
    const int lane = threadIdx.x % 32;
    const long long warp0 = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const long long nwarps = static_cast<long long>(gridDim.x) * blockDim.x / 32;
    const int pairs = K / 2;
    for (long long row = warp0; row < rows; row += nwarps) {
        const double neg = means ? -means[row] : -0.0;
        const double s = kScale ? scales[row / nx_i] : 1.0;
        if (kScale && skip_zero && s == 0.0) continue;
        double2* p = reinterpret_cast<double2*>(q + static_cast<size_t>(row) * ld);
        for (int c = lane; c < pairs; c += 32 * kApplyBatch) {
            double2 v[kApplyBatch];
#pragma unroll
            for (int u = 0; u < kApplyBatch; ++u) {
                if (c + 32 * u < pairs) v[u] = __ldcs(p + c + 32 * u);
            }
#pragma unroll
            for (int u = 0; u < kApplyBatch; ++u) {
                if (c + 32 * u < pairs) {
                    double2 w;
                    w.x = kScale ? (v[u].x + neg) / s : v[u].x + neg;
                    w.y = kScale ? (v[u].y + neg) / s : v[u].y + neg;
                    __stcs(p + c + 32 * u, w);
                }
            }
        }
        if ((K & 1) && lane == 0) {
            double* last = q + static_cast<size_t>(row) * ld + (K - 1);
            *last = kScale ? (*last + neg) / s : *last + neg;
        }
    }
}

}  // namespace

cudaError_t launch_stats(const double* q, size_t ld, long long rows, int K, long long nx_i,
                         int n_vars, bool center, double* means, double* var_max, int num_sms,
                         cudaStream_t stream) {
    const long long groups = (rows + kRowsPerWarp - 1) / kRowsPerWarp;
    const long long want = (groups + kStatsWarps - 1) / kStatsWarps;
    const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(want, num_sms * 8LL)));
    stats_kernel<<<grid, kStatsWarps * 32, 0, stream>>>(q, ld, rows, K, nx_i, n_vars, center ? 1 : 0,
                                                        means, var_max);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_apply(double* q, size_t ld, long long rows, int K, long long nx_i,
                         const double* means, const double* scales, int num_sms,
                         cudaStream_t stream, bool skip_zero_scale) {
    const long long want = (rows + 7) / 8;
    const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>(want, num_sms * 16LL)));
    if (scales) {
        apply_kernel<true><<<grid, 256, 0, stream>>>(q, ld, rows, K, nx_i, means, scales, skip_zero_scale ? 1 : 0);
    } else {
        apply_kernel<false><<<grid, 256, 0, stream>>>(q, ld, rows, K, nx_i, means, scales, 0);
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace transform
}  // namespace dopinf_b200
