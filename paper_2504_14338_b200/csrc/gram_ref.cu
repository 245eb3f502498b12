// gram_ref.cu — the Gram in the reference's own summation order (the
// reference-order mode, dopinf_b200_set_gram_order).
//
// linalg::gram (linalg.cpp:50-58) loops rows outer and adds q(l, i)·q.row(l)
// to c.row(i) with axpy (kernels_avx2.cpp:69-78: one FMA per element), so
// entry (i, j) is the FMA chain c = fma(q(l, i), q(l, j), c) over the rows l in
// ascending order. This kernel evaluates exactly that chain for every upper-
// triangle entry — no split over rows, one thread per 8×8 entries walking all
// rows in order — so the result is the reference's D bit for bit (and, with
// the ORDERED cross-rank sum, the in-process reference's at any rank count).
// It runs on the DFMA side of the FP64 pipe: same peak as DMMA on B200, but
// bounded by how many 128×128 tiles the triangle has (K=600: 15 CTAs), so the
// tensor-pipe kernel (gram.cu) stays the default.
//
// CTA: 256 threads = 16×16, tile 128×128 entries; thread (ti, tj) owns rows
// i = i0 + 8·ti + x (x < 8, contiguous: 128-bit broadcast loads) and columns
// j = j0 + tj + 16·y (y < 8, strided: each 64-bit load is 16 consecutive
// doubles per half-warp, conflict free). Rows stream through a double-
// buffered shared-memory stage of 16 rows × (128 + 128) columns via cp.async
// (zero-filled beyond the block).
#include "common.cuh"
#include "gram.h"

namespace dopinf_b200 {
namespace gram {

namespace {

constexpr int kRefEdge = 128;
constexpr int kRefThreads = 256;
constexpr int kRefRows = 16;
constexpr int kRefChunks = kRefEdge / 2;                                           // 16-byte chunks per tile row
constexpr size_t kRefSmemBytes = size_t(2) * 2 * kRefRows * kRefEdge * sizeof(double);  // 64 KiB

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}

__global__ void __launch_bounds__(kRefThreads, 1)
    gram_ref_kernel(const double* __restrict__ q, size_t ld, long long rows, int K, int nb,
                    double* __restrict__ packed, int accumulate) {
    extern __shared__ __align__(16) double smem[];  // [buf][side][kRefRows][kRefEdge]
    int t = blockIdx.x, bi = 0;
    while (t >= nb - bi) {
        t -= nb - bi;
        ++bi;
    }
    const int bj = bi + t;
    const int i0 = bi * kRefEdge, j0 = bj * kRefEdge;
    const int tid = threadIdx.x, ti = tid / 16, tj = tid % 16;
    const size_t Kz = static_cast<size_t>(K);

    auto packed_at = [&](int i, int j) { return static_cast<size_t>(i) * (2 * Kz - i + 1) / 2 + (j - i); };
    double acc[8][8];
#pragma unroll
    for (int x = 0; x < 8; ++x) {
#pragma unroll
        for (int y = 0; y < 8; ++y) {
            const int i = i0 + 8 * ti + x, j = j0 + tj + 16 * y;
            acc[x][y] = (accumulate && i < K && j < K && j >= i) ? packed[packed_at(i, j)] : 0.0;
        }
    }

    const uint32_t sbase = smem_u32(smem);
    auto load_stage = [&](long long s, int buf) {
        const long long r0 = s * kRefRows;
        for (int c = tid; c < 2 * kRefRows * kRefChunks; c += kRefThreads) {
            const int side = c / (kRefRows * kRefChunks);
            const int rem = c % (kRefRows * kRefChunks);
            const int rr = rem / kRefChunks, cc = rem % kRefChunks;
            const int col = (side ? j0 : i0) + 2 * cc;
            const long long row = r0 + rr;
            const bool ok = row < rows && col < K;
            const double* src = ok ? q + static_cast<size_t>(row) * ld + col : q;
            const uint32_t dst =
                sbase + static_cast<uint32_t>((((buf * 2 + side) * kRefRows + rr) * kRefEdge + 2 * cc) * sizeof(double));
            cp16(dst, src, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    const long long stages = (rows + kRefRows - 1) / kRefRows;
    if (stages > 0) load_stage(0, 0);
    for (long long s = 0; s < stages; ++s) {
        const int buf = static_cast<int>(s & 1);
        if (s + 1 < stages) {
            load_stage(s + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const double* sI = smem + static_cast<size_t>(buf * 2 + 0) * kRefRows * kRefEdge + 8 * ti;
        const double* sJ = smem + static_cast<size_t>(buf * 2 + 1) * kRefRows * kRefEdge + tj;
        const long long left = rows - s * kRefRows;
        const int nr = left < kRefRows ? static_cast<int>(left) : kRefRows;
#pragma unroll 2
        for (int r = 0; r < nr; ++r) {
            double a[8], b[8];
#pragma unroll
            for (int x = 0; x < 8; x += 2) {
                const double2 v = lds128(sI + r * kRefEdge + x);
                a[x] = v.x;
                a[x + 1] = v.y;
            }
#pragma unroll
            for (int y = 0; y < 8; ++y) b[y] = sJ[r * kRefEdge + 16 * y];
#pragma unroll
            for (int x = 0; x < 8; ++x) {
#pragma unroll
                for (int y = 0; y < 8; ++y) acc[x][y] = __fma_rn(a[x], b[y], acc[x][y]);
            }
        }
        __syncthreads();  // the buffer is refilled two stages on
    }

#pragma unroll
    for (int x = 0; x < 8; ++x) {
#pragma unroll
        for (int y = 0; y < 8; ++y) {
            const int i = i0 + 8 * ti + x, j = j0 + tj + 16 * y;
            if (i < K && j < K && j >= i) packed[packed_at(i, j)] = acc[x][y];
        }
    }
}

}  // namespace

cudaError_t launch_gram_reference_order(const double* q, size_t ld, long long rows, int K, double* packed,
                                        bool accumulate, cudaStream_t stream) {
    if (K < 1 || (ld % 2) != 0 || (reinterpret_cast<uintptr_t>(q) % 16) != 0) return cudaErrorInvalidValue;
    const int nb = (K + kRefEdge - 1) / kRefEdge;
    const int tiles = nb * (nb + 1) / 2;
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(gram_ref_kernel), static_cast<int>(kRefSmemBytes));
    if (e != cudaSuccess) return e;
    gram_ref_kernel<<<tiles, kRefThreads, kRefSmemBytes, stream>>>(q, ld, rows, K, nb, packed, accumulate ? 1 : 0);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gram
}  // namespace dopinf_b200
