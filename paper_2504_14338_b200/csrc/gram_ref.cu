// gram_ref.cu — the Gram in the reference's own summation order (the
// reference-order mode, dopinf_b200_set_gram_order).
//
// linalg::gram (linalg.cpp:50-58) loops rows outer and adds q(l, i)·q.row(l)
// to c.row(i) with axpy (kernels_avx2.cpp:69-78: one FMA per element), so
// entry (i, j) is the FMA chain c = fma(q(l, i), q(l, j), c) over the rows l in
// ascending order. This kernel evaluates exactly that chain for every upper-
// triangle entry — no split over rows, each thread walking all rows in order
// for its own entries — so the result is the reference's D bit for bit
// (and, with the ORDERED cross-rank sum, the in-process reference's at any
// rank count). It runs on the DFMA side of the FP64 pipe (peak 36.5 TFLOP/s,
// `profiles/r01_fp64_peak.txt`).
//
// Without a split over rows the parallelism is the number of entries, and
// smaller tiles cost more operand traffic per FMA, so the tile size follows K:
//  * small tiles (fewer than two waves of large tiles, e.g. K = 1200): CTA =
//    32 × 64 entries, the upper or lower half of a 64 × 64 tile of the upper
//    triangle (K = 1200: 380 CTAs); 8, 4 or 2 warps with 8, 16 or 32
//    independent FMA chains per thread (2 × 4, 4 × 4 or 8 × 4 entries) as the
//    CTA count grows; C2: 0.135 s;
//  * large tiles (K = 4096: 528 tiles): CTA = 8 warps = 128 × 128 entries, 8 × 8
//    per thread, 0.375× the operand bytes per FMA (the small tiles would make
//    the kernel L2-bandwidth bound there); C3 K = 4096: 3.4 s.
// Small tiles: warp w covers rows i0 + 2·TI·w .. of D: thread (ti = lane / 16,
// tj = lane % 16) owns i = i0 + 2·TI·w + TI·ti + x (x < TI, contiguous: 128-bit
// loads, broadcast across the half-warp) and j = j0 + tj + 16·y (y < 4,
// strided: each 64-bit load is 16 consecutive doubles per half-warp, conflict
// free). Large tiles: the
// same pattern with 8 × 8 entries per thread over a 16 × 16 thread grid. Rows
// stream through a double-buffered cp.async stage (zero-filled beyond the
// block).
#include "common.cuh"
#include "gram.h"

namespace dopinf_b200 {
namespace gram {

namespace {

constexpr int kRefEdge = 64;                // square tiles of the triangle
constexpr int kRefHalf = kRefEdge / 2;      // rows of D per CTA (half a tile)
// threads of a small-tile CTA: 2 warps with 8 × 4 entries per thread, 4 warps with 4 × 4
template <int TI>
__host__ __device__ constexpr int ref_threads() { return 32 * kRefHalf / (2 * TI); }
constexpr int kRefRows = 32;                // rows of Q per stage
constexpr int kRefCols = kRefHalf + kRefEdge;  // I columns then J columns of a stage row
constexpr size_t kRefSmemBytes = size_t(2) * kRefRows * kRefCols * sizeof(double);  // 48 KiB

__device__ __forceinline__ void cp16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}

template <int kRefTI>
__global__ void __launch_bounds__(ref_threads<kRefTI>())
    gram_ref_kernel(const double* __restrict__ q, size_t ld, long long rows, int K, int nb,
                    double* __restrict__ packed, int accumulate) {
    extern __shared__ __align__(16) double smem[];  // [buf][kRefRows][kRefCols]: I | J
    int t = blockIdx.x / 2, bi = 0;
    const int half = blockIdx.x % 2;
    while (t >= nb - bi) {
        t -= nb - bi;
        ++bi;
    }
    const int bj = bi + t;
    const int i0 = bi * kRefEdge + half * kRefHalf, j0 = bj * kRefEdge;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int ti = lane / 16, tj = lane % 16;
    const int ib = 2 * kRefTI * warp + kRefTI * ti;  // first of this thread's kRefTI rows of D in the tile
    const size_t Kz = static_cast<size_t>(K);

    auto packed_at = [&](int i, int j) { return static_cast<size_t>(i) * (2 * Kz - i + 1) / 2 + (j - i); };
    double acc[kRefTI][4];
#pragma unroll
    for (int x = 0; x < kRefTI; ++x) {
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int i = i0 + ib + x, j = j0 + tj + 16 * y;
            acc[x][y] = (accumulate && i < K && j < K && j >= i) ? packed[packed_at(i, j)] : 0.0;
        }
    }

    const uint32_t sbase = smem_u32(smem);
    auto load_stage = [&](long long s, int buf) {
        const long long r0 = s * kRefRows;
#pragma unroll 4
        for (int c = threadIdx.x; c < kRefRows * (kRefCols / 2); c += ref_threads<kRefTI>()) {
            const int rr = c / (kRefCols / 2), cc = 2 * (c % (kRefCols / 2));  // stage column
            const int col = cc < kRefHalf ? i0 + cc : j0 + (cc - kRefHalf);
            const long long row = r0 + rr;
            const bool ok = row < rows && col < K;
            const double* src = ok ? q + static_cast<size_t>(row) * ld + col : q;
            const uint32_t dst =
                sbase + static_cast<uint32_t>(((buf * kRefRows + rr) * kRefCols + cc) * sizeof(double));
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
        const double* sI = smem + static_cast<size_t>(buf) * kRefRows * kRefCols + ib;
        const double* sJ = smem + static_cast<size_t>(buf) * kRefRows * kRefCols + kRefHalf + tj;
        const long long left = rows - s * kRefRows;
        const int nr = left < kRefRows ? static_cast<int>(left) : kRefRows;
#pragma unroll 2
        for (int r = 0; r < nr; ++r) {
            double a[kRefTI], b[4];
#pragma unroll
            for (int x = 0; x < kRefTI; x += 2) {
                const double2 v = lds128(sI + r * kRefCols + x);
                a[x] = v.x;
                a[x + 1] = v.y;
            }
#pragma unroll
            for (int y = 0; y < 4; ++y) b[y] = sJ[r * kRefCols + 16 * y];
#pragma unroll
            for (int x = 0; x < kRefTI; ++x) {
#pragma unroll
                for (int y = 0; y < 4; ++y) acc[x][y] = __fma_rn(a[x], b[y], acc[x][y]);
            }
        }
        __syncthreads();  // the buffer is refilled two stages on
    }

#pragma unroll
    for (int x = 0; x < kRefTI; ++x) {
#pragma unroll
        for (int y = 0; y < 4; ++y) {
            const int i = i0 + ib + x, j = j0 + tj + 16 * y;
            if (i < K && j < K && j >= i) packed[packed_at(i, j)] = acc[x][y];
        }
    }
}

// ---- large tiles (128 × 128 entries, 8 × 8 per thread) ----
constexpr int kBigEdge = 128;
constexpr int kBigThreads = 256;
constexpr int kBigRows = 16;
constexpr int kBigChunks = kBigEdge / 2;                                           // 16-byte chunks per tile row
constexpr size_t kBigSmemBytes = size_t(2) * 2 * kBigRows * kBigEdge * sizeof(double);  // 64 KiB

__global__ void __launch_bounds__(kBigThreads, 1)
    gram_ref_big_kernel(const double* __restrict__ q, size_t ld, long long rows, int K, int nb,
                    double* __restrict__ packed, int accumulate) {
    extern __shared__ __align__(16) double smem[];  // [buf][side][kBigRows][kBigEdge]
    int t = blockIdx.x, bi = 0;
    while (t >= nb - bi) {
        t -= nb - bi;
        ++bi;
    }
    const int bj = bi + t;
    const int i0 = bi * kBigEdge, j0 = bj * kBigEdge;
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
        const long long r0 = s * kBigRows;
        for (int c = tid; c < 2 * kBigRows * kBigChunks; c += kBigThreads) {
            const int side = c / (kBigRows * kBigChunks);
            const int rem = c % (kBigRows * kBigChunks);
            const int rr = rem / kBigChunks, cc = rem % kBigChunks;
            const int col = (side ? j0 : i0) + 2 * cc;
            const long long row = r0 + rr;
            const bool ok = row < rows && col < K;
            const double* src = ok ? q + static_cast<size_t>(row) * ld + col : q;
            const uint32_t dst =
                sbase + static_cast<uint32_t>((((buf * 2 + side) * kBigRows + rr) * kBigEdge + 2 * cc) * sizeof(double));
            cp16(dst, src, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    const long long stages = (rows + kBigRows - 1) / kBigRows;
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
        const double* sI = smem + static_cast<size_t>(buf * 2 + 0) * kBigRows * kBigEdge + 8 * ti;
        const double* sJ = smem + static_cast<size_t>(buf * 2 + 1) * kBigRows * kBigEdge + tj;
        const long long left = rows - s * kBigRows;
        const int nr = left < kBigRows ? static_cast<int>(left) : kBigRows;
#pragma unroll 2
        for (int r = 0; r < nr; ++r) {
            double a[8], b[8];
#pragma unroll
            for (int x = 0; x < 8; x += 2) {
                const double2 v = lds128(sI + r * kBigEdge + x);
                a[x] = v.x;
                a[x + 1] = v.y;
            }
#pragma unroll
            for (int y = 0; y < 8; ++y) b[y] = sJ[r * kBigEdge + 16 * y];
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
    const int nb_big = (K + kBigEdge - 1) / kBigEdge;
    const int tiles_big = nb_big * (nb_big + 1) / 2;
    cudaError_t e;
    if (tiles_big >= 2 * 148) {  // enough large tiles for ~2 waves: the cheaper operand traffic wins
        e = set_smem_attr_once(reinterpret_cast<const void*>(gram_ref_big_kernel), static_cast<int>(kBigSmemBytes));
        if (e != cudaSuccess) return e;
        gram_ref_big_kernel<<<tiles_big, kBigThreads, kBigSmemBytes, stream>>>(q, ld, rows, K, nb_big, packed,
                                                                                accumulate ? 1 : 0);
    } else {
        const int nb = (K + kRefEdge - 1) / kRefEdge;
        const int tiles = nb * (nb + 1) / 2;
        // Every thread walks all rows, so the time is rows × the per-row step of
        // its chains, and more warps hide that step better while the CTAs are
        // few; with many CTAs the larger thread tiles' lower operand traffic
        // wins (tools/refgram_probe.py, profiles/r02_refgram_ti_ab.txt):
        //   < 1 CTA per SM:  2 × 4 entries per thread, 8 warps (K = 256: 78 → 69 ms, config 1: 2.5 → 2.2 ms)
        //   < 4 CTAs per SM: 4 × 4, 4 warps (config 2: 150 → 135 ms)
        //   otherwise:       8 × 4, 2 warps (K = 2048: 74 ms; 4 × 4 84 ms)
        const int ctas = 2 * tiles;
        auto run = [&](auto kern, int threads) {
            cudaError_t err = set_smem_attr_once(reinterpret_cast<const void*>(kern), static_cast<int>(kRefSmemBytes));
            if (err != cudaSuccess) return err;
            kern<<<ctas, threads, kRefSmemBytes, stream>>>(q, ld, rows, K, nb, packed, accumulate ? 1 : 0);
            return cudaSuccess;
        };
        if (ctas < 148) {
            e = run(gram_ref_kernel<2>, ref_threads<2>());
        } else if (ctas < 4 * 148) {
            e = run(gram_ref_kernel<4>, ref_threads<4>());
        } else {
            e = run(gram_ref_kernel<8>, ref_threads<8>());
        }
        if (e != cudaSuccess) return e;
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace gram
}  // namespace dopinf_b200
