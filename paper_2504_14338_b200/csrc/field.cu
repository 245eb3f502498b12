// field.cu — Step V field reconstruction (reference postprocess.cpp:63-70,
// transform.cpp:62-72): X = Φ_r · Q̃ᵀ in original coordinates,
//   X[row][t] = fma(s_row, Σ_k Φ_r[row][k] · Q̃[t][k], mean_row),
// s_row = scales[row / nx_i] (1 with scaling off), i.e. the reference's
// linalg::matmul_nt followed by inverse_transform_block's scale_shift (one FMA
// per output, kernels_avx2.cpp:125-133).
//
// Shape: rows × nt_p outputs with an inner dimension of only r (10–80), so the
// kernel is bound by max(FP64 tensor, HBM write): 2r flop per 8-byte output;
// the ridge is r ≈ 23 on B200. The product runs on DMMA.8x8x4 with the inverse
// transform fused into the epilogue, so X is written to HBM exactly once and
// never re-read.
//
// CTA tile 128 rows × 64 times, 8 warps of 32×32. The CTA's Φ_r tile (128 × r)
// stays in shared memory while the CTA walks its group of 64-wide time chunks;
// the chunks of Q̃ (64 × r, L2-resident: nt_p·r·8 bytes) stream through a
// two-slot cp.async ring. Operand rows are padded to a pitch P ≡ 8 (mod 16)
// doubles so each quarter-warp's 128-bit fragment loads hit 8 distinct 16-byte
// bank groups (conflict-free). Work items = (row tile, chunk group), strided
// over a persistent grid.
#include <algorithm>

#include "common.cuh"
#include "field.h"

namespace dopinf_b200 {
namespace field {
namespace {

constexpr int BM = 128;
constexpr int BN = 64;
constexpr int THREADS = 256;  // 8 warps: 4 (rows) × 2 (times), 32×32 each
constexpr int kMaxPitch = 104;  // r_pad ≤ 96 keeps Φ tile + 2 Q̃ slots ≤ 213 KB

__host__ __device__ constexpr int pitch_for(int r_pad) { return r_pad % 16 == 8 ? r_pad : r_pad + 8; }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// rows [row0, row0 + n) of a (limit × r_pad) row-major matrix (pitch ld) →
// shared (n × P); rows ≥ limit are zero-filled.
__device__ __forceinline__ void load_rows(uint32_t dst, const double* __restrict__ src, size_t ld, long long row0,
                                          int n, long long limit, int r_pad, int P) {
    const int per_row = r_pad / 2;  // 16-byte pieces
    for (int i = threadIdx.x; i < n * per_row; i += THREADS) {
        const int rr = i / per_row, cc = (i % per_row) * 2;
        const long long row = row0 + rr;
        const bool ok = row < limit;
        const double* s = src + (ok ? static_cast<size_t>(row) * ld + cc : 0);
        cp_async16(dst + static_cast<uint32_t>((rr * P + cc) * sizeof(double)), s, ok);
    }
}

__global__ void __launch_bounds__(THREADS, 1)
    field_dmma_kernel(const double* __restrict__ phi, size_t ldphi, const double* __restrict__ qt, size_t ldq,
                      long long rows, int nt_p, int r_pad, const double* __restrict__ means,
                      const double* __restrict__ scales, long long nx_i, long long row_base, double* __restrict__ out,
                      size_t ldo,
                      int n_groups, int chunks_per_group, int accumulate) {
    extern __shared__ __align__(16) double smem[];
    const int P = pitch_for(r_pad);
    double* as = smem;                 // BM × P   Φ_r tile
    double* bs = smem + BM * P;        // 2 × BN × P  Q̃ chunk slots
    const uint32_t as_u = smem_u32(as), bs_u = smem_u32(bs);
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int wm = warp & 3, wn = warp >> 2;
    const int g = lane >> 2, t = lane & 3;
    const long long n_rt = (rows + BM - 1) / BM;
    const int n_chunks = (nt_p + BN - 1) / BN;
    const long long n_items = n_rt * n_groups;
    long long cur_rt = -1;

    for (long long item = blockIdx.x; item < n_items; item += gridDim.x) {
        const long long rt = item / n_groups;
        const int cg = static_cast<int>(item % n_groups);
        const int c_begin = cg * chunks_per_group;
        const int c_end = min(n_chunks, c_begin + chunks_per_group);
        if (c_begin >= c_end) continue;
        __syncthreads();  // the previous item is done with both tiles
        if (rt != cur_rt) {
            load_rows(as_u, phi, ldphi, rt * BM, BM, rows, r_pad, P);
            cur_rt = rt;
        }
        load_rows(bs_u, qt, ldq, static_cast<long long>(c_begin) * BN, BN, nt_p, r_pad, P);
        cp_async_commit();

        // epilogue constants of this thread's 4 rows
        double s_row[4], m_row[4];
        long long row_of[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            const long long row = rt * BM + wm * 32 + mi * 8 + g;
            row_of[mi] = row;
            const bool ok = row < rows;
            s_row[mi] = ok && scales ? scales[(row_base + row) / nx_i] : 1.0;
            m_row[mi] = ok && means ? means[row] : 0.0;
        }

        for (int c = c_begin; c < c_end; ++c) {
            const int slot = (c - c_begin) & 1;
            if (c + 1 < c_end) {
                load_rows(bs_u + static_cast<uint32_t>((slot ^ 1) * BN * P * sizeof(double)), qt, ldq,
                          static_cast<long long>(c + 1) * BN, BN, nt_p, r_pad, P);
                cp_async_commit();
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();

            double acc[4][4][2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
            const uint32_t a0 = as_u + static_cast<uint32_t>(((wm * 32 + g) * P + 2 * t) * sizeof(double));
            const uint32_t b0 =
                bs_u + static_cast<uint32_t>(((slot * BN + wn * 32 + g) * P + 2 * t) * sizeof(double));
            const uint32_t step8 = static_cast<uint32_t>(8 * P * sizeof(double));  // 8 rows
#pragma unroll 2
            for (int k8 = 0; k8 < r_pad; k8 += 8) {
                const uint32_t ko = static_cast<uint32_t>(k8 * sizeof(double));
                double2 a[4], b[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    a[i] = lds128(a0 + i * step8 + ko);
                    b[i] = lds128(b0 + i * step8 + ko);
                }
                // k pairs (2t, 2t+1) of the 8-wide slab: the same permutation of
                // the contraction on both operands
#pragma unroll
                for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                    for (int ni = 0; ni < 4; ++ni) {
                        dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi].x, b[ni].x);
                        dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi].y, b[ni].y);
                    }
            }
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                if (row_of[mi] >= rows) continue;
                double* dst = out + static_cast<size_t>(row_of[mi]) * ldo;
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) {
                    const int col = c * BN + wn * 32 + ni * 8 + 2 * t;
                    if (accumulate && col < nt_p) {  // r > max_r_pad(): earlier k-slabs' raw sums
                        acc[mi][ni][0] += dst[col];
                        if (col + 1 < nt_p) acc[mi][ni][1] += dst[col + 1];
                    }
                    const double v0 = fma(s_row[mi], acc[mi][ni][0], m_row[mi]);
                    const double v1 = fma(s_row[mi], acc[mi][ni][1], m_row[mi]);
                    if (col + 1 < nt_p) {
                        __stcs(reinterpret_cast<double2*>(dst + col), make_double2(v0, v1));
                    } else if (col < nt_p) {
                        __stcs(dst + col, v0);
                    }
                }
            }
            __syncthreads();  // slot is refilled two chunks later
        }
    }
}

}  // namespace

int max_r_pad() { return kMaxPitch - 8; }

cudaError_t launch_field(const double* phi, size_t ldphi, const double* qt, size_t ldq, long long rows, int nt_p,
                         int r_pad, const double* means, const double* scales, long long nx_i, long long row_base,
                         double* out, size_t ldo, int accumulate, int num_sms, cudaStream_t stream) {
    if (rows <= 0 || nt_p <= 0) return cudaSuccess;
    if (r_pad % 8 != 0 || r_pad > max_r_pad() || ldo % 2 != 0 || ldphi % 2 != 0 || ldq % 2 != 0) {
        return cudaErrorInvalidValue;
    }
    const int P = pitch_for(r_pad);
    const size_t smem = static_cast<size_t>(BM + 2 * BN) * P * sizeof(double);
    // the attribute is set once per device: set it for the widest tile
    constexpr size_t kMaxSmem = static_cast<size_t>(BM + 2 * BN) * kMaxPitch * sizeof(double);
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(field_dmma_kernel), static_cast<int>(kMaxSmem));
    if (e != cudaSuccess) return e;
    // enough items for ~4 per CTA; the Φ tile is reused across a group's chunks
    const long long n_rt = (rows + BM - 1) / BM;
    const int n_chunks = (nt_p + BN - 1) / BN;
    const long long want = 4LL * num_sms;
    int n_groups = static_cast<int>(std::min<long long>(n_chunks, std::max<long long>(1, (want + n_rt - 1) / n_rt)));
    const int cpg = (n_chunks + n_groups - 1) / n_groups;
    n_groups = (n_chunks + cpg - 1) / cpg;
    const long long n_items = n_rt * n_groups;
    const int grid = static_cast<int>(std::min<long long>(n_items, num_sms));
    field_dmma_kernel<<<grid, THREADS, smem, stream>>>(phi, ldphi, qt, ldq, rows, nt_p, r_pad, means, scales,
                                                       nx_i, row_base, out, ldo, n_groups, cpg,
                                                       accumulate);
    note_launch();
    return cudaGetLastError();
}

}  // namespace field
}  // namespace dopinf_b200
