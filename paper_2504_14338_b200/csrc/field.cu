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
// TMA ring. The kernel is instantiated per contraction extent RP = r rounded
// up to 4 (a last k-step of four when RP ≡ 4 mod 8), so no DMMA multiplies
// padding. Operand rows are padded to a pitch P ≡ 8 (mod 16)
// doubles so each quarter-warp's 128-bit fragment loads hit 8 distinct 16-byte
// bank groups (conflict-free). Work items = (row tile, chunk group), strided
// over a persistent grid.
#include <algorithm>

#include "common.cuh"
#include "field.h"

namespace dopinf_b200 {
namespace field {
namespace {

constexpr int THREADS = 256;  // 8 warps: 4 (rows) × 2 (times), 32×32 each
constexpr int kMaxPitch = 104;  // r_pad ≤ 96 keeps Φ tile + 2 Q̃ slots ≤ 213 KB

// Shared-memory pitch of a row of RP doubles: the smallest P ≥ RP with
// P ≡ 8 (mod 16), so each quarter-warp's 128-bit fragment loads hit 8
// distinct 16-byte bank groups.
__host__ __device__ constexpr int pitch_for(int rp) { return rp + ((8 - rp % 16) + 16) % 16; }

__device__ __forceinline__ double lds64(uint32_t saddr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(saddr));
    return v;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0)
                 : "memory");
}

constexpr int BM = 128;  // rows per tile: 4 warp rows of 32
constexpr int BN = 64;   // times per chunk: 2 warp columns of 32

// rows [row0, row0 + N) of a (limit × RP) row-major matrix (pitch ld) → shared
// (N × P); rows ≥ limit are zero-filled. Each thread's copies complete on
// their own; the caller ties them to an mbarrier.
template <int RP, int N>
__device__ __forceinline__ void load_rows(uint32_t dst, const double* __restrict__ src, size_t ld, long long row0,
                                          long long limit) {
    constexpr int per_row = RP / 2;  // 16-byte pieces
    constexpr int P = pitch_for(RP);
#pragma unroll
    for (int j = 0; j < (N * per_row + THREADS - 1) / THREADS; ++j) {
        const int i = threadIdx.x + j * THREADS;
        if ((N * per_row) % THREADS != 0 && i >= N * per_row) break;
        const int rr = i / per_row, cc = (i % per_row) * 2;
        const long long row = row0 + rr;
        const bool ok = row < limit;
        const double* s = src + (ok ? static_cast<size_t>(row) * ld + cc : 0);
        cp_async16(dst + static_cast<uint32_t>((rr * P + cc) * sizeof(double)), s, ok);
    }
}

__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

template <int RP, int S>
struct FieldSmem {
    static constexpr int P = pitch_for(RP);
    double b[S][BN * P];    // ring of Q̃ chunks (TMA destinations, 128-byte aligned)
    double a[BM * P];       // Φ_r tile of the current item
    double scale[BM];       // epilogue s_row
    double mean[BM];        // epilogue mean_row
    uint64_t full[S];       // chunk landed (TMA transaction count)
    int released[S];        // warps done with the chunk in the slot
};

// Items = (row tile, chunk group). Within an item each warp walks the chunks
// on its own; the LAST warp to release a chunk's slot refills it with the
// chunk S ahead by TMA (one elected thread, no waiting), so no warp ever waits
// for another inside an item and one warp's epilogue (the HBM stores)
// overlaps the others' DMMA. CTA barriers only at item boundaries.
template <int RP, int S>
__global__ void __launch_bounds__(THREADS, 2)
    field_dmma_kernel(const __grid_constant__ CUtensorMap qmap, const double* __restrict__ phi, size_t ldphi,
                      long long rows, int nt_p, const double* __restrict__ means, const double* __restrict__ scales,
                      long long nx_i, long long row_base, double* __restrict__ out, size_t ldo, int n_groups,
                      int chunks_per_group, int accumulate) {
    using Sm = FieldSmem<RP, S>;
    constexpr int P = Sm::P;
    constexpr uint32_t kSlotBytes = BN * P * sizeof(double);
    constexpr int kWarps = THREADS / kWarp;
    extern __shared__ unsigned char smem_raw[];
    Sm& sm = *reinterpret_cast<Sm*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~static_cast<uintptr_t>(127));
    const uint32_t as_u = smem_u32(sm.a), bs_u = smem_u32(sm.b[0]);
    const int warp = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    const int wm = warp & 3, wn = warp >> 2;
    const int g = lane >> 2, t = lane & 3;
    const long long n_rt = (rows + BM - 1) / BM;
    const int n_chunks = (nt_p + BN - 1) / BN;
    const long long n_items = n_rt * n_groups;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&qmap);
        for (int s = 0; s < S; ++s) {
            mbar_init(&sm.full[s], 1);
            sm.released[s] = 0;
        }
        fence_mbar_init();
    }
    __syncthreads();

    uint32_t q = 0;  // this CTA's running chunk sequence number (same in every thread)
    for (long long item = blockIdx.x; item < n_items; item += gridDim.x) {
        const long long rt = item / n_groups;
        const int cg = static_cast<int>(item % n_groups);
        const int c_begin = cg * chunks_per_group;
        const int c_end = min(n_chunks, c_begin + chunks_per_group);
        if (c_begin >= c_end) continue;
        __syncthreads();  // every warp is done with the previous item's tiles
        if (threadIdx.x < BM) {
            const long long row = rt * BM + threadIdx.x;
            const bool ok = row < rows;
            sm.scale[threadIdx.x] = ok && scales ? scales[(row_base + row) / nx_i] : 1.0;
            sm.mean[threadIdx.x] = ok && means ? means[row] : 0.0;
        }
        if (threadIdx.x == 0) {  // the first S chunks of the item
            fence_proxy_async();
            for (int k = 0; k < S && c_begin + k < c_end; ++k) {
                const uint32_t slot = (q + k) % S;
                mbar_arrive_expect_tx(&sm.full[slot], kSlotBytes);
                tma_load_2d(sm.b[slot], &qmap, 0, (c_begin + k) * BN, &sm.full[slot]);
            }
        }
        load_rows<RP, BM>(as_u, phi, ldphi, rt * BM, rows);
        cp_async_wait_all();
        __syncthreads();  // Φ_r tile and epilogue constants visible

        for (int c = c_begin; c < c_end; ++c, ++q) {
            const uint32_t slot = q % S, phase = (q / S) & 1u;
            mbar_wait(&sm.full[slot], phase);

            double acc[4][4][2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
            const uint32_t a0 = as_u + static_cast<uint32_t>(((wm * 32 + g) * P + 2 * t) * sizeof(double));
            const uint32_t b0 =
                bs_u + slot * kSlotBytes + static_cast<uint32_t>(((wn * 32 + g) * P + 2 * t) * sizeof(double));
            constexpr uint32_t step8 = 8 * P * sizeof(double);  // 8 rows
            // two passes over k, one per half of the warp's 32 times: the stores
            // of the first half issue while the second half's DMMAs drain
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
                for (int k8 = 0; k8 + 8 <= RP; k8 += 8) {
                    const uint32_t ko = static_cast<uint32_t>(k8 * sizeof(double));
                    double2 a[4], b[2];
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[i] = lds128(a0 + i * step8 + ko);
#pragma unroll
                    for (int j = 0; j < 2; ++j) b[j] = lds128(b0 + (2 * h + j) * step8 + ko);
                    // k pairs (2t, 2t+1) of the 8-wide slab: the same permutation of
                    // the contraction on both operands
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            dmma_8x8x4(acc[mi][2 * h + j][0], acc[mi][2 * h + j][1], a[mi].x, b[j].x);
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            dmma_8x8x4(acc[mi][2 * h + j][0], acc[mi][2 * h + j][1], a[mi].y, b[j].y);
                }
                if constexpr (RP % 8 == 4) {  // a last k-step of four: lane (g, t) takes k = RP − 4 + t
                    const uint32_t at = as_u + static_cast<uint32_t>(((wm * 32 + g) * P + RP - 4 + t) * sizeof(double));
                    const uint32_t bt = bs_u + slot * kSlotBytes +
                                        static_cast<uint32_t>(((wn * 32 + g) * P + RP - 4 + t) * sizeof(double));
                    double a[4], b[2];
#pragma unroll
                    for (int i = 0; i < 4; ++i) a[i] = lds64(at + i * step8);
#pragma unroll
                    for (int j = 0; j < 2; ++j) b[j] = lds64(bt + (2 * h + j) * step8);
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            dmma_8x8x4(acc[mi][2 * h + j][0], acc[mi][2 * h + j][1], a[mi], b[j]);
                }
            }
            // every DMMA above consumed its shared-memory operands (scoreboard), so
            // the warp is done reading the slot
            __syncwarp();
            if (lane == 0 && c + S < c_end) {
                if (atomicAdd(&sm.released[slot], 1) == kWarps - 1) {
                    sm.released[slot] = 0;
                    fence_proxy_async();  // generic-proxy reads before the async-proxy write
                    mbar_arrive_expect_tx(&sm.full[slot], kSlotBytes);
                    tma_load_2d(sm.b[slot], &qmap, 0, (c + S) * BN, &sm.full[slot]);
                }
            }

            // epilogue half by half: the first half's results are final while the
            // second half's DMMAs still drain. Interior chunks of full row tiles
            // (all but the last chunk at nt_p % 64 != 0) take a branch-free path.
            if (!accumulate && (c + 1) * BN <= nt_p && (rt + 1) * BM <= rows) {
                const uint32_t sc_u = smem_u32(sm.scale), mn_u = smem_u32(sm.mean);
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) {
                        const int lr = wm * 32 + mi * 8 + g;
                        const double s_row = lds64(sc_u + lr * 8), m_row = lds64(mn_u + lr * 8);
                        double* dst = out + static_cast<size_t>(rt * BM + lr) * ldo + c * BN + wn * 32 + 2 * t;
#pragma unroll
                        for (int ni = 2 * h; ni < 2 * h + 2; ++ni) {
                            __stcs(reinterpret_cast<double2*>(dst + ni * 8),
                                   make_double2(fma(s_row, acc[mi][ni][0], m_row), fma(s_row, acc[mi][ni][1], m_row)));
                        }
                    }
                continue;
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const int lr = wm * 32 + mi * 8 + g;
                const long long row = rt * BM + lr;
                if (row >= rows) continue;
                const double s_row = sm.scale[lr], m_row = sm.mean[lr];
                double* dst = out + static_cast<size_t>(row) * ldo;
#pragma unroll
                for (int ni = 2 * h; ni < 2 * h + 2; ++ni) {
                    const int col = c * BN + wn * 32 + ni * 8 + 2 * t;
                    if (accumulate && col < nt_p) {  // r > max_r_pad(): earlier k-slabs' raw sums
                        acc[mi][ni][0] += dst[col];
                        if (col + 1 < nt_p) acc[mi][ni][1] += dst[col + 1];
                    }
                    const double v0 = fma(s_row, acc[mi][ni][0], m_row);
                    const double v1 = fma(s_row, acc[mi][ni][1], m_row);
                    if (col + 1 < nt_p) {
                        __stcs(reinterpret_cast<double2*>(dst + col), make_double2(v0, v1));
                    } else if (col < nt_p) {
                        __stcs(dst + col, v0);
                    }
                }
            }
        }
    }
}

}  // namespace

int max_r_pad() { return kMaxPitch - 8; }

namespace {

// Q̃ (nt_p × RP, pitch ldq) as a 2-D tensor; a box is one chunk of BN rows ×
// P columns (columns ≥ RP and rows ≥ nt_p arrive as zeros).
cudaError_t q_map(CUtensorMap* map, const double* qt, size_t ldq, int nt_p, int rp, int p) {
    auto fn = tensor_map_encoder();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rp), static_cast<cuuint64_t>(nt_p)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldq * sizeof(double))};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(p), static_cast<cuuint32_t>(BN)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(qt), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int RP>
cudaError_t launch_rp(const double* phi, size_t ldphi, const double* qt, size_t ldq, long long rows, int nt_p,
                      const double* means, const double* scales, long long nx_i, long long row_base, double* out,
                      size_t ldo, int accumulate, int num_sms, cudaStream_t stream) {
    // three ring slots while two CTAs still fit an SM, else two
    constexpr bool kThree = 2 * (sizeof(FieldSmem<RP, 3>) + 128 + 1024) <= 228 * 1024;
    constexpr int S = kThree ? 3 : 2;
    constexpr size_t smem = sizeof(FieldSmem<RP, S>) + 128;
    auto kern = field_dmma_kernel<RP, S>;
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    CUtensorMap qmap;
    e = q_map(&qmap, qt, ldq, nt_p, RP, FieldSmem<RP, S>::P);
    if (e != cudaSuccess) return e;
    // enough items for ~8 per CTA slot; the Φ_r tile is reused across a group's chunks
    const long long n_rt = (rows + BM - 1) / BM;
    const int n_chunks = (nt_p + BN - 1) / BN;
    const long long want = 8LL * num_sms;
    int n_groups = static_cast<int>(std::min<long long>(n_chunks, std::max<long long>(1, (want + n_rt - 1) / n_rt)));
    const int cpg = (n_chunks + n_groups - 1) / n_groups;
    n_groups = (n_chunks + cpg - 1) / cpg;
    const long long n_items = n_rt * n_groups;
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem) != cudaSuccess || per_sm < 1) {
        per_sm = 1;
    }
    const int grid = static_cast<int>(std::min<long long>(n_items, static_cast<long long>(num_sms) * per_sm));
    kern<<<grid, THREADS, smem, stream>>>(qmap, phi, ldphi, rows, nt_p, means, scales, nx_i, row_base, out, ldo,
                                          n_groups, cpg, accumulate);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_field(const double* phi, size_t ldphi, const double* qt, size_t ldq, long long rows, int nt_p,
                         int k_ext, const double* means, const double* scales, long long nx_i, long long row_base,
                         double* out, size_t ldo, int accumulate, int num_sms, cudaStream_t stream) {
    if (rows <= 0 || nt_p <= 0) return cudaSuccess;
    if (k_ext % 4 != 0 || k_ext < 4 || k_ext > max_r_pad() || ldo % 2 != 0 || ldphi % 2 != 0 || ldq % 2 != 0) {
        return cudaErrorInvalidValue;
    }
#define DOPINF_FIELD(RP) \
    case RP / 4:         \
        return launch_rp<RP>(phi, ldphi, qt, ldq, rows, nt_p, means, scales, nx_i, row_base, out, ldo, accumulate, \
                             num_sms, stream)
    switch (k_ext / 4) {
        DOPINF_FIELD(4);
        DOPINF_FIELD(8);
        DOPINF_FIELD(12);
        DOPINF_FIELD(16);
        DOPINF_FIELD(20);
        DOPINF_FIELD(24);
        DOPINF_FIELD(28);
        DOPINF_FIELD(32);
        DOPINF_FIELD(36);
        DOPINF_FIELD(40);
        DOPINF_FIELD(44);
        DOPINF_FIELD(48);
        DOPINF_FIELD(52);
        DOPINF_FIELD(56);
        DOPINF_FIELD(60);
        DOPINF_FIELD(64);
        DOPINF_FIELD(68);
        DOPINF_FIELD(72);
        DOPINF_FIELD(76);
        DOPINF_FIELD(80);
        DOPINF_FIELD(84);
        DOPINF_FIELD(88);
        DOPINF_FIELD(92);
        default: DOPINF_FIELD(96);
    }
#undef DOPINF_FIELD
}

}  // namespace field
}  // namespace dopinf_b200
