// project.cu — the products after the Gram (reference pod.cpp, postprocess.cpp).
//
//  * project_kernel: Q̂ = T_rᵀ D (pod::project → linalg::matmul_tn,
//    pod.cpp:103-105, linalg.cpp:28-37). Each output is the reference's FMA
//    chain over l = 0..K−1 in order (c[i][j] = fma(T_r[l][i], D[l][j], c)), so
//    Q̂ is bit-identical to the reference's for the same T_r and D. D and T_r
//    slabs are staged through shared memory so the chains run at FMA latency.
//  * basis_rows_kernel: postprocess::basis_rows (postprocess.cpp:12-34), the
//    reference's unfused acc + q·tr loop in order → bit-identical.
//  * basis_dmma_kernel: Φ_r = Q·T_r (postprocess.cpp:66 reconstruct_field's
//    linalg::matmul), a tall-skinny GEMM on the FP64 tensor pipe. Q row-slabs
//    (BM rows × 16 snapshots) and the matching slab of T_rᵀ stream through a
//    TMA ring with 128-byte swizzle; consumers read both operands with
//    conflict-free 128-bit shared loads (two k-steps per load) and run
//    DMMA.8x8x4. One CTA covers all r columns (padded to a multiple of 8 only),
//    so Q is read from HBM exactly once.
#include <algorithm>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "project.h"

namespace dopinf_b200 {
namespace project {

namespace {

// ---- Q̂ = T_rᵀ D, reference order ---------------------------------------------
// One FMA chain per output (the chains are the parallelism: r·K of them), so a
// step costs one FMA latency once its operands are in shared memory. Block =
// 8 warps = 8 rows i × 32 columns j; slabs of kPjL values of l (D rows and T_r
// rows) arrive by cp.async into a double buffer while the previous slab's
// chains run.
constexpr int kPjCols = 32;   // columns j per block (lane = j)
constexpr int kPjWarps = 8;   // rows i per block (warp = i)
constexpr int kPjL = 128;     // l-slab staged in shared memory

__device__ __forceinline__ void cp_async8(uint32_t dst, const double* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0)
                 : "memory");
}

struct ProjectSmem {
    double ds[2][kPjL][kPjCols];
    double ts[2][kPjL][kPjWarps];
};

__global__ void __launch_bounds__(kPjCols * kPjWarps)
    project_kernel(const double* __restrict__ tr, const double* __restrict__ d, int K, int r,
                   double* __restrict__ qhat) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ProjectSmem& sm = *reinterpret_cast<ProjectSmem*>(smem_raw);
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
    const int j0 = blockIdx.x * kPjCols, i0 = blockIdx.y * kPjWarps;
    const int j = j0 + lane, i = i0 + w;
    const int n_slabs = (K + kPjL - 1) / kPjL;
    auto stage = [&](int slab, int buf) {
        const int l0 = slab * kPjL;
        for (int e = threadIdx.x; e < kPjL * kPjCols; e += blockDim.x) {
            const int l = e / kPjCols, c = e % kPjCols;
            const bool ok = l0 + l < K && j0 + c < K;
            cp_async8(smem_u32(&sm.ds[buf][l][c]), ok ? d + static_cast<size_t>(l0 + l) * K + j0 + c : d, ok);
        }
        for (int e = threadIdx.x; e < kPjL * kPjWarps; e += blockDim.x) {
            const int l = e / kPjWarps, c = e % kPjWarps;
            const bool ok = l0 + l < K && i0 + c < r;
            cp_async8(smem_u32(&sm.ts[buf][l][c]), ok ? tr + static_cast<size_t>(l0 + l) * r + i0 + c : tr, ok);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    double acc = 0.0;
    stage(0, 0);
    for (int slab = 0; slab < n_slabs; ++slab) {
        const int buf = slab & 1;
        if (slab + 1 < n_slabs) {
            stage(slab + 1, buf ^ 1);  // the buffer the previous slab used (all threads are past it)
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        const int nl = min(kPjL, K - slab * kPjL);
#pragma unroll 8
        for (int l = 0; l < nl; ++l) acc = fma(sm.ts[buf][l][w], sm.ds[buf][l][lane], acc);
        __syncthreads();  // everyone is done with `buf` before it is refilled
    }
    if (j < K && i < r) qhat[static_cast<size_t>(i) * K + j] = acc;
}

__global__ void basis_rows_kernel(const double* __restrict__ q, size_t ld, int K,
                                  const double* __restrict__ tr, int r,
                                  const long long* __restrict__ rows, int nsel,
                                  double* __restrict__ out) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<long long>(nsel) * r) return;
    const int k = static_cast<int>(e / r), jj = static_cast<int>(e % r);
    const double* qr = q + static_cast<size_t>(rows[k]) * ld;
    double acc = 0.0;
    for (int t = 0; t < K; ++t) acc = __dadd_rn(acc, __dmul_rn(qr[t], tr[static_cast<size_t>(t) * r + jj]));
    out[e] = acc;
}

// postprocess::reconstruct_probes (postprocess.cpp:36-61): series[t] =
// kernels::dot(basis_row, Q̃.row(t), r) in the AVX2 order (kernels_avx2.cpp:
// 32-46: two 4-lane FMA accumulators over blocks of 8, the trailing block of
// 4 into the first, (v0+v2)+(v1+v3), then the tail with a rounded product),
// then inverse_transform_row's scale_shift: fma(s, x, mean). One thread per
// (probe, t) → bit-identical to the reference.
__global__ void probe_series_kernel(const double* __restrict__ basis, int r, const double* __restrict__ qt,
                                    int nt_p, const long long* __restrict__ rows, const double* __restrict__ means,
                                    const double* __restrict__ scales, long long nx_i, int nsel,
                                    double* __restrict__ out) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<long long>(nsel) * nt_p) return;
    const int k = static_cast<int>(e / nt_p), t = static_cast<int>(e % nt_p);
    const double* a = basis + static_cast<size_t>(k) * r;
    const double* b = qt + static_cast<size_t>(t) * r;
    double c0[4] = {0.0, 0.0, 0.0, 0.0}, c1[4] = {0.0, 0.0, 0.0, 0.0};
    int i = 0;
    for (; i + 8 <= r; i += 8) {
#pragma unroll
        for (int l = 0; l < 4; ++l) {
            c0[l] = __fma_rn(a[i + l], b[i + l], c0[l]);
            c1[l] = __fma_rn(a[i + 4 + l], b[i + 4 + l], c1[l]);
        }
    }
    for (; i + 4 <= r; i += 4) {
#pragma unroll
        for (int l = 0; l < 4; ++l) c0[l] = __fma_rn(a[i + l], b[i + l], c0[l]);
    }
    double v[4];
#pragma unroll
    for (int l = 0; l < 4; ++l) v[l] = __dadd_rn(c0[l], c1[l]);
    double acc = __dadd_rn(__dadd_rn(v[0], v[2]), __dadd_rn(v[1], v[3]));
    for (; i < r; ++i) acc = __dadd_rn(acc, __dmul_rn(a[i], b[i]));
    const long long row = rows[k];
    const double s = scales ? scales[row / nx_i] : 1.0;
    out[e] = __fma_rn(s, acc, means[row]);
}

// ---- Φ_r = Q · T_r on DMMA ---------------------------------------------------
// Warp grid WM × WN (8 consumer warps); warp tile 32 rows × 8·NT columns.
// CTA tile BM = 32·WM rows × BN = 8·NT·WN columns.
constexpr int BKB = 16;     // snapshots per stage (128 B rows → 128B swizzle)
constexpr int CONSUMERS = 8;
constexpr int THREADS = (CONSUMERS + 1) * 32;

template <int WM, int WN, int NT>
struct Cfg {
    static constexpr int BM = 32 * WM;
    static constexpr int BN = 8 * NT * WN;
    static constexpr int STAGES = (BM + BN) * BKB * 8 * 6 <= 200 * 1024 ? 6 : 5;
};

template <int WM, int WN, int NT>
struct __align__(1024) BasisSmem {
    using C = Cfg<WM, WN, NT>;
    double a[C::STAGES][C::BM * BKB];
    double b[C::STAGES][((C::BN * BKB + 127) / 128) * 128];  // 1 KiB-aligned slabs
    uint64_t full[C::STAGES];
    uint64_t empty[C::STAGES];
};

// (row, chunk) of a [rows][16 doubles] tile written by TMA with 128B swizzle.
__device__ __forceinline__ const double* swz(const double* base, int row, int chunk) {
    return base + row * BKB + ((chunk ^ (row & 7)) << 1);
}

template <int WM, int WN, int NT>
__global__ void __launch_bounds__(THREADS, 1)
    basis_dmma_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap tmap,
                      long long rows, int K, double* __restrict__ phi, int ldp) {
    using C = Cfg<WM, WN, NT>;
    constexpr int BM = C::BM, BN = C::BN, STAGES = C::STAGES;
    extern __shared__ unsigned char smem_raw[];
    BasisSmem<WM, WN, NT>& s = *reinterpret_cast<BasisSmem<WM, WN, NT>*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const long long n_rb = (rows + BM - 1) / BM;
    const int nkb = (K + BKB - 1) / BKB;
    const int col0 = blockIdx.y * BN;

    if (threadIdx.x == 0) {
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(&s.full[st], 1);
            mbar_init(&s.empty[st], CONSUMERS);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == CONSUMERS) {
        if (lane == 0) {
            tma_prefetch_desc(&qmap);
            tma_prefetch_desc(&tmap);
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t bytes = (BM + BN) * BKB * sizeof(double);
            for (long long rb = blockIdx.x; rb < n_rb; rb += gridDim.x) {
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&s.empty[stage], phase ^ 1u);
                    mbar_arrive_expect_tx(&s.full[stage], bytes);
                    tma_load_2d(s.a[stage], &qmap, kb * BKB, static_cast<int>(rb * BM), &s.full[stage]);
                    tma_load_2d(s.b[stage], &tmap, kb * BKB, col0, &s.full[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else {
        const int g = lane >> 2, t = lane & 3;
        const int wm = warp % WM, wn = warp / WM;
        int stage = 0;
        uint32_t phase = 0;
        for (long long rb = blockIdx.x; rb < n_rb; rb += gridDim.x) {
            double acc[4][NT][2];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
                for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&s.full[stage], phase);
                const double* as = s.a[stage];
                const double* bs = s.b[stage];
#pragma unroll
                for (int kh = 0; kh < 2; ++kh) {
                    const int chunk = kh * 4 + t;
                    double2 a[4], b[NT];
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) a[mi] = lds128(swz(as, wm * 32 + mi * 8 + g, chunk));
#pragma unroll
                    for (int ni = 0; ni < NT; ++ni) b[ni] = lds128(swz(bs, wn * 8 * NT + ni * 8 + g, chunk));
#pragma unroll
                    for (int mi = 0; mi < 4; ++mi) {
#pragma unroll
                        for (int ni = 0; ni < NT; ++ni) {
                            dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi].x, b[ni].x);
                            dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], a[mi].y, b[ni].y);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.empty[stage]);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const long long row = rb * BM + wm * 32 + mi * 8 + g;
                if (row < rows) {
                    double* dst = phi + static_cast<size_t>(row) * ldp + col0 + wn * 8 * NT + 2 * t;
#pragma unroll
                    for (int ni = 0; ni < NT; ++ni) {
                        __stcs(reinterpret_cast<double2*>(dst + ni * 8),
                               make_double2(acc[mi][ni][0], acc[mi][ni][1]));
                    }
                }
            }
        }
    }
}


cudaError_t map_2d(CUtensorMap* map, const double* base, long long rows, int cols, size_t ld,
                   int box_rows) {
    auto fn = tensor_map_encoder();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * sizeof(double))};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(BKB), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int WM, int WN, int NT>
cudaError_t launch_basis_cfg(const double* q, size_t ld, long long rows, int K, const double* trt,
                             size_t ldt, int col_blocks, double* phi, int ldp, int num_sms,
                             cudaStream_t stream) {
    using Cf = Cfg<WM, WN, NT>;
    CUtensorMap qmap, tmap;
    cudaError_t e = map_2d(&qmap, q, rows, K, ld, Cf::BM);
    if (e != cudaSuccess) return e;
    e = map_2d(&tmap, trt, static_cast<long long>(col_blocks) * Cf::BN, K, ldt, Cf::BN);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(BasisSmem<WM, WN, NT>) + 1024;
    e = set_smem_attr_once(reinterpret_cast<const void*>(basis_dmma_kernel<WM, WN, NT>), static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const long long n_rb = (rows + Cf::BM - 1) / Cf::BM;
    const int gx = static_cast<int>(std::max<long long>(
        1, std::min<long long>(n_rb, std::max(1, num_sms / col_blocks))));
    basis_dmma_kernel<WM, WN, NT><<<dim3(gx, col_blocks), THREADS, smem, stream>>>(qmap, tmap, rows, K, phi, ldp);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

// Padded Φ_r width: a multiple of 8 up to 48 (one warp column, 256-row CTA
// tiles), else a multiple of 16 up to 128 (two warp columns), else of 128.
int basis_cols_pad(int r) {
    if (r <= 48) return std::max(8, (r + 7) / 8 * 8);
    if (r <= 128) return (r + 15) / 16 * 16;
    return (r + 127) / 128 * 128;
}

cudaError_t launch_project(const double* tr, const double* d, int K, int r, double* qhat,
                           cudaStream_t stream) {
    dim3 grid((K + kPjCols - 1) / kPjCols, (r + kPjWarps - 1) / kPjWarps);
    const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(project_kernel),
                                             static_cast<int>(sizeof(ProjectSmem)));
    if (e != cudaSuccess) return e;
    project_kernel<<<grid, kPjCols * kPjWarps, sizeof(ProjectSmem), stream>>>(tr, d, K, r, qhat);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_basis_rows(const double* q, size_t ld, int K, const double* tr, int r,
                              const long long* rows, int nsel, double* out, cudaStream_t stream) {
    const long long total = static_cast<long long>(nsel) * r;
    if (total == 0) return cudaSuccess;
    basis_rows_kernel<<<static_cast<int>((total + 127) / 128), 128, 0, stream>>>(q, ld, K, tr, r,
                                                                                rows, nsel, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_probe_series(const double* basis, int r, const double* qt, int nt_p, const long long* rows,
                                const double* means, const double* scales, long long nx_i, int nsel, double* out,
                                cudaStream_t stream) {
    const long long total = static_cast<long long>(nsel) * nt_p;
    if (total == 0) return cudaSuccess;
    probe_series_kernel<<<static_cast<int>((total + 127) / 128), 128, 0, stream>>>(basis, r, qt, nt_p, rows, means,
                                                                                 scales, nx_i, nsel, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_basis(const double* q, size_t ld, long long rows, int K, const double* trt,
                         size_t ldt, int r_pad, double* phi, int num_sms, cudaStream_t stream) {
#define DOPINF_BASIS(WM, WN, NT, CB) \
    return launch_basis_cfg<WM, WN, NT>(q, ld, rows, K, trt, ldt, CB, phi, r_pad, num_sms, stream)
    if (r_pad > 128) DOPINF_BASIS(4, 2, 8, r_pad / 128);
    if (r_pad > 48) {
        switch (r_pad / 16) {
            case 4: DOPINF_BASIS(4, 2, 4, 1);
            case 5: DOPINF_BASIS(4, 2, 5, 1);
            case 6: DOPINF_BASIS(4, 2, 6, 1);
            case 7: DOPINF_BASIS(4, 2, 7, 1);
            default: DOPINF_BASIS(4, 2, 8, 1);
        }
    }
    switch (r_pad / 8) {
        case 1: DOPINF_BASIS(8, 1, 1, 1);
        case 2: DOPINF_BASIS(8, 1, 2, 1);
        case 3: DOPINF_BASIS(8, 1, 3, 1);
        case 4: DOPINF_BASIS(8, 1, 4, 1);
        case 5: DOPINF_BASIS(8, 1, 5, 1);
        default: DOPINF_BASIS(8, 1, 6, 1);
    }
#undef DOPINF_BASIS
}

}  // namespace project
}  // namespace dopinf_b200
