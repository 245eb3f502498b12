// rom.cu — §8(f) next-row 2: the OpInf regularisation grid search on the
// device (reference proj/src/rom_search.cpp:185-262, opinf.cpp:34-92).
//
// The reference, per candidate pair (β1, β2): rebuilds Dhatᵀ Dhat, solves
// (DhatᵀDhat + diag γ) X = Dhatᵀ Qhat2ᵀ with LAPACK dposv, integrates the
// quadratic ROM for nt_p steps and scores it. Here the pair-independent work
// runs once — Dhat (assemble_data) on the device, DhatᵀDhat on the FP64
// tensor pipe (the Gram kernel), Dhatᵀ Qhat2ᵀ in the reference's FMA order —
// then every pair of this rank's slice gets its Cholesky solve (cuSOLVER
// dpotrf/dpotrs), all pairs integrate concurrently (one CTA per pair) and are
// scored in one kernel; the winner is chosen as the reference does.
//
// The integrator reproduces rom_step_into (rom_search.cpp:38-48) bit for bit:
// per output i, c_i + dot(A_i, q) + dot(F_i, quad(q)) with kernels::dot's
// AVX2 order (kernels_avx2.cpp:32-46: lanes l = 0..7 each an FMA chain over
// elements 8b + l, lanes 0..3 also take the trailing block of four; then
// (l0+l4, l1+l5, l2+l6, l3+l7) summed as ((v0+v2)+(v1+v3)); the scalar tail
// unfused). Eight threads run the eight chains of one output. The scores
// follow training_error / growth_ratio (rom_search.cpp:94-145) in the
// reference's (unfused) order.
#include <cooperative_groups.h>

#include <algorithm>

#include "common.cuh"
#include "rom.h"

namespace dopinf_b200 {
namespace rom {

namespace {

// opinf.cpp:34-58 assemble_data: Dhat row k = [q_k, quad(q_k), 1], target row
// k = q_{k+1}; qhat is r × nt row-major (pitch nt).
__global__ void assemble_kernel(const double* __restrict__ qhat, int r, int nt, double* __restrict__ dhat,
                                size_t ldd, double* __restrict__ q2t) {
    const int k = blockIdx.x;  // 0 .. nt-2
    const int s = r * (r + 1) / 2;
    double* row = dhat + static_cast<size_t>(k) * ldd;
    for (int i = threadIdx.x; i < r; i += blockDim.x) {
        row[i] = qhat[static_cast<size_t>(i) * nt + k];
        q2t[static_cast<size_t>(k) * r + i] = qhat[static_cast<size_t>(i) * nt + k + 1];
    }
    // quad_features_into (opinf.cpp:8-15): pos runs over i ≤ j in row order
    for (int pos = threadIdx.x; pos < s; pos += blockDim.x) {
        // invert pos = i*r - i*(i-1)/2 + (j - i)
        int i = 0, base = 0;
        while (base + (r - i) <= pos) {
            base += r - i;
            ++i;
        }
        const int j = i + (pos - base);
        row[r + pos] = __dmul_rn(qhat[static_cast<size_t>(i) * nt + k], qhat[static_cast<size_t>(j) * nt + k]);
    }
    if (threadIdx.x == 0) {
        row[r + s] = 1.0;
        for (size_t c = r + s + 1; c < ldd; ++c) row[c] = 0.0;  // pitch padding
    }
}

// rhs (d × r, column-major: rhs[i + j·d]) = Dhatᵀ Qhat2ᵀ with linalg::matmul_tn's
// order (linalg.cpp:28-37: c.row(i) += a(l, i)·b.row(l) by axpy, an FMA chain over l).
__global__ void matmul_tn_cm_kernel(const double* __restrict__ a, size_t lda, const double* __restrict__ b, int K,
                                    int d, int r, double* __restrict__ out) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<long long>(d) * r) return;
    const int i = static_cast<int>(e % d), j = static_cast<int>(e / d);
    double acc = 0.0;
    for (int l = 0; l < K; ++l) acc = __fma_rn(a[static_cast<size_t>(l) * lda + i], b[static_cast<size_t>(l) * r + j], acc);
    out[e] = acc;
}

// G = DhatᵀDhat in linalg::gram's order (linalg.cpp:50-58: c.row(i) +=
// a(l, i)·a.row(l) by axpy → G(i, j) an FMA chain over l), so G is
// bit-identical to the reference's (and bitwise symmetric: the products
// commute). One thread per (i, j ≥ i); the CTA's warp runs along j.
__global__ void gram_exact_kernel(const double* __restrict__ a, size_t lda, int K, int d, double* __restrict__ g) {
    const int i = blockIdx.y;
    const int j = i + blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= d) return;
    double acc = 0.0;
    for (int l = 0; l < K; ++l) acc = __fma_rn(a[static_cast<size_t>(l) * lda + i], a[static_cast<size_t>(l) * lda + j], acc);
    g[static_cast<size_t>(i) * d + j] = acc;
    g[static_cast<size_t>(j) * d + i] = acc;
}

// Pair p's system: lhs_p = G + diag(γ_p) (opinf.cpp:76-77; build_regularizer
// opinf.cpp:60-67: β1 on the r state columns and the ones column, β2 on the s
// quadratic ones), rhs_p = rhs.
__global__ void systems_kernel(const double* __restrict__ g, int d, int r, const double* __restrict__ beta1,
                               const double* __restrict__ beta2, const double* __restrict__ rhs,
                               double* __restrict__ lhs, double* __restrict__ rhs_batch) {
    const int p = blockIdx.y;
    const size_t dd = static_cast<size_t>(d) * d;
    const int s = r * (r + 1) / 2;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < dd;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double v = g[e];
        const int i = static_cast<int>(e / d), j = static_cast<int>(e % d);
        if (i == j) v = __dadd_rn(v, (i >= r && i < r + s) ? beta2[p] : beta1[p]);
        lhs[static_cast<size_t>(p) * dd + e] = v;
    }
    const size_t dr = static_cast<size_t>(d) * r;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < dr;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        rhs_batch[static_cast<size_t>(p) * dr + e] = rhs[e];
    }
}

// One kernels::dot (kernels_avx2.cpp:32-46) by the 8 lanes of a group:
// lane l's FMA chain, the lane combine and hsum, lane 0's unfused tail.
// Returns the dot on lane 0 of the group (other lanes: garbage).
__device__ __forceinline__ double group_dot(const double* __restrict__ a, const double* __restrict__ b, int n,
                                            int l, unsigned gmask) {
    const int nb8 = n / 8;
    const bool four = n - 8 * nb8 >= 4;
    double acc = 0.0;
    int blk = 0;
    // eight loads in flight ahead of each eight-long stretch of the FMA chain
    for (; blk + 8 <= nb8; blk += 8) {
        double x[8], y[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            x[u] = a[8 * (blk + u) + l];  // global or shared (generic load)
            y[u] = b[8 * (blk + u) + l];
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __fma_rn(x[u], y[u], acc);
    }
    for (; blk < nb8; ++blk) acc = __fma_rn(a[8 * blk + l], b[8 * blk + l], acc);
    if (four && l < 4) acc = __fma_rn(a[8 * nb8 + l], b[8 * nb8 + l], acc);
    // v_l = acc0_l + acc1_l (lanes l and l + 4)
    const double hi = __shfl_down_sync(gmask, acc, 4, 8);
    const double v = __dadd_rn(acc, hi);
    // hsum: (v0 + v2) + (v1 + v3)
    const double v2 = __shfl_down_sync(gmask, v, 2, 8);
    const double w = __dadd_rn(v, v2);  // lane 0: v0+v2, lane 1: v1+v3
    const double w1 = __shfl_down_sync(gmask, w, 1, 8);
    double h = __dadd_rn(w, w1);
    if (l == 0) {
        for (int t = 8 * nb8 + (four ? 4 : 0); t < n; ++t) h = __dadd_rn(h, __dmul_rn(a[t], b[t]));
    }
    return h;
}

// All pairs' ROMs in parallel, one CTA per pair: integrate (rom_search.cpp:
// 62-87) from q0 for n_steps rows. ops_p: column-major d × r (column i =
// [A_i (r), F_i (s), c_i]: the solve's output layout). traj_p: n_steps × r.
__global__ void __launch_bounds__(1024)
    integrate_kernel(const double* __restrict__ ops, int r, const double* __restrict__ q0, int n_steps,
                     double* __restrict__ traj) {
    extern __shared__ double sm[];
    const int s = r * (r + 1) / 2;
    const int d = r + s + 1;
    const int p = blockIdx.x;
    const double* x = ops + static_cast<size_t>(p) * d * r;
    double* tp = traj + static_cast<size_t>(p) * n_steps * r;
    double* q = sm;           // r: current state
    double* feat = sm + r;    // s: quad(q)
    int* pi = reinterpret_cast<int*>(feat + s);  // s: (i << 16 | j) of feature pos
    const int groups = blockDim.x / 8;
    const int g = threadIdx.x / 8, l = threadIdx.x % 8;
    const unsigned gmask = 0xFFu << (8 * ((threadIdx.x % 32) / 8));
    for (int i = 0, pos = 0; i < r; ++i) {
        for (int j = i; j < r; ++j, ++pos) {
            if (pos % blockDim.x == static_cast<int>(threadIdx.x)) pi[pos] = (i << 16) | j;
        }
    }
    for (int i = threadIdx.x; i < r; i += blockDim.x) {
        q[i] = q0[i];
        tp[i] = q0[i];
    }
    __syncthreads();
    for (int k = 0; k + 1 < n_steps; ++k) {
        for (int pos = threadIdx.x; pos < s; pos += blockDim.x) {
            const int e = pi[pos];
            feat[pos] = __dmul_rn(q[e >> 16], q[e & 0xFFFF]);
        }
        __syncthreads();
        double outv[8];  // outputs of this group (r ≤ 8·groups·8)
        int n_out = 0;
        for (int i = g; i < r; i += groups, ++n_out) {
            const double* col = x + static_cast<size_t>(i) * d;
            const double da = group_dot(col, q, r, l, gmask);
            const double df = group_dot(col + r, feat, s, l, gmask);
            outv[n_out & 7] = __dadd_rn(__dadd_rn(col[r + s], da), df);  // c_i + dot(A_i, q) + dot(F_i, feat)
        }
        __syncthreads();  // everyone has read q and feat
        n_out = 0;
        for (int i = g; i < r; i += groups, ++n_out) {
            if (l == 0) {
                q[i] = outv[n_out & 7];
                tp[static_cast<size_t>(k + 1) * r + i] = outv[n_out & 7];
            }
        }
        __syncthreads();
    }
}

// The same integration with each pair's operators resident in shared memory:
// a cluster of CL CTAs per pair, CTA k holding the operator columns of outputs
// [k·rpc, (k+1)·rpc) (rpc·d doubles). Every CTA forms quad(q) itself, computes
// its outputs from shared memory, and writes them into every cluster member's
// next-state buffer (distributed shared memory); one cluster barrier per step.
// Same arithmetic, same order as integrate_kernel (group_dot), so the same bits.
__global__ void __launch_bounds__(1024)
    integrate_cluster_kernel(const double* __restrict__ ops, int r, const double* __restrict__ q0, int n_steps,
                             int rpc, double* __restrict__ traj) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double smc[];
    const int s = r * (r + 1) / 2;
    const int d = r + s + 1;
    const int CL = static_cast<int>(cluster.num_blocks());
    const int cr = static_cast<int>(cluster.block_rank());
    const int p = blockIdx.x / CL;
    const int i0 = cr * rpc, i1 = min(r, i0 + rpc);
    const double* x = ops + static_cast<size_t>(p) * d * r;
    double* tp = traj + static_cast<size_t>(p) * n_steps * r;
    double* cols = smc;                                     // rpc × d: this CTA's operator columns
    double* qb = cols + static_cast<size_t>(rpc) * d;       // 2 × r: state, double-buffered
    double* feat = qb + 2 * r;                              // s
    int* pi = reinterpret_cast<int*>(feat + s);             // s
    const int g = threadIdx.x / 8, l = threadIdx.x % 8;
    const unsigned gmask = 0xFFu << (8 * ((threadIdx.x % 32) / 8));
    for (size_t e = threadIdx.x; e < static_cast<size_t>(i1 - i0) * d; e += blockDim.x) {
        cols[e] = x[static_cast<size_t>(i0) * d + e];
    }
    for (int i = 0, pos = 0; i < r; ++i) {
        for (int j = i; j < r; ++j, ++pos) {
            if (pos % blockDim.x == static_cast<int>(threadIdx.x)) pi[pos] = (i << 16) | j;
        }
    }
    for (int i = threadIdx.x; i < r; i += blockDim.x) {
        qb[i] = q0[i];
        if (cr == 0) tp[i] = q0[i];
    }
    cluster.sync();
    int cur = 0;
    for (int k = 0; k + 1 < n_steps; ++k) {
        const double* q = qb + cur * r;
        for (int pos = threadIdx.x; pos < s; pos += blockDim.x) {
            const int e = pi[pos];
            feat[pos] = __dmul_rn(q[e >> 16], q[e & 0xFFFF]);
        }
        __syncthreads();
        const int i = i0 + g;
        if (i < i1) {
            const double* col = cols + static_cast<size_t>(g) * d;
            const double da = group_dot(col, q, r, l, gmask);
            const double df = group_dot(col + r, feat, s, l, gmask);
            const double v = __dadd_rn(__dadd_rn(col[r + s], da), df);  // c_i + dot(A_i, q) + dot(F_i, feat)
            if (l == 0) {
                for (int m = 0; m < CL; ++m) cluster.map_shared_rank(qb + (cur ^ 1) * r, m)[i] = v;
                tp[static_cast<size_t>(k + 1) * r + i] = v;
            }
        }
        cluster.sync();  // next state complete everywhere; q and feat no longer read
        cur ^= 1;
    }
}

// X = L⁻ᵀ L⁻¹ B for one pair's Cholesky factor (column-major, lower: L[i + j·d])
// and a chunk of kSolveCols right-hand sides held in shared memory, in blocks
// of kSolveBlock unknowns (two CTA barriers per block instead of per unknown):
//  forward  — the block's small triangle solved by one lane per right-hand
//             side, then every row below updated with the block's solutions
//             (8-term FMA sums along L's contiguous columns);
//  backward — each warp forms, for one unknown of the block, the dots of its
//             L column below the block with the solved x (two lanes per
//             right-hand side), then the block's triangle is solved upward.
constexpr int kSolveCols = 16;
constexpr int kSolveThreads = 256;
constexpr int kSolveBlock = 8;

__global__ void __launch_bounds__(kSolveThreads)
    chol_solve_kernel(const double* __restrict__ lbatch, int d, double* __restrict__ bbatch, int r) {
    extern __shared__ double xs[];  // d × kSolveCols, column c at xs[c·d]
    __shared__ double part[kSolveBlock][kSolveCols];
    const int p = blockIdx.y;
    const int c0 = blockIdx.x * kSolveCols;
    const int nc = min(kSolveCols, r - c0);
    const double* L = lbatch + static_cast<size_t>(p) * d * d;
    double* B = bbatch + static_cast<size_t>(p) * d * r;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int e = threadIdx.x; e < d * nc; e += blockDim.x) {
        const int c = e / d, i = e % d;
        xs[c * d + i] = B[static_cast<size_t>(c0 + c) * d + i];
    }
    __syncthreads();
    // ---- forward: L y = b ----
    for (int j0 = 0; j0 < d; j0 += kSolveBlock) {
        const int nb = min(kSolveBlock, d - j0);
        if (threadIdx.x < nc) {
            double* x = xs + threadIdx.x * d;
            for (int jj = 0; jj < nb; ++jj) {
                const int j = j0 + jj;
                const double y = x[j] / L[static_cast<size_t>(j) * d + j];
                x[j] = y;
                for (int kk = jj + 1; kk < nb; ++kk) x[j0 + kk] = fma(-L[static_cast<size_t>(j) * d + j0 + kk], y, x[j0 + kk]);
            }
        }
        __syncthreads();
        const int rows = d - j0 - nb;
        for (int e = threadIdx.x; e < rows * nc; e += blockDim.x) {
            const int c = e / rows, i = j0 + nb + e % rows;
            double acc = xs[c * d + i];
#pragma unroll
            for (int jj = 0; jj < kSolveBlock; ++jj) {
                if (jj < nb) acc = fma(-L[static_cast<size_t>(j0 + jj) * d + i], xs[c * d + j0 + jj], acc);
            }
            xs[c * d + i] = acc;
        }
        __syncthreads();
    }
    // ---- backward: Lᵀ x = y ----
    const int nblk = (d + kSolveBlock - 1) / kSolveBlock;
    for (int blk = nblk - 1; blk >= 0; --blk) {
        const int j0 = blk * kSolveBlock, nb = min(kSolveBlock, d - j0);
        // warp w: unknown j0 + w; lanes (c, half): dot of L column j below the block with x
        if (warp < nb) {
            const int j = j0 + warp, c = lane / 2, h = lane % 2;
            double acc = 0.0;
            if (c < nc) {
                const double* col = L + static_cast<size_t>(j) * d;
                for (int i = j0 + nb + h; i < d; i += 2) acc = fma(col[i], xs[c * d + i], acc);
            }
            acc += __shfl_down_sync(0xFFFFFFFFu, acc, 1);
            if (h == 0 && c < kSolveCols) part[warp][c] = acc;
        }
        __syncthreads();
        if (threadIdx.x < nc) {
            const int c = threadIdx.x;
            double* x = xs + c * d;
            for (int jj = nb - 1; jj >= 0; --jj) {
                const int j = j0 + jj;
                double v = x[j] - part[jj][c];
                for (int kk = jj + 1; kk < nb; ++kk) v = fma(-L[static_cast<size_t>(j) * d + j0 + kk], x[j0 + kk], v);
                x[j] = v / L[static_cast<size_t>(j) * d + j];
            }
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < d * nc; e += blockDim.x) {
        const int cc = e / d, i = e % d;
        B[static_cast<size_t>(c0 + cc) * d + i] = xs[cc * d + i];
    }
}

// Scores of one pair per CTA: finite (integrate's check), training_error over
// the first nt rows against qhat_rows (nt × r), growth_ratio; flags a zero-norm
// reference row / constant training data the way the reference throws.
__global__ void __launch_bounds__(256)
    score_kernel(const double* __restrict__ traj, int n_steps, int r, const double* __restrict__ qrows, int nt,
                 double* __restrict__ out) {
    const int p = blockIdx.x;
    const double* t = traj + static_cast<size_t>(p) * n_steps * r;
    __shared__ double red[256];
    __shared__ int flag;
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    // finite over the whole trajectory
    int bad = 0;
    for (size_t e = threadIdx.x; e < static_cast<size_t>(n_steps) * r; e += blockDim.x) bad |= !isfinite(t[e]);
    if (bad) atomicOr(&flag, 1);
    __syncthreads();
    const bool finite = flag == 0;
    // training_error (rom_search.cpp:94-115): max over rows of sqrt(num/den)
    double worst = 0.0;
    int zero_row = -1;
    for (int k = threadIdx.x; k < nt; k += blockDim.x) {
        double num = 0.0, den = 0.0;
        for (int j = 0; j < r; ++j) {
            const double ref = qrows[static_cast<size_t>(k) * r + j];
            const double diff = __dsub_rn(t[static_cast<size_t>(k) * r + j], ref);
            num = __dadd_rn(num, __dmul_rn(diff, diff));
            den = __dadd_rn(den, __dmul_rn(ref, ref));
        }
        if (den == 0.0) {
            if (zero_row < 0) zero_row = k;
        } else {
            worst = fmax(worst, sqrt(num / den));
        }
    }
    red[threadIdx.x] = worst;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + st]);
        __syncthreads();
    }
    const double train_err = red[0];
    __syncthreads();
    // growth_ratio (rom_search.cpp:117-145): per-mode mean of the training rows
    double train_dev = 0.0, trial_dev = 0.0;
    for (int j = threadIdx.x; j < r; j += blockDim.x) {
        double mu = 0.0;
        for (int k = 0; k < nt; ++k) mu = __dadd_rn(mu, qrows[static_cast<size_t>(k) * r + j]);
        mu = __ddiv_rn(mu, static_cast<double>(nt));
        for (int k = 0; k < nt; ++k) train_dev = fmax(train_dev, fabs(__dsub_rn(qrows[static_cast<size_t>(k) * r + j], mu)));
        for (int k = 0; k < n_steps; ++k) trial_dev = fmax(trial_dev, fabs(__dsub_rn(t[static_cast<size_t>(k) * r + j], mu)));
    }
    red[threadIdx.x] = train_dev;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + st]);
        __syncthreads();
    }
    const double tdev = red[0];
    __syncthreads();
    red[threadIdx.x] = trial_dev;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + st]);
        __syncthreads();
    }
    const double rdev = red[0];
    __syncthreads();
    // first zero-norm row over the block
    __shared__ int zr;
    if (threadIdx.x == 0) zr = 0x7FFFFFFF;
    __syncthreads();
    if (zero_row >= 0) atomicMin(&zr, zero_row);
    __syncthreads();
    if (threadIdx.x == 0) {
        double* o = out + static_cast<size_t>(p) * kScoreFields;
        o[0] = finite ? 1.0 : 0.0;
        o[1] = train_err;
        o[2] = tdev == 0.0 ? 0.0 : rdev / tdev;
        o[3] = zr == 0x7FFFFFFF ? -1.0 : static_cast<double>(zr);
        o[4] = tdev == 0.0 ? 1.0 : 0.0;
    }
}

__global__ void transpose_kernel(const double* __restrict__ a, int rows, int cols, double* __restrict__ t) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<long long>(rows) * cols) return;
    const int i = static_cast<int>(e / cols), j = static_cast<int>(e % cols);
    t[static_cast<size_t>(j) * rows + i] = a[e];
}

}  // namespace

cudaError_t launch_assemble(const double* qhat, int r, int nt, double* dhat, size_t ldd, double* q2t,
                            cudaStream_t stream) {
    if (nt < 2) return cudaSuccess;
    assemble_kernel<<<nt - 1, 256, 0, stream>>>(qhat, r, nt, dhat, ldd, q2t);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_gram_exact(const double* dhat, size_t ldd, int K, int d, double* g, cudaStream_t stream) {
    gram_exact_kernel<<<dim3((d + 127) / 128, d), 128, 0, stream>>>(dhat, ldd, K, d, g);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_rhs(const double* dhat, size_t ldd, const double* q2t, int K, int d, int r, double* rhs_cm,
                       cudaStream_t stream) {
    const long long total = static_cast<long long>(d) * r;
    matmul_tn_cm_kernel<<<static_cast<int>((total + 127) / 128), 128, 0, stream>>>(dhat, ldd, q2t, K, d, r, rhs_cm);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_systems(const double* g, int d, int r, const double* beta1, const double* beta2, int n_pairs,
                           const double* rhs_cm, double* lhs, double* rhs_batch, cudaStream_t stream) {
    if (n_pairs <= 0) return cudaSuccess;
    const size_t dd = static_cast<size_t>(d) * d;
    const int gx = static_cast<int>(std::min<size_t>((dd + 255) / 256, 256));
    systems_kernel<<<dim3(gx, n_pairs), 256, 0, stream>>>(g, d, r, beta1, beta2, rhs_cm, lhs, rhs_batch);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_integrate(const double* ops, int r, const double* q0, int n_steps, int n_pairs, double* traj,
                             cudaStream_t stream) {
    if (n_pairs <= 0) return cudaSuccess;
    const int s = r * (r + 1) / 2;
    const int d = r + s + 1;
    constexpr size_t kSmemCap = 200 * 1024;
    // Operators that fit L1 stay there (one CTA per pair, the plain kernel);
    // larger ones are held in shared memory by the smallest cluster (2..8
    // CTAs) whose slices of operator columns fit.
    const bool l1_resident = static_cast<size_t>(r) * d * sizeof(double) <= 160 * 1024;
    for (int CL = 2; !l1_resident && CL <= 8; CL *= 2) {
        const int rpc = (r + CL - 1) / CL;
        if (rpc > 128) continue;  // ≤ 1024 threads: 8 per output
        const size_t smem = (static_cast<size_t>(rpc) * d + 2 * r + s) * sizeof(double) + s * sizeof(int);
        if (smem > kSmemCap) continue;
        cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(integrate_cluster_kernel), kSmemCap);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n_pairs * CL);
        cfg.blockDim = dim3(std::max(32, (8 * rpc + 31) / 32 * 32));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = CL;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, integrate_cluster_kernel, ops, r, q0, n_steps, rpc, traj);
        note_launch();
        return e != cudaSuccess ? e : cudaGetLastError();
    }
    // operators in L1 (or too large even for a cluster's shared memory: L2)
    const int threads = std::min(1024, std::max(32, ((8 * r + 31) / 32) * 32));
    const int groups = threads / 8;
    if ((r + groups - 1) / groups > 8) return cudaErrorInvalidValue;  // outputs per group
    const size_t smem = static_cast<size_t>(r + s) * sizeof(double) + static_cast<size_t>(s) * sizeof(int);
    if (smem > kSmemCap) return cudaErrorInvalidValue;
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(integrate_kernel), kSmemCap);
    if (e != cudaSuccess) return e;
    integrate_kernel<<<n_pairs, threads, smem, stream>>>(ops, r, q0, n_steps, traj);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_chol_solve(const double* l, int d, int batch, double* b, int r, cudaStream_t stream) {
    if (batch <= 0) return cudaSuccess;
    const size_t smem = static_cast<size_t>(d) * kSolveCols * sizeof(double);
    if (smem > 220 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(chol_solve_kernel), 220 * 1024);
    if (e != cudaSuccess) return e;
    chol_solve_kernel<<<dim3((r + kSolveCols - 1) / kSolveCols, batch), kSolveThreads, smem, stream>>>(l, d, b, r);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_score(const double* traj, int n_steps, int r, const double* qrows, int nt, int n_pairs,
                         double* out, cudaStream_t stream) {
    if (n_pairs <= 0) return cudaSuccess;
    score_kernel<<<n_pairs, 256, 0, stream>>>(traj, n_steps, r, qrows, nt, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_transpose(const double* a, int rows, int cols, double* t, cudaStream_t stream) {
    const long long total = static_cast<long long>(rows) * cols;
    if (total == 0) return cudaSuccess;
    transpose_kernel<<<static_cast<int>((total + 255) / 256), 256, 0, stream>>>(a, rows, cols, t);
    note_launch();
    return cudaGetLastError();
}

}  // namespace rom
}  // namespace dopinf_b200
