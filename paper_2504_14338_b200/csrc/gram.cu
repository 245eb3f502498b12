// gram.cu — D = QᵀQ, upper triangle only, on the FP64 tensor pipe (sm_100a).
//
// Replaces pod::local_gram → linalg::gram (reference proj/src/pod.cpp:11-13,
// proj/src/linalg.cpp:50-58), which loops over the FULL square with
// kernels::axpy. Here:
//   * Q (rows × K, row-major, pitch ld) is cut into 128-column blocks; only
//     output tiles (I, J) with I <= J are computed (K(K+1)/2 useful entries).
//   * The contraction dimension (rows) is split into S chunks (4K rows, the
//     last ones quartered so the final wave ends together); a work item is
//     (split s, tile). Items are handed out s-major from a global
//     atomic queue, so the CTAs running at any moment read the same rows of
//     Q (L2 reuse across the ~tiles CTAs that need them).
//   * Each persistent CTA = 1 TMA producer warp + 16 consumer warps. The
//     producer streams 48×128 row-slabs of the I and J column blocks (8 boxes
//     of 16 columns, 128-byte swizzle; boxes wholly beyond column K are not
//     loaded) through a double-buffered mbarrier ring
//     (cp.async.bulk.tensor, OOB rows/cols zero-filled); consumers run
//     mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) on 32×32 warp tiles with
//     fragments read as conflict-free 128-bit shared loads.
//   * Diagonal tiles skip warp tiles / mma tiles strictly below the diagonal
//     and edge tiles skip columns >= K — through compile-time mma masks (the
//     few partial shapes that occur), never predicated DMMA; tiles with fewer
//     than 16 active warp tiles have their largest ones cut in halves so every
//     consumer warp works, and the warp tiles are balanced over the 4 SM
//     sub-partitions on the host (exact min-max assignment, planned once per K).
//   * Each item's partial goes to a workspace in fragment order; a second
//     kernel sums the S partials of every tile in split order s = 0..S-1 (in
//     two fixed levels — groups of consecutive splits, then the groups — when
//     the tiles alone cannot fill the GPU) — fixed order, no atomics on data,
//     bitwise reproducible — and writes the packed upper triangle. A third kernel expands it to the symmetric K×K
//     D (bitwise symmetric, as linalg.hpp:17 promises for the reference).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <vector>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "gram.h"

namespace dopinf_b200 {
namespace gram {

namespace {

constexpr int BT = kTileEdge;         // 128 columns per block
constexpr int BK = kRowsPerStage;     // rows per stage
#ifndef DOPINF_GRAM_STAGES  // (build-time tuning knob)
#define DOPINF_GRAM_STAGES 2
#endif
constexpr int STAGES = DOPINF_GRAM_STAGES;
constexpr int CONSUMERS = kConsumerWarps;  // 16 = 4 consumer warpgroups
constexpr int THREADS = (CONSUMERS + 1) * kWarp;  // + one TMA producer warp
constexpr int FLAG_FIRST = 1, FLAG_LAST = 2, FLAG_DONE = 4;

struct __align__(1024) Smem {
    double a[STAGES][BK * BT];
    double b[STAGES][BK * BT];
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    int meta_item[STAGES];
    int meta_flags[STAGES];
};

// Warp-tile entry: wm | wn << 2 | diag << 4 | mma mask << 16 (0 mask = idle).
__host__ __device__ __forceinline__ void decode(uint32_t e, int& wm, int& wn, bool& diag, uint32_t& mask) {
    wm = e & 3;
    wn = (e >> 2) & 3;
    diag = (e >> 4) & 1;
    mask = e >> 16;
}

// Operand tile of one stage: 8 TMA boxes of BK rows × 16 doubles (one 128 B
// line per row) written with the 128-byte swizzle: element (row, col) of box
// col/16 sits in 16-byte chunk ((col%16)/2) ^ (row%8) of its line.
//
// Fragment loads: lane (g, t) reads, for mma k-step ks, Q row
// (ks/2)*8 + ks%2 + 2t — so within a quarter-warp the four rows have
// row%8 ∈ {0,2,4,6} (or {1,3,5,7}) — and columns 2g, 2g+1 as one 128-bit load.
// The swizzle then puts the quarter-warp's 8 loads in 8 distinct chunks:
// conflict-free (4 wavefronts per 512 B). ks permutes the contraction order
// only; the output mapping is unchanged.
// MASK: the mma tiles (bit mi*4 + ni) of the warp tile, fixed at compile
// time so skipped tiles cost nothing (a predicated-off DMMA still occupies
// the tensor pipe). The partial masks that occur for any K are few:
// diagonal 0x8CEF, column edge 0x1111/0x3333/0x7777, and their combinations
// 0x0001/0x0023/0x0033/0x0467; plus the halves plan_tiles cuts from warp tiles
// of tiles with fewer than 16 active warp tiles (0x3333/0xCCCC, 0x0023/0x8CCC,
// 0x3333/0x4444 by columns; 0x0033/0x3300, 0x00CC/0xCC00 by rows).
// Diagonal warp tiles: rows and columns of an mma tile are interleaved (even
// or odd members of a 16-block), so inside a diagonal 16-block the (odd rows,
// even columns) mma tile holds only entries whose transposes the (even rows,
// odd columns) one computes; it is skipped (12 -> 10 mma) and the reduction
// writes those entries from their transposes (D is symmetric, and the two
// dot products are the same products summed in the same k order).
// Where accumulator element c of lane `lane` in mma tile `mma` of warp tile
// (wm, wn) of output tile (I, J) lands in the packed upper triangle, or -1
// (below the diagonal or beyond K). Below-diagonal entries of an (even rows,
// odd columns) mma tile inside a diagonal 16-block are the entries of the
// skipped (odd, even) tile: they land at their transposes. Shared by the
// reduction and the host-side coverage check (dopinf_b200_debug_gram_coverage).
__host__ __device__ __forceinline__ long long scatter_index(int I, int J, int wm, int wn, bool diag, int mma,
                                                            int lane, int c, int K) {
    const int g = lane >> 2, t = lane & 3;
    const int mi = mma >> 2, ni = mma & 3;
    const int row = I * BT + wm * 32 + (mi >> 1) * 16 + 2 * g + (mi & 1);
    const int col = J * BT + wn * 32 + (ni >> 1) * 16 + 2 * (2 * t + c) + (ni & 1);
    if (row >= K || col >= K) return -1;
    const long long Kl = K;
    if (row <= col) return static_cast<long long>(row) * (2 * Kl - row + 1) / 2 + (col - row);
    if (diag && wm == wn && (mi >> 1) == (ni >> 1) && (mi & 1) == 0 && (ni & 1) == 1)
        return static_cast<long long>(col) * (2 * Kl - col + 1) / 2 + (row - col);
    return -1;
}

template <uint32_t MASK>
__device__ __forceinline__ void stage_mma(double (&acc)[16][2], const double* __restrict__ as,
                                          const double* __restrict__ bs, int xg0, int xg1, uint32_t mask) {
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
        const int off = ((ks >> 1) * 8 + (ks & 1)) * 16 + ((ks & 1) ? xg1 : xg0);
        const double2 a0 = lds128(as + off);
        const double2 a1 = lds128(as + off + BK * 16);
        const double2 b0 = lds128(bs + off);
        const double2 b1 = lds128(bs + off + BK * 16);
        const double a[4] = {a0.x, a0.y, a1.x, a1.y};
        const double b[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const bool on = MASK != 0 ? ((MASK >> (mi * 4 + ni)) & 1u) != 0 : ((mask >> (mi * 4 + ni)) & 1u) != 0;
                if (on) dmma_8x8x4(acc[mi * 4 + ni][0], acc[mi * 4 + ni][1], a[mi], b[ni]);
            }
        }
    }
}

// Dispatch on the warp tile's mask (warp-uniform); MASK 0 = generic predicated path.
__device__ __forceinline__ void stage_mma_any(double (&acc)[16][2], const double* __restrict__ as,
                                              const double* __restrict__ bs, int xg0, int xg1, uint32_t mask) {
    switch (mask) {
        case 0xFFFFu: stage_mma<0xFFFFu>(acc, as, bs, xg0, xg1, mask); break;
        case 0x8CEFu: stage_mma<0x8CEFu>(acc, as, bs, xg0, xg1, mask); break;
        case 0x8CCCu: stage_mma<0x8CCCu>(acc, as, bs, xg0, xg1, mask); break;
        case 0x0023u: stage_mma<0x0023u>(acc, as, bs, xg0, xg1, mask); break;
        case 0x7777u: stage_mma<0x7777u>(acc, as, bs, xg0, xg1, mask); break;
        case 0x3333u: stage_mma<0x3333u>(acc, as, bs, xg0, xg1, mask); break;
        case 0x1111u: stage_mma<0x1111u>(acc, as, bs, xg0, xg1, mask); break;
        case 0x0467u: stage_mma<0x0467u>(acc, as, bs, xg0, xg1, mask); break;
        case 0x0033u: stage_mma<0x0033u>(acc, as, bs, xg0, xg1, mask); break;
        case 0x0001u: stage_mma<0x0001u>(acc, as, bs, xg0, xg1, mask); break;
        case 0xCCCCu: stage_mma<0xCCCCu>(acc, as, bs, xg0, xg1, mask); break;
        case 0x4444u: stage_mma<0x4444u>(acc, as, bs, xg0, xg1, mask); break;
        case 0x3300u: stage_mma<0x3300u>(acc, as, bs, xg0, xg1, mask); break;
        case 0x00CCu: stage_mma<0x00CCu>(acc, as, bs, xg0, xg1, mask); break;
        case 0xCC00u: stage_mma<0xCC00u>(acc, as, bs, xg0, xg1, mask); break;
        default: stage_mma<0u>(acc, as, bs, xg0, xg1, mask); break;
    }
}

__global__ void __launch_bounds__(THREADS, 1)
    gram_dmma_kernel(const __grid_constant__ CUtensorMap tmap, const TileInfo* __restrict__ tiles,
                     int n_tiles, int n_items, long long n_rows, int K, int chunk_rows, int big_splits,
                     int small_rows,
                     double* __restrict__ work, int* __restrict__ counters, int accumulate, int keep_partials) {
    extern __shared__ unsigned char smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int warp = threadIdx.x / kWarp;
    const int lane = threadIdx.x % kWarp;

    if (threadIdx.x == 0) {
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(&s.full[st], 1);
            mbar_init(&s.empty[st], CONSUMERS);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == CONSUMERS) {
        // ---------------- TMA producer (one lane) ----------------
        if (lane == 0) {
            tma_prefetch_desc(&tmap);
            int stage = 0;
            uint32_t phase = 0;
            for (;;) {
                const int item = atomicAdd(&counters[0], 1);
                if (item >= n_items) {
                    mbar_wait(&s.empty[stage], phase ^ 1u);
                    s.meta_flags[stage] = FLAG_DONE;
                    mbar_arrive(&s.full[stage]);
                    break;
                }
                const int tile = item % n_tiles;
                const int split = item / n_tiles;
                const int I = tiles[tile].I, J = tiles[tile].J;
                // Guided split sizes: big_splits chunks of chunk_rows, then short
                // chunks of small_rows so the last wave of items ends together.
                const long long row0 = split < big_splits
                                           ? static_cast<long long>(split) * chunk_rows
                                           : static_cast<long long>(big_splits) * chunk_rows +
                                                 static_cast<long long>(split - big_splits) * small_rows;
                const long long rows =
                    min(static_cast<long long>(split < big_splits ? chunk_rows : small_rows), n_rows - row0);
                const int nkb = static_cast<int>((rows + BK - 1) / BK);
                const bool diag = (I == J);
                // boxes entirely beyond column K are never read by an active mma
                // tile: skip them (no TMA, no zero fill)
                const int boxes_a = min(BT / 16, (K - I * BT + 15) / 16);
                const int boxes_b = diag ? 0 : min(BT / 16, (K - J * BT + 15) / 16);
                const uint32_t bytes = static_cast<uint32_t>(boxes_a + boxes_b) * BK * 16 * sizeof(double);
                for (int kb = 0; kb < nkb; ++kb) {
                    mbar_wait(&s.empty[stage], phase ^ 1u);
                    s.meta_item[stage] = item;
                    s.meta_flags[stage] = (kb == 0 ? FLAG_FIRST : 0) | (kb == nkb - 1 ? FLAG_LAST : 0);
                    mbar_arrive_expect_tx(&s.full[stage], bytes);
                    const int y = static_cast<int>(row0 + static_cast<long long>(kb) * BK);
                    for (int box = 0; box < boxes_a; ++box) {
                        tma_load_2d(s.a[stage] + box * BK * 16, &tmap, I * BT + box * 16, y, &s.full[stage]);
                    }
                    for (int box = 0; box < boxes_b; ++box) {
                        tma_load_2d(s.b[stage] + box * BK * 16, &tmap, J * BT + box * 16, y, &s.full[stage]);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1u;
                    }
                }
            }
        }
    } else {
        // ---------------- DMMA consumers ----------------
        const int g = lane >> 2, t = lane & 3;
        const int xg0 = (g ^ (2 * t)) << 1, xg1 = (g ^ (2 * t + 1)) << 1;
        double acc[16][2];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.0;
        int wm = 0, wn = 0;
        bool diag = false;
        uint32_t mask = 0;
        int stage = 0;
        uint32_t phase = 0;
        for (;;) {
            mbar_wait(&s.full[stage], phase);
            const int flags = s.meta_flags[stage];
            if (flags & FLAG_DONE) break;
            const int item = s.meta_item[stage];
            if (flags & FLAG_FIRST) decode(tiles[item % n_tiles].warp[warp], wm, wn, diag, mask);
            if (mask) {
                const double* as = s.a[stage] + (2 * wm) * BK * 16 + 2 * t * 16;
                const double* bs = (diag ? s.a[stage] : s.b[stage]) + (2 * wn) * BK * 16 + 2 * t * 16;
                stage_mma_any(acc, as, bs, xg0, xg1, mask);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.empty[stage]);
            if ((flags & FLAG_LAST) && mask) {
                double* w = work + (static_cast<size_t>(item) * CONSUMERS + warp) * kWarpFragDoubles +
                            lane * 2;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if ((mask >> i) & 1u) {
                        double2* p = reinterpret_cast<double2*>(w + i * 64);
                        double2 v = make_double2(acc[i][0], acc[i][1]);
                        if (accumulate) {  // streamed chunks: slot += this chunk's partial, chunk order
                            const double2 old = __ldcg(p);
                            v.x = old.x + v.x;
                            v.y = old.y + v.y;
                        }
                        // one-launch partials are read once by the reduce: evict-first keeps
                        // Q's rows in L2 (-0.15 GB of re-reads at C2); streamed launches
                        // re-read their slots in the next chunk: keep those in L2
                        if (keep_partials) {
                            __stcg(p, v);
                        } else {
                            __stcs(p, v);
                        }
                    }
                    acc[i][0] = acc[i][1] = 0.0;
                }
            }
            if (++stage == STAGES) {
                stage = 0;
                phase ^= 1u;
            }
        }
    }

    // Self-resetting queue: the last CTA out zeroes the counters for the next launch.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const int prev = atomicAdd(&counters[1], 1);
        if (prev == static_cast<int>(gridDim.x) - 1) {
            counters[0] = 0;
            counters[1] = 0;
            __threadfence();
        }
    }
}

// Fixed-order split-n reduction: block = (split group, tile, warp slot),
// thread = (mma, lane). With one group the S partials of a tile are summed in
// split order and scattered into the packed triangle; with several (few tiles,
// many splits: the tiles alone cannot fill the GPU) each group's consecutive
// splits are summed in order into group_out, whose layout is the workspace's
// with "split" = group, and a second launch with one group sums those in group
// order. Either way the order is fixed: bitwise reproducible.
__global__ void __launch_bounds__(512)
    gram_reduce_kernel(const TileInfo* __restrict__ tiles, int n_tiles, int n_splits, int K,
                       const double* __restrict__ work, double* __restrict__ packed, int n_groups,
                       double* __restrict__ group_out) {
    const int per_group_blocks = n_tiles * CONSUMERS;
    const int grp = blockIdx.x / per_group_blocks;
    const int tile = (blockIdx.x % per_group_blocks) / CONSUMERS;
    const int slot = blockIdx.x % CONSUMERS;
    int wm, wn;
    bool diag;
    uint32_t mask;
    decode(tiles[tile].warp[slot], wm, wn, diag, mask);
    const int mma = threadIdx.x / kWarp, lane = threadIdx.x % kWarp;
    if (!((mask >> mma) & 1u)) return;
    const int per = (n_splits + n_groups - 1) / n_groups;
    const int sp0 = grp * per, sp1 = min(n_splits, sp0 + per);
    if (sp0 >= sp1) return;
    const size_t frag = static_cast<size_t>(slot) * kWarpFragDoubles + mma * 64 + lane * 2;
    const size_t item_stride = static_cast<size_t>(n_tiles) * CONSUMERS * kWarpFragDoubles;
    const double* p = work + static_cast<size_t>(tile) * CONSUMERS * kWarpFragDoubles + frag;
    double2 sum = __ldcg(reinterpret_cast<const double2*>(p + sp0 * item_stride));
    // kReduceBatch loads in flight per thread, then the adds in split order
    // (the summation order, hence the bits, do not depend on the batching)
    constexpr int kReduceBatch = 8;
    int sp = sp0 + 1;
    for (; sp + kReduceBatch <= sp1; sp += kReduceBatch) {
        double2 v[kReduceBatch];
#pragma unroll
        for (int u = 0; u < kReduceBatch; ++u)
            v[u] = __ldcs(reinterpret_cast<const double2*>(p + (sp + u) * item_stride));
#pragma unroll
        for (int u = 0; u < kReduceBatch; ++u) {
            sum.x += v[u].x;
            sum.y += v[u].y;
        }
    }
    for (; sp < sp1; ++sp) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(p + sp * item_stride));
        sum.x += v.x;
        sum.y += v.y;
    }
    if (n_groups > 1) {
        __stcg(reinterpret_cast<double2*>(group_out + grp * item_stride +
                                          static_cast<size_t>(tile) * CONSUMERS * kWarpFragDoubles + frag),
               sum);
        return;
    }
    const double vals[2] = {sum.x, sum.y};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        const long long idx = scatter_index(tiles[tile].I, tiles[tile].J, wm, wn, diag, mma, lane, c, K);
        if (idx >= 0) packed[idx] = vals[c];
    }
}

// packed upper triangle (row-major) -> full symmetric K×K, row-major, pitch K.
__global__ void unpack_kernel(const double* __restrict__ packed, int K, double* __restrict__ d) {
    const size_t total = static_cast<size_t>(K) * K;
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t i = e / K, j = e % K;
        const size_t r = i < j ? i : j, c = i < j ? j : i;
        d[e] = packed[r * (2 * static_cast<size_t>(K) - r + 1) / 2 + (c - r)];
    }
}

// Streamed pass: D = Σ_v (G_v / s_v) / s_v over the per-variable Grams of the
// centered rows, variables in order (scales == nullptr: plain Σ_v G_v). Two
// divisions rather than one by s_v²: s_v² leaves the double range for
// |s_v| outside ~[1e-154, 1e154] where the reference's scaled values are fine.
__global__ void combine_vars_kernel(const double* __restrict__ gv, int n_vars, size_t count,
                                    const double* __restrict__ scales, double* __restrict__ out) {
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double acc = 0.0;
        for (int v = 0; v < n_vars; ++v) {
            const double g = gv[static_cast<size_t>(v) * count + e];
            acc += scales ? g / scales[v] / scales[v] : g;
        }
        out[e] = acc;
    }
}

// Ascending-rank sum of p packed triangles (comm_inprocess.cpp:101-112 order).
__global__ void ordered_sum_kernel(const double* __restrict__ parts, int p, size_t count, size_t stride,
                                   double* __restrict__ out) {
    for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double acc = parts[e];
        for (int r = 1; r < p; ++r) acc += parts[static_cast<size_t>(r) * stride + e];
        out[e] = acc;
    }
}


}  // namespace

// ---------------------------------------------------------------------------
// Host planning.

std::vector<TileInfo> plan_tiles_uncached(int K) {
    const int nb = (K + BT - 1) / BT;
    std::vector<TileInfo> out;
    for (int I = 0; I < nb; ++I) {
        for (int J = I; J < nb; ++J) {
            TileInfo ti{};
            ti.I = I;
            ti.J = J;
            struct Entry {
                int wm, wn, cost;
                uint32_t mask;
            };
            std::vector<Entry> entries;
            for (int wm = 0; wm < 4; ++wm) {
                for (int wn = 0; wn < 4; ++wn) {
                    uint32_t mask = 0;
                    for (int mi = 0; mi < 4; ++mi) {
                        for (int ni = 0; ni < 4; ++ni) {
                            const int rmin = I * BT + wm * 32 + (mi >> 1) * 16 + (mi & 1);
                            const int cmin = J * BT + wn * 32 + (ni >> 1) * 16 + (ni & 1);
                            bool need = rmin < K && cmin < K;
                            if (I == J) need = need && rmin <= cmin + 14;
                            // the (odd rows, even columns) tile of a diagonal 16-block:
                            // the reduction takes it from the (even, odd) tile's transpose
                            if (I == J && wm == wn && (mi >> 1) == (ni >> 1) && (mi & 1) == 1 && (ni & 1) == 0)
                                need = false;
                            if (need) mask |= 1u << (mi * 4 + ni);
                        }
                    }
                    if (mask) entries.push_back({wm, wn, __builtin_popcount(mask), mask});
                }
            }
            // Diagonal and edge tiles leave warps idle (10 or fewer of 16 active),
            // and 2-3 warps per SM sub-partition hide the fragment-load latency
            // poorly: cut the largest warp tiles (≥ 8 mma) into column halves
            // (mma columns {0,1} / {2,3}; rows {0,1} / {2,3} when no column cut
            // applies) until every consumer warp has work. Each half is its own
            // warp slot; the reduction scatters per mma, so halves need nothing else.
            while (entries.size() < static_cast<size_t>(kConsumerWarps)) {
                int best = -1;
                for (int pass = 0; pass < 2 && best < 0; ++pass) {
                    const uint32_t lo = pass == 0 ? 0x3333u : 0x00FFu, hi = pass == 0 ? 0xCCCCu : 0xFF00u;
                    for (size_t k = 0; k < entries.size(); ++k) {
                        const uint32_t m = entries[k].mask;
                        if (entries[k].cost >= 8 && (m & lo) && (m & hi) &&
                            (best < 0 || entries[k].cost > entries[best].cost)) {
                            best = static_cast<int>(k);
                        }
                    }
                    if (best >= 0) {
                        const Entry e = entries[best];
                        entries[best] = {e.wm, e.wn, __builtin_popcount(e.mask & lo), e.mask & lo};
                        entries.push_back({e.wm, e.wn, __builtin_popcount(e.mask & hi), e.mask & hi});
                    }
                }
                if (best < 0) break;
            }
            // Balance the warp tiles over the 4 SM sub-partitions (warp w runs
            // on SMSP w % 4, at most 4 each): exact min-max assignment by a
            // pruned search (≤ 16 tiles of a few distinct costs), which beats
            // LPT on diagonal tiles (6 × 16 + 4 × 12 mma: LPT max 40, optimum 36).
            std::stable_sort(entries.begin(), entries.end(),
                             [](const Entry& a, const Entry& b) { return a.cost > b.cost; });
            const int n = static_cast<int>(entries.size());
            std::vector<int> cur(n, 0), best_assign(n, 0);
            int load[4] = {0, 0, 0, 0}, used[4] = {0, 0, 0, 0};
            int best_max = 1 << 30;
            int total = 0;
            for (const Entry& e : entries) total += e.cost;
            const int bound = (total + 3) / 4;  // no assignment beats an even split
            {  // LPT start (at most 4 per SMSP): the search only has to beat it
                int l[4] = {0, 0, 0, 0}, u[4] = {0, 0, 0, 0};
                for (int k = 0; k < n; ++k) {
                    int c = -1;
                    for (int q = 0; q < 4; ++q)
                        if (u[q] < 4 && (c < 0 || l[q] < l[c])) c = q;
                    l[c] += entries[k].cost;
                    ++u[c];
                    best_assign[k] = c;
                }
                best_max = std::max(std::max(l[0], l[1]), std::max(l[2], l[3]));
            }
            std::function<void(int, int)> dfs = [&](int k, int cur_max) {
                if (cur_max >= best_max || best_max <= bound) return;
                if (k == n) {
                    best_max = cur_max;
                    best_assign = cur;
                    return;
                }
                for (int c = 0; c < 4; ++c) {
                    if (used[c] >= 4) continue;
                    bool seen = false;  // SMSPs in the same state are interchangeable
                    for (int c2 = 0; c2 < c; ++c2) seen |= used[c2] < 4 && load[c2] == load[c] && used[c2] == used[c];
                    if (seen) continue;
                    load[c] += entries[k].cost;
                    ++used[c];
                    cur[k] = c;
                    dfs(k + 1, std::max(cur_max, load[c]));
                    load[c] -= entries[k].cost;
                    --used[c];
                }
            };
            dfs(0, 0);
            int slot[4] = {0, 0, 0, 0};
            for (int k = 0; k < n; ++k) {
                const Entry& e = entries[k];
                const int q = best_assign[k];
                const int w = q + 4 * slot[q]++;
                ti.warp[w] = static_cast<uint32_t>(e.wm) | (static_cast<uint32_t>(e.wn) << 2) |
                             (static_cast<uint32_t>(I == J) << 4) | (e.mask << 16);
            }
            out.push_back(ti);
        }
    }
    return out;
}

// The tile table depends on K only: planned once per K per process (the
// streamed passes re-plan every chunk).
std::vector<TileInfo> plan_tiles(int K) {
    static std::mutex mu;
    static std::map<int, std::vector<TileInfo>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(K);
    if (it == cache.end()) it = cache.emplace(K, plan_tiles_uncached(K)).first;
    return it->second;
}

Plan make_plan(long long n_rows, int K, int num_sms, size_t workspace_cap_bytes) {
    Plan p;
    p.K = K;
    p.n_rows = n_rows;
    p.n_tiles = static_cast<int>(plan_tiles(K).size());
    // Enough items for load balance, and chunks short enough (kTargetChunkRows)
    // that the CTAs working on one split stay within an L2-resident window of
    // rows (measured at C2 with 40-row stages: 8K-row chunks re-read Q 2.5x
    // from HBM, 4K-row 1.2x; the extra split partials cost ~0.1 ms of reduce).
    const long long target_items = static_cast<long long>(num_sms) * kItemsPerCta;
    long long S = (target_items + p.n_tiles - 1) / p.n_tiles;
    S = std::max<long long>(S, (n_rows + kTargetChunkRows - 1) / kTargetChunkRows);
    // Keep the fixed-order reduction cheap relative to the contraction.
    S = std::min<long long>(S, std::max<long long>(1, n_rows / kMinRowsPerSplit));
    const long long per_item = static_cast<long long>(kItemDoubles) * sizeof(double);
    S = std::min<long long>(
        S, std::max<long long>(1, static_cast<long long>(workspace_cap_bytes) / (per_item * p.n_tiles)));
    S = std::max<long long>(1, S);
    long long chunk = (n_rows + S - 1) / S;
    if (const char* env = std::getenv("DOPINF_B200_GRAM_CHUNK_ROWS")) {  // tuning knob
        const long long c = std::atoll(env);
        if (c > 0) chunk = c;
    }
    chunk = std::max<long long>(BK, (chunk + BK - 1) / BK * BK);
    S = std::max<long long>(1, (n_rows + chunk - 1) / chunk);
    // Guided tail: the last T big splits (about two waves of items) become 4T
    // quarter-size splits so the final items finish close together.
    const long long T = (2LL * num_sms + p.n_tiles - 1) / p.n_tiles;
    long long big = S, small = chunk, n_small = 0;
    if (S > 2 * T && chunk >= 4 * BK) {
        big = S - T;
        const long long rest = n_rows - big * chunk;
        small = std::max<long long>(BK, ((rest + 4 * T - 1) / (4 * T) + BK - 1) / BK * BK);
        n_small = (rest + small - 1) / small;
    }
    p.n_splits = static_cast<int>(big + n_small);
    p.chunk_rows = static_cast<int>(chunk);
    p.big_splits = static_cast<int>(big);
    p.small_rows = static_cast<int>(small);
    p.n_items = p.n_splits * p.n_tiles;
    p.grid = std::min(num_sms, p.n_items);
    p.workspace_doubles = static_cast<size_t>(p.n_items) * kItemDoubles;
    return p;
}

cudaError_t make_tensor_map(CUtensorMap* map, const double* q, long long n_rows, int K, size_t ld) {
    auto fn = tensor_map_encoder();
    if (!fn) return cudaErrorNotSupported;
    if (n_rows >= (1LL << 31)) return cudaErrorInvalidValue;  // TMA row coordinates are int32
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(n_rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * sizeof(double))};
    const cuuint32_t box[2] = {16u, static_cast<cuuint32_t>(BK)};  // 128 B rows → 128B swizzle
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(q), dims,
                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

size_t smem_bytes() { return sizeof(Smem) + 1024; }

cudaError_t launch_gram(const Plan& plan, const CUtensorMap& map, const TileInfo* d_tiles,
                        double* work, int* counters, cudaStream_t stream, bool accumulate) {
    const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void*>(gram_dmma_kernel),
                                             static_cast<int>(smem_bytes()));
    if (e != cudaSuccess) return e;
    gram_dmma_kernel<<<plan.grid, THREADS, smem_bytes(), stream>>>(
        map, d_tiles, plan.n_tiles, plan.n_items, plan.n_rows, plan.K, plan.chunk_rows, plan.big_splits,
        plan.small_rows,
        work, counters, accumulate ? 1 : 0, plan.streamed ? 1 : 0);
    note_launch();
    return cudaGetLastError();
}

Plan make_stream_plan(long long chunk_rows, int K, int num_sms, long long split_rows) {
    Plan p;
    p.K = K;
    p.n_rows = chunk_rows;
    p.n_tiles = static_cast<int>(plan_tiles(K).size());
    const long long split = std::max<long long>(BK, (split_rows + BK - 1) / BK * BK);
    p.chunk_rows = static_cast<int>(split);
    p.n_splits = static_cast<int>(std::max<long long>(1, (chunk_rows + split - 1) / split));
    p.big_splits = p.n_splits;
    p.small_rows = p.chunk_rows;
    p.streamed = true;
    p.n_items = p.n_splits * p.n_tiles;
    p.grid = std::min(num_sms, p.n_items);
    p.workspace_doubles = static_cast<size_t>(p.n_items) * kItemDoubles;
    return p;
}

cudaError_t launch_combine_vars(const double* gv, int n_vars, size_t count, const double* scales,
                                double* out, cudaStream_t stream) {
    const int grid = static_cast<int>(std::min<size_t>((count + 255) / 256, 148 * 16));
    combine_vars_kernel<<<std::max(grid, 1), 256, 0, stream>>>(gv, n_vars, count, scales, out);
    note_launch();
    return cudaGetLastError();
}

int reduce_groups(const Plan& plan, int num_sms) {
    const long long blocks = static_cast<long long>(plan.n_tiles) * CONSUMERS;
    const long long want = 4LL * num_sms;
    if (blocks >= want || plan.n_splits < 16) return 1;
    const long long g = std::max<long long>(1, std::min<long long>((want + blocks - 1) / blocks, plan.n_splits / 8));
    // no empty group: ceil(S / ceil(S / g)) groups of ceil(S / g) splits
    const long long per = (plan.n_splits + g - 1) / g;
    return static_cast<int>((plan.n_splits + per - 1) / per);
}

size_t reduce_scratch_doubles(const Plan& plan, int groups) {
    return groups > 1 ? static_cast<size_t>(groups) * plan.n_tiles * kItemDoubles : 0;
}

cudaError_t launch_reduce(const Plan& plan, const TileInfo* d_tiles, const double* work,
                          double* packed, cudaStream_t stream, int groups, double* scratch) {
    if (groups > 1 && scratch) {
        gram_reduce_kernel<<<groups * plan.n_tiles * CONSUMERS, 512, 0, stream>>>(
            d_tiles, plan.n_tiles, plan.n_splits, plan.K, work, packed, groups, scratch);
        note_launch();
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        gram_reduce_kernel<<<plan.n_tiles * CONSUMERS, 512, 0, stream>>>(d_tiles, plan.n_tiles, groups, plan.K,
                                                                          scratch, packed, 1, nullptr);
    } else {
        gram_reduce_kernel<<<plan.n_tiles * CONSUMERS, 512, 0, stream>>>(d_tiles, plan.n_tiles, plan.n_splits,
                                                                          plan.K, work, packed, 1, nullptr);
    }
    note_launch();
    return cudaGetLastError();
}

CoverageReport coverage(int K) {
    CoverageReport r;
    const std::vector<TileInfo> tiles = plan_tiles(K);
    const size_t count = packed_count(K);
    std::vector<unsigned char> hits(count, 0);
    for (const TileInfo& ti : tiles) {
        for (int w = 0; w < kConsumerWarps; ++w) {
            int wm, wn;
            bool diag;
            uint32_t mask;
            decode(ti.warp[w], wm, wn, diag, mask);
            for (int mma = 0; mma < 16; ++mma) {
                if (!((mask >> mma) & 1u)) continue;
                ++r.mma_tiles;
                for (int lane = 0; lane < kWarp; ++lane) {
                    for (int c = 0; c < 2; ++c) {
                        const long long idx = scatter_index(ti.I, ti.J, wm, wn, diag, mma, lane, c, K);
                        if (idx < 0) continue;
                        if (hits[idx] == 1) ++r.duplicates;
                        if (hits[idx] < 2) ++hits[idx];
                    }
                }
            }
        }
    }
    for (unsigned char h : hits) r.covered += h ? 1 : 0;
    r.entries = static_cast<long long>(count);
    return r;
}

cudaError_t launch_unpack(const double* packed, int K, double* d, cudaStream_t stream) {
    const size_t total = static_cast<size_t>(K) * K;
    const int grid = static_cast<int>(std::min<size_t>((total + 255) / 256, 148 * 16));
    unpack_kernel<<<std::max(grid, 1), 256, 0, stream>>>(packed, K, d);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_ordered_sum(const double* parts, int p, size_t count, size_t stride, double* out,
                               cudaStream_t stream) {
    const int grid = static_cast<int>(std::min<size_t>((count + 255) / 256, 148 * 16));
    ordered_sum_kernel<<<std::max(grid, 1), 256, 0, stream>>>(parts, p, count, stride, out);
    note_launch();
    return cudaGetLastError();
}

}  // namespace gram
}  // namespace dopinf_b200
