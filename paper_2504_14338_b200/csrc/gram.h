// gram.h — host interface of the DMMA Gram kernels (gram.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

namespace dopinf_b200 {
namespace gram {

constexpr int kTileEdge = 128;       // columns of Q per block (CTA output tile edge)
#ifndef DOPINF_GRAM_ROWS_PER_STAGE  // (build-time tuning knob)
#define DOPINF_GRAM_ROWS_PER_STAGE 48
#endif
// rows of Q per TMA stage (round 1: 16→48.1 ms, 32→47.0, 40→46.6, 56→48.0 at C2;
// round 2, two stages unless noted: 24×4→43.58, 32×3→43.01, 40→42.75, 48→42.64,
// 56→43.41 — profiles/r02_gram_stage_variants.txt)
constexpr int kRowsPerStage = DOPINF_GRAM_ROWS_PER_STAGE;
constexpr int kConsumerWarps = 16;   // 4×4 grid of 32×32 warp tiles
constexpr int kWarpFragDoubles = 16 * 32 * 2;                   // 16 mma × 32 lanes × 2
constexpr int kItemDoubles = kConsumerWarps * kWarpFragDoubles;  // 16384 (128 KiB)
constexpr int kItemsPerCta = 16;     // queue granularity target (tail vs workspace)
constexpr long long kMinRowsPerSplit = 768;
constexpr long long kTargetChunkRows = 4096;  // L2 window of rows shared by a split's CTAs (C2: 8K rows re-read Q 2.5x from HBM with 40-row stages, 4K rows 1.2x)
constexpr size_t kWorkspaceCapBytes = size_t(2) << 30;

struct TileInfo {
    int I, J;
    uint32_t warp[kConsumerWarps];  // wm | wn<<2 | diag<<4 | mma-mask<<16
};

struct Plan {
    int K = 0;
    long long n_rows = 0;
    int n_tiles = 0;
    int n_splits = 0;
    int chunk_rows = 0;   // rows of the first big_splits splits
    int big_splits = 0;
    int small_rows = 0;   // rows of the remaining (tail) splits
    int n_items = 0;
    int grid = 0;
    bool streamed = false;  // make_stream_plan: the split slots are re-read by the next chunk's launch
    size_t workspace_doubles = 0;
};

std::vector<TileInfo> plan_tiles(int K);
Plan make_plan(long long n_rows, int K, int num_sms, size_t workspace_cap_bytes);
cudaError_t make_tensor_map(CUtensorMap* map, const double* q, long long n_rows, int K, size_t ld);
size_t smem_bytes();
cudaError_t launch_gram(const Plan& plan, const CUtensorMap& map, const TileInfo* d_tiles,
                        double* work, int* counters, cudaStream_t stream, bool accumulate = false);
// Plan for one streamed chunk of `chunk_rows` rows cut into splits of
// `split_rows`; its items accumulate into the same split slots chunk after chunk.
Plan make_stream_plan(long long chunk_rows, int K, int num_sms, long long split_rows);
// D = Σ_v (gv[v] / scales[v]) / scales[v] (scales == nullptr: Σ_v gv[v]), variables in order.
cudaError_t launch_combine_vars(const double* gv, int n_vars, size_t count, const double* scales,
                                double* out, cudaStream_t stream);
// Split groups for the fixed-order reduction (1 = one pass over all splits;
// more when the tiles alone would leave most SMs idle) and the scratch they need.
int reduce_groups(const Plan& plan, int num_sms);
size_t reduce_scratch_doubles(const Plan& plan, int groups);
cudaError_t launch_reduce(const Plan& plan, const TileInfo* d_tiles, const double* work,
                          double* packed, cudaStream_t stream, int groups = 1, double* scratch = nullptr);
cudaError_t launch_unpack(const double* packed, int K, double* d, cudaStream_t stream);
// Host-side check of the tile plan for K: how many packed upper-triangle
// entries the reduction writes (covered, of entries) and how many it would
// write twice; mma_tiles = 8×8 DMMA tiles executed per 4-row k-step over all
// output tiles (the executed work, for the useful-work ratio).
struct CoverageReport {
    long long entries = 0, covered = 0, duplicates = 0, mma_tiles = 0;
};
CoverageReport coverage(int K);
// out[e] = parts[0][e] + parts[1][e] + ... (rank r's part at parts + r*stride).
cudaError_t launch_ordered_sum(const double* parts, int p, size_t count, size_t stride, double* out,
                               cudaStream_t stream);

// Reference-order mode (gram_ref.cu): every upper-triangle entry is the FMA
// chain of linalg::gram (linalg.cpp:50-58) over the rows in order, written to
// the packed triangle (accumulate: the chain continues from packed's values,
// for row ranges processed in order). q 16-byte aligned, ld even.
cudaError_t launch_gram_reference_order(const double* q, size_t ld, long long rows, int K, double* packed,
                                        bool accumulate, cudaStream_t stream);

inline size_t packed_count(int K) { return static_cast<size_t>(K) * (K + 1) / 2; }

}  // namespace gram
}  // namespace dopinf_b200
