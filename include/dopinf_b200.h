/*
 * dopinf_b200.h — C ABI of the B200-native dOpInf snapshot pass.
 *
 * Drop-in boundary for the reference's Steps II–III and the Φ_r/projection
 * products (paths relative to /root/reference/proj). Every entry point is
 * synchronous at the boundary (the reference has value semantics), takes plain
 * pointers and sizes, never throws, and returns a dopinf_b200_status whose
 * values map one-to-one onto the reference exception classes
 * (include/dopinf/errors.hpp:9-73); the message is kept per context
 * (dopinf_b200_last_error). Host matrices are row-major fp64 with an explicit
 * leading dimension, as dopinf::Matrix (include/dopinf/matrix.hpp:13-53).
 *
 * Replaces                                               with
 *   comm::Comm rank/size/allreduce/barrier (comm.hpp:13-31)  dopinf_b200_ctx_* + allreduce/barrier
 *   data::partition_rows (data.hpp:47, data.cpp:86-103)      dopinf_b200_partition_rows
 *   data::LocalBlock values (data.hpp:38-42)                 dopinf_b200_block (device resident)
 *   transform::center_in_place (transform.hpp:27)            dopinf_b200_center
 *   transform::compute_global_scales (transform.hpp:32-34)   dopinf_b200_global_scales
 *   transform::scale_in_place (transform.hpp:37)             dopinf_b200_scale
 *   pod::local_gram (pod.hpp:28)                             dopinf_b200_local_gram
 *   pod::global_gram (pod.hpp:31)                            dopinf_b200_global_gram
 *   pod::project (pod.hpp:49)                                dopinf_b200_project / _project_host
 *   postprocess::reconstruct_field's Φ_r = Q·T_r (postprocess.cpp:66)
 *                                                            dopinf_b200_basis
 *   postprocess::basis_rows (postprocess.hpp:25-26)          dopinf_b200_basis_rows
 *   data::read_header (data.hpp:52, data.cpp:133-162)        dopinf_b200_snp1_header
 *   data::read_block (data.hpp:54, data.cpp:164-202)         dopinf_b200_block_read
 *   pipeline::run_rank read + Steps II-III (pipeline.cpp:254-280)
 *                                                            dopinf_b200_snapshot_pass_file
 *   rom_search::grid_search (rom_search.cpp:185-262)        dopinf_b200_grid_search
 *   rom_search::integrate (rom_search.cpp:62-87)            dopinf_b200_rom_integrate
 *   postprocess::reconstruct_probes (postprocess.cpp:36-61)  dopinf_b200_reconstruct_probes
 *   postprocess::reconstruct_field (postprocess.cpp:63-70)   dopinf_b200_reconstruct_field
 *   Step V field_rank<r>.snp1 output (pipeline.cpp:330-350) dopinf_b200_write_field
 *
 * The eigensolve (pod::eig_sym_desc), rank selection, reduced_map, the OpInf
 * solve and the ROM search stay on the reference code path: the host D
 * returned by dopinf_b200_global_gram is the reference's Matrix D, and the
 * T_r it produces is handed back to dopinf_b200_project / _basis.
 */
#ifndef DOPINF_B200_H
#define DOPINF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DOPINF_B200_ABI_VERSION 2
#define DOPINF_B200_UNIQUE_ID_BYTES 128

typedef enum dopinf_b200_status {
    DOPINF_B200_OK = 0,
    DOPINF_B200_ERR_INVALID_ARGUMENT = 1,   /* InvalidArgumentError   (errors.hpp:70-73) */
    DOPINF_B200_ERR_PARTITION = 2,          /* PartitionError         (errors.hpp:21-24) */
    DOPINF_B200_ERR_COLLECTIVE = 3,         /* CollectiveError        (errors.hpp:28-31) */
    DOPINF_B200_ERR_DEGENERATE_VARIABLE = 4,/* DegenerateVariableError(errors.hpp:34-37) */
    DOPINF_B200_ERR_DEVICE = 5,             /* CUDA / NCCL failure (surfaced as dopinf::Error) */
    DOPINF_B200_ERR_OUT_OF_MEMORY = 6,      /* device allocation failure (dopinf::Error)      */
    DOPINF_B200_ERR_NOT_PSD = 7,            /* NotPsdError            (errors.hpp:40-43) */
    DOPINF_B200_ERR_RANK_DEFICIENCY = 8,    /* RankDeficiencyError    (errors.hpp:46-49) */
    DOPINF_B200_ERR_SOLVE = 9,              /* SolveError             (errors.hpp:52-55) */
    DOPINF_B200_ERR_DATA_FORMAT = 10,       /* DataFormatError        (errors.hpp:15-18) */
    DOPINF_B200_ERR_NO_ADMISSIBLE_PAIR = 11 /* NoAdmissiblePairError  (errors.hpp:57-60) */
} dopinf_b200_status;

/* Collective ops, same order as comm::ReduceOp (comm.hpp:9). */
typedef enum dopinf_b200_reduce_op {
    DOPINF_B200_SUM = 0,
    DOPINF_B200_MAX = 1,
    DOPINF_B200_MIN = 2
} dopinf_b200_reduce_op;

/* How the K×K Gram partials of the ranks are combined (pod.cpp:15-18).
 * NCCL (default): one ncclAllReduce(Sum) of the packed upper triangle over
 * NVLink — the north star's single all-reduce, and the reference's MPI
 * backend (comm_mpi.cpp:44-47, MPI_Allreduce); identical on every rank.
 * ORDERED: ncclAllGather of the packed triangles, then a device sum in
 * ascending rank order — the reduction order of the reference's in-process
 * backend (comm_inprocess.cpp:101-112), bitwise reproducible for a fixed rank
 * count regardless of NCCL's algorithm choice. */
typedef enum dopinf_b200_gram_reduce {
    DOPINF_B200_GRAM_REDUCE_ORDERED = 0,
    DOPINF_B200_GRAM_REDUCE_NCCL = 1
} dopinf_b200_gram_reduce;

/* Summation order of the local Gram (dopinf_b200_set_gram_order).
 * TENSOR (default): the DMMA upper-triangle kernel with split-n partials reduced
 * in a fixed order — bitwise reproducible, within ~1e-15 of the reference.
 * REFERENCE: linalg::gram's own order (linalg.cpp:50-58; every entry one FMA
 * chain over the rows, ascending), on the DFMA pipe — bit-identical to the
 * reference's D; selecting it also selects the ORDERED cross-rank sum (the
 * in-process backend's order), so D is the reference's at any rank count and
 * everything downstream of it on the reference path (eig, reduced map, Q̂,
 * the OpInf solve and ROM) is too. Streamed passes support it for resident
 * blocks (host / file sources), not for dopinf_b200_stream_pass_synth. */
typedef enum dopinf_b200_gram_order {
    DOPINF_B200_GRAM_ORDER_TENSOR = 0,
    DOPINF_B200_GRAM_ORDER_REFERENCE = 1
} dopinf_b200_gram_order;

/* Device-timed stages recorded per context (CUDA events on its stream). */
typedef enum dopinf_b200_stage {
    DOPINF_B200_STAGE_UPLOAD = 0,
    DOPINF_B200_STAGE_STATS = 1,      /* center: mean + row max-abs pass        */
    DOPINF_B200_STAGE_SCALES = 2,     /* MAX all-reduce of per-variable scales  */
    DOPINF_B200_STAGE_APPLY = 3,      /* (x - mean) / s pass                    */
    DOPINF_B200_STAGE_GRAM = 4,       /* DMMA upper-triangle Gram kernel        */
    DOPINF_B200_STAGE_GRAM_REDUCE = 5,/* split-n fix-up (fixed order)           */
    DOPINF_B200_STAGE_ALLREDUCE = 6,  /* cross-rank Gram reduction              */
    DOPINF_B200_STAGE_UNPACK = 7,     /* packed triangle -> symmetric K×K       */
    DOPINF_B200_STAGE_PROJECT = 8,    /* Q̂ = T_rᵀ D                             */
    DOPINF_B200_STAGE_BASIS = 9,      /* Φ_r = Q T_r                            */
    DOPINF_B200_STAGE_DOWNLOAD = 10,
    DOPINF_B200_STAGE_STREAM = 11,    /* whole streamed pass (first H2D -> D ready) */
    DOPINF_B200_STAGE_STREAM_GRAM = 12,/* sum of the streamed pass's Gram launches */
    DOPINF_B200_STAGE_FIELD = 13,     /* Φ_r·Q̃ᵀ + inverse transform (reconstruct_field) */
    DOPINF_B200_STAGE_COUNT = 14
} dopinf_b200_stage;

/* dopinf_b200_ctx_create_ex flags. */
#define DOPINF_B200_CTX_NCCL 1u /* an NCCL communicator even at size 1: the collective
                                 * code paths run (and are testable) on one GPU */

/* dopinf_b200_debug_inject faults (test support). */
#define DOPINF_B200_INJECT_STALL 1 /* the next collective is followed on the stream by a
                                    * device stall the library releases only when it
                                    * aborts: drives the timeout → abort → poison path */
#define DOPINF_B200_INJECT_OOB_STORE 2 /* one device store just past a library buffer, now
                                        * (guarded allocations only): the positive control
                                        * of dopinf_b200_debug_guard_violations */

typedef struct dopinf_b200_ctx dopinf_b200_ctx;
typedef struct dopinf_b200_block dopinf_b200_block;

/* ---- library ---------------------------------------------------------- */
int dopinf_b200_abi_version(void);
const char* dopinf_b200_status_string(int status);
/* Number of kernel launches this process has issued through the library. */
uint64_t dopinf_b200_kernel_launches(void);

/* ---- per-rank context (replaces the comm::Comm a rank runs against) ----- */
/* Fill `id` (DOPINF_B200_UNIQUE_ID_BYTES) with an ncclUniqueId; rank 0 calls
 * this and distributes the bytes (any transport) to the other ranks. */
int dopinf_b200_get_unique_id(unsigned char* id);
/* One context per rank: binds `device`, creates a stream and, when size > 1,
 * an NCCL communicator from `id` (ignored when size == 1). The communicator
 * is initialised non-blocking and waited for with the collective deadline
 * (env DOPINF_B200_COLLECTIVE_TIMEOUT seconds, default 60): a peer that never
 * joins gives COLLECTIVE ("collective timed out waiting for peer ranks"). */
int dopinf_b200_ctx_create(int device, int rank, int size, const unsigned char* id,
                           dopinf_b200_ctx** out);
/* A context on the caller's NCCL communicator and CUDA stream (plain
 * pointers: ncclComm_t and cudaStream_t; either may be NULL — no
 * communicator means one rank, no stream means the context makes its own).
 * Rank and size come from the communicator. Neither is destroyed with the
 * context; the caller keeps them alive until dopinf_b200_ctx_destroy. */
int dopinf_b200_ctx_create_external(int device, void* nccl_comm, void* stream, dopinf_b200_ctx** out);
/* ctx_create with flags (DOPINF_B200_CTX_NCCL: create the communicator from
 * `id` even when size == 1). */
int dopinf_b200_ctx_create_ex(int device, int rank, int size, const unsigned char* id, unsigned flags,
                              dopinf_b200_ctx** out);
void dopinf_b200_ctx_destroy(dopinf_b200_ctx* ctx);
int dopinf_b200_ctx_rank(const dopinf_b200_ctx* ctx);
int dopinf_b200_ctx_size(const dopinf_b200_ctx* ctx);
const char* dopinf_b200_last_error(const dopinf_b200_ctx* ctx);
int dopinf_b200_set_gram_reduce(dopinf_b200_ctx* ctx, int mode);
/* DOPINF_B200_GRAM_ORDER_* (REFERENCE also sets the ORDERED reduction). */
int dopinf_b200_set_gram_order(dopinf_b200_ctx* ctx, int order);
/* Comm::allreduce / barrier (comm.hpp:20-30) on a HOST span, over NCCL;
 * SUM in ascending rank order (all-gather + ordered device sum). */
int dopinf_b200_allreduce(dopinf_b200_ctx* ctx, double* data, size_t count, int op);
int dopinf_b200_barrier(dopinf_b200_ctx* ctx);
/* Group failure semantics (comm_inprocess.cpp:41-87). Waiting for a queued
 * collective is bounded by `seconds` (default 60, the reference's kTimeout);
 * an NCCL asynchronous error or the deadline aborts the communicator
 * (ncclCommAbort) and poisons the context: that call and every later
 * collective fail with COLLECTIVE ("collective timed out waiting for peer
 * ranks"). A rank-local failure inside a fused call (snapshot_pass, the grid
 * search) is carried to the peers in the collective that follows, which then
 * fail with COLLECTIVE "rank r aborted" while the failing rank reports its own
 * error. */
int dopinf_b200_set_collective_timeout(dopinf_b200_ctx* ctx, double seconds);
/* verify_uniform (comm_inprocess.cpp:139-151): when enabled, every collective
 * is preceded by an all-gather of (sequence, count, op) and all ranks fail
 * with the same COLLECTIVE verdict on a mismatch (debugging aid: one extra
 * small collective each). */
int dopinf_b200_set_collective_checks(dopinf_b200_ctx* ctx, int enabled);
/* 1 when a collective failure has poisoned the context. */
int dopinf_b200_ctx_poisoned(const dopinf_b200_ctx* ctx);
/* The agreement rule itself, host only: `table` holds p rows of
 * (sequence, count, tag) as all-gathered; COLLECTIVE with the reference's
 * message ("<what>: rank R passed count X, rank S passed count Y") written to
 * msg when rank `rank` sees a disagreement. */
int dopinf_b200_check_uniform(const long long* table, int p, int rank, const char* what, char* msg,
                              size_t msg_cap);
/* Guarded allocations (debug aid in place of compute-sanitizer's memcheck):
 * with the environment variable DOPINF_B200_GUARD_BYTES=G, every device buffer
 * the library allocates is bracketed by G bytes of a known pattern. Returns
 * the number of buffers whose guards were found overwritten (freed ones
 * included), or -1 when guards are off. */
long long dopinf_b200_debug_guard_violations(void);
/* Fault injection for tests (DOPINF_B200_INJECT_*; 0 clears). */
int dopinf_b200_debug_inject(dopinf_b200_ctx* ctx, int what);
/* Host-only check of the Gram tile plan for K (no GPU needed): the number of
 * packed upper-triangle entries (K(K+1)/2), how many of them the split-n
 * reduction writes, how many it would write more than once, and the 8x8 DMMA
 * tiles executed per 4-row k-step over all output tiles. */
int dopinf_b200_debug_gram_coverage(int K, long long* entries, long long* covered, long long* duplicates,
                                    long long* mma_tiles);
/* The combine step of the ORDERED reduction on the device: out = parts[0] +
 * parts[1] + ... + parts[p-1] element-wise, left to right (kernels::add in
 * ascending rank order, comm_inprocess.cpp:101-112). parts: host p x count. */
int dopinf_b200_ordered_sum(dopinf_b200_ctx* ctx, const double* parts, int p, size_t count, double* out);
/* Device milliseconds of `stage` in the most recent call that ran it. */
int dopinf_b200_stage_ms(const dopinf_b200_ctx* ctx, int stage, double* ms);
/* The context's CUDA stream (cudaStream_t), for callers that interoperate. */
void* dopinf_b200_ctx_stream(dopinf_b200_ctx* ctx);

/* ---- sharding (data.cpp:86-103) --------------------------------------- */
/* floor(nx/p) rows per rank, remainder on the last rank; begin/end have p
 * entries. PARTITION unless 1 <= p <= nx. */
int dopinf_b200_partition_rows(size_t nx, int p, size_t* begin, size_t* end);

/* ---- device-resident LocalBlock (data.hpp:38-42) ----------------------- */
/* (n_vars * nx_i) x nt fp64; block row j*nx_i + k is variable j at global
 * spatial index row_begin + k. Device pitch is nt rounded up to even. */
int dopinf_b200_block_create(dopinf_b200_ctx* ctx, size_t n_vars, size_t nx_i, size_t row_begin,
                             size_t nt, dopinf_b200_block** out);
void dopinf_b200_block_destroy(dopinf_b200_block* block);
int dopinf_b200_block_upload(dopinf_b200_block* block, const double* host, size_t host_ld);
/* Materialises any pending transform, then copies the values to the host. */
int dopinf_b200_block_download(dopinf_b200_block* block, double* host, size_t host_ld);
/* Rows [row0, row0 + nrows) of the (materialised) block to the host, pitch
 * host_ld: a block larger than host memory is read out in slices. */
int dopinf_b200_block_download_rows(dopinf_b200_block* block, size_t row0, size_t nrows, double* host,
                                    size_t host_ld);
/* {n_vars, nx_i, row_begin, nt} of a block (e.g. one dopinf_b200_block_read made). */
int dopinf_b200_block_shape(const dopinf_b200_block* block, size_t* dims);
/* Device pointer and pitch (elements) of the block values. */
int dopinf_b200_block_device(dopinf_b200_block* block, double** values, size_t* ld);
/* Seeded synthetic snapshots on the device (BASELINE.json configs 1, 2, 4):
 * Q[i,k] = amp_v * Σ_j sin(jπx_i + θ_j) e^{-γ_j t_k} cos(ω_j t_k + φ_j)
 *          + noise * N(0,1),  t_k = k*dt, x_i = seeded U[0,1) per global point.
 * Mode draws (θ, ω, γ, φ) are seeded per variable; amp_v = amps[v] (NULL: 1).
 * The generator is plumbing for the bench/tests, not part of the pass. */
int dopinf_b200_block_synth_oscillator(dopinf_b200_block* block, uint64_t seed, int n_modes,
                                       double dt, double noise, const double* amps);
/* The same generator for variables var0 .. var0 + n_vars - 1 of a larger
 * dataset (amps: n_vars entries for those variables, or NULL): the bytes one
 * variable's rows have inside a streamed pass over the whole dataset. */
int dopinf_b200_block_synth_oscillator_vars(dopinf_b200_block* block, int var0, uint64_t seed, int n_modes,
                                            double dt, double noise, const double* amps);
/* Seeded i.i.d. N(0,1) plus amplitude * (rank-`rank` low-rank component)
 * (BASELINE.json config 3). */
int dopinf_b200_block_synth_lowrank(dopinf_b200_block* block, uint64_t seed, int rank,
                                    double amplitude);

/* ---- Step II transform (transform.cpp) --------------------------------- */
/* center_in_place (transform.cpp:10-20): writes the per-row temporal means
 * (rows = n_vars*nx_i; host, may be NULL). The subtraction is fused into the
 * next pass over the block (apply or download); results are those of the
 * reference's separate passes. */
int dopinf_b200_center(dopinf_b200_block* block, double* means);
/* compute_global_scales (transform.cpp:22-41): per-variable max |centered q|,
 * MAX all-reduced over the ranks. DEGENERATE_VARIABLE when a scale is 0, with
 * *degenerate_var set to the first such variable. scales: host [n_vars]. */
int dopinf_b200_global_scales(dopinf_b200_block* block, double* scales, size_t* degenerate_var);
/* The rank-local half of compute_global_scales (transform.cpp:28-31: the
 * per-variable kernels::max_abs over this block's centered rows) with no
 * collective and no zero check: for callers that reduce over their own
 * comm::Comm (transform.cpp:32) — e.g. several in-process ranks sharing one
 * GPU, each with a size-1 context. maxabs: host [n_vars]. */
int dopinf_b200_local_maxabs(dopinf_b200_block* block, double* maxabs);
/* scale_in_place (transform.cpp:43-49): q /= scales[var] (IEEE division). */
int dopinf_b200_scale(dopinf_b200_block* block, const double* scales);

/* ---- Step III Gram / projection (pod.cpp) ------------------------------ */
/* local_gram (pod.cpp:11-13): D_i = Q_iᵀ Q_i, upper triangle on the FP64
 * tensor pipe, split-n partials reduced in fixed order; kept on the device
 * and, when d != NULL, written to the host as the full symmetric nt x nt. */
int dopinf_b200_local_gram(dopinf_b200_block* block, double* d);
/* global_gram (pod.cpp:15-18): the SUM over the ranks of the context's last
 * local Gram (its device copy; nt must be its size, else INVALID_ARGUMENT),
 * identical on every rank, optionally written to the host (d: nt x nt). Like
 * the reference's pure function it can be repeated: each call reduces the
 * same local partial. Fails after set_gram (no local partial). */
int dopinf_b200_global_gram(dopinf_b200_ctx* ctx, double* d, size_t nt);
/* project (pod.cpp:103-105): Q̂ = T_rᵀ D with the context's device D;
 * tr is host nt x r (NULL: the device T_r of dopinf_b200_reduced_map),
 * qhat host r x nt. */
int dopinf_b200_project(dopinf_b200_ctx* ctx, const double* tr, size_t nt, size_t r,
                        double* qhat);
/* §8(f) next-row 1 — the eigensolve on the device. eig_sym_desc
 * (pod.cpp:20-65): cuSOLVER dsyevd of the context's device D; eigenvalues
 * descending, negatives within −1e-10·λ1 clamped to 0 (NOT_PSD below that),
 * each eigenvector flipped so its largest-magnitude entry (lowest index on
 * ties) is positive. lambda: host [nt]; vectors: host nt x nt row-major,
 * column k ↔ lambda[k]; either may be NULL. */
int dopinf_b200_eig_sym_desc(dopinf_b200_ctx* ctx, double* lambda, double* vectors);
/* Make a host nt x nt symmetric D the context's device Gram (for
 * eig_sym_desc(const Matrix& d) callers that hold D on the host). */
int dopinf_b200_set_gram(dopinf_b200_ctx* ctx, const double* d, size_t nt);
/* reduced_map (pod.cpp:84-101): T_r = U_r · (1/√λ_k) from the context's
 * eigendecomposition, kept on the device (project / basis with tr == NULL use
 * it); RANK_DEFICIENCY when λ_r is 0. tr: host nt x r, may be NULL. */
int dopinf_b200_reduced_map(dopinf_b200_ctx* ctx, size_t r, double* tr);
/* project with a caller-provided host D (nt x nt). */
int dopinf_b200_project_host(dopinf_b200_ctx* ctx, const double* tr, const double* d, size_t nt,
                             size_t r, double* qhat);

/* ---- Step V products (postprocess.cpp) --------------------------------- */
/* Φ_r = Q T_r over the (transformed) block: rows x r. tr: host nt x r, or
 * NULL for the context's device T_r. phi (host) may be NULL to keep the
 * result on the device only (dopinf_b200_basis_device). */
int dopinf_b200_basis(dopinf_b200_block* block, const double* tr, size_t r, double* phi);
int dopinf_b200_basis_device(dopinf_b200_block* block, double** phi, size_t* ld);
/* basis_rows (postprocess.cpp:12-34): out[k] = Q[rows[k]] T_r. */
int dopinf_b200_basis_rows(dopinf_b200_block* block, const double* tr, size_t r,
                           const size_t* rows, size_t nsel, double* out);

/* ---- fused Steps II-III: one call per rank ------------------------------ */
/* center (+ global scales + scale when scaling != 0) + local + global Gram.
 * means [rows], scales [n_vars], d [nt x nt]: host, each may be NULL. */
int dopinf_b200_snapshot_pass(dopinf_b200_block* block, int scaling, double* means,
                              double* scales, double* d);
/* The same Steps II-III with the block's values arriving from HOST memory
 * (row-major, pitch host_ld): rows stream in chunks on a copy stream while the
 * compute stream centers each landed chunk and accumulates its Gram; scaling
 * is folded into the Gram (D = Σ_v G_v / s_v², G_v the Gram of variable v's
 * centered rows) so no pass waits for the global scales, and each variable is
 * scaled as soon as its MAX is final. The block ends resident and transformed
 * exactly as dopinf_b200_snapshot_pass leaves it (bit-identical values, means
 * and scales; D within the same tolerance). Host memory should be pinned for
 * the copies to overlap. On DegenerateVariableError, variables finished before
 * the degenerate one are left scaled. */
int dopinf_b200_snapshot_pass_host(dopinf_b200_block* block, const double* host, size_t host_ld,
                                   int scaling, double* means, double* scales, double* d);
/* Steps II-III for a block too large to hold (BASELINE config 4: 8 vars ×
 * 4,194,304 points × K=1500 is 403 GB per GPU): the rows are generated on the
 * device chunk by chunk (the seeded oscillator of
 * dopinf_b200_block_synth_oscillator, same bytes) into a two-slot ring and
 * streamed through stats, centering and the per-variable Gram; the block is
 * never resident, so only the means (rows), scales (n_vars) and D (nt x nt)
 * come back. Ranks pass their own (nx_i, row_begin). */
int dopinf_b200_stream_pass_synth(dopinf_b200_ctx* ctx, size_t n_vars, size_t nx_i, size_t row_begin,
                                  size_t nt, uint64_t seed, int n_modes, double dt, double noise,
                                  const double* amps, int scaling, double* means, double* scales,
                                  double* d);

/* ---- SNP1 snapshot files (data.hpp:11-15) --------------------------------- */
/* data::read_header (data.cpp:133-162): parse and validate the header of the
 * SNP1 file at `path` (magic, n_vars/nx/nt, names, payload size) with the
 * reference's checks and DataFormatError messages. dims receives
 * {n_vars, nx, nt, data_offset}; `names` (capacity names_cap, may be NULL)
 * receives the variable names NUL-terminated back to back; *names_len (may be
 * NULL) the bytes they need. Context-free: the message of a failed call is
 * dopinf_b200_last_error(NULL) on the calling thread. */
int dopinf_b200_snp1_header(const char* path, uint64_t* dims, char* names, size_t names_cap,
                            size_t* names_len);
/* data::read_block (data.cpp:164-202): rows [row_begin, row_end) of every
 * variable (the rank's plan entry; the C++ mirror checks the plan itself)
 * into a new device block, each variable's slice one contiguous byte range of
 * the file, read through a pinned two-slot ring whose H2D copies overlap the
 * next read. */
int dopinf_b200_block_read(dopinf_b200_ctx* ctx, const char* path, size_t row_begin, size_t row_end,
                           dopinf_b200_block** out);
/* Read + Steps II-III in one streamed call (pipeline.cpp:254-280): the rank's
 * slice is read chunk by chunk into the pinned ring; while chunk c+1 is read
 * and copied, chunk c is centered and its Gram accumulated on the device
 * (as dopinf_b200_snapshot_pass_host). *out receives the resident, transformed
 * block; means [n_vars*(row_end-row_begin)], scales [n_vars], d [nt x nt] as
 * in dopinf_b200_snapshot_pass. On any error *out stays NULL. */
int dopinf_b200_snapshot_pass_file(dopinf_b200_ctx* ctx, const char* path, size_t row_begin,
                                   size_t row_end, int scaling, dopinf_b200_block** out, double* means,
                                   double* scales, double* d);

/* ---- Step IV: OpInf regularisation grid search (rom_search.hpp) ----------- */
/* rom_search::grid_search (rom_search.cpp:185-262) on the device. qhat: host
 * r x nt (pod::project's Q̂), or NULL for the context's device Q̂ of the last
 * dopinf_b200_project (r, nt must match it). Candidate pair idx = i1*n2 + i2
 * is (b1[i1], b2[i2]); pairs are split over the context's ranks as
 * distribute_pairs does, each rank solves, integrates and scores its slice
 * (DhatᵀDhat and Dhatᵀ Qhat2ᵀ once; cuSOLVER Cholesky per pair; all ROMs
 * integrated concurrently, bit-identical steps to rom_search::integrate for
 * the same operators), and the winner — lowest training error among the
 * admissible pairs, first index on ties — is agreed with MIN collectives and
 * its trajectory broadcast from the owner. Outputs (host, each may be NULL):
 * pair_opt[2] = {beta1, beta2}, train_err, owner, rom_seconds (device time of
 * the integration launch), trajectory nt_p x r. Errors as the reference:
 * InvalidArgumentError, SolveError, NoAdmissiblePairError (same messages). */
/* rom_search::distribute_pairs (rom_search.cpp:136-149): the contiguous slice
 * [*begin, *end) of n_reg candidates owned by `rank` of `size` (remainder to
 * the last rank; ranks beyond n_reg get empty slices). Host only. */
int dopinf_b200_distribute_pairs(size_t n_reg, int rank, int size, size_t* begin, size_t* end);
int dopinf_b200_grid_search(dopinf_b200_ctx* ctx, const double* qhat, size_t r, size_t nt, const double* b1,
                            size_t n1, const double* b2, size_t n2, double max_growth, size_t nt_p,
                            double* pair_opt, double* train_err, int* owner, double* rom_seconds,
                            double* trajectory);
/* rom_search::integrate (rom_search.cpp:62-87): q_{k+1} = A q_k + F quad(q_k) + c
 * from q0 for n_steps rows (row 0 = q0), bit-identical to the reference for
 * the same operators. a: r x r, f: r x r(r+1)/2, c: r, q0: r (host);
 * traj: host n_steps x r; finite: 1 iff every entry is finite. */
int dopinf_b200_rom_integrate(dopinf_b200_ctx* ctx, const double* a, const double* f, const double* c, size_t r,
                              const double* q0, size_t n_steps, double* traj, int* finite);

/* ---- Step V: field reconstruction (postprocess.hpp:40-45) ----------------- */
/* postprocess::reconstruct_field (postprocess.cpp:63-70): this rank's field
 * (n_vars*nx_i) x nt_p in original coordinates,
 *   field = inverse_transform_block(matmul_nt(Q·T_r, Q̃))  (transform.cpp:62-72),
 * i.e. X[row][t] = s_row · (Φ_r[row]·Q̃[t]) + mean_row with one FMA. The block
 * must hold the transformed values (after a snapshot pass). tr: host K x r, or
 * NULL for the context's device T_r (dopinf_b200_reduced_map). qtilde: host
 * nt_p x r (the ROM trajectory, rows = time). means [rows] and scales [n_vars]
 * are the TransformParams (scales ignored unless scaling). field: host
 * (rows x nt_p) or NULL to keep it on the device (dopinf_b200_field_device).
 * Φ_r is left on the device as after dopinf_b200_basis. */
int dopinf_b200_reconstruct_field(dopinf_b200_block* block, const double* tr, size_t r, const double* qtilde,
                                  size_t nt_p, const double* means, const double* scales, int scaling,
                                  double* field);
/* postprocess::reconstruct_probes (postprocess.cpp:36-61): the time series
 * of every probe this rank owns — probe i is (var[i], index[i]), owned when
 * index[i] lies in [row_begin, row_begin + nx_i) — in original coordinates:
 * series[i][t] = s·dot(Q[row]·T_r, Q̃[t]) + mean with the reference's
 * basis_rows, kernels::dot and scale_shift orders, so bit-identical to the
 * reference for the same block, T_r, Q̃ and TransformParams. tr: host K x r,
 * or NULL for the context's device T_r; qtilde: host nt_p x r; means [rows],
 * scales [n_vars] (scaling); series: host n_probes x nt_p (rows of unowned
 * probes untouched); owned: n_probes flags, may be NULL. */
int dopinf_b200_reconstruct_probes(dopinf_b200_block* block, const double* tr, size_t r, const double* qtilde,
                                   size_t nt_p, const size_t* var, const size_t* index, size_t n_probes,
                                   const double* means, const double* scales, int scaling, double* series, int* owned);
/* Device pointer and pitch (elements) of the last reconstructed field. */
int dopinf_b200_field_device(dopinf_b200_block* block, double** field, size_t* ld);
/* Step V field output (pipeline.cpp:330-350): reconstruct_field + write_snapshots
 * of the SNP1 file `path` (n_vars, nx = nx_i, nt = nt_p; `names` = n_vars
 * NUL-terminated names back to back), streamed: row chunks of the field are
 * computed on the device, copied into a pinned ring and written while the next
 * chunk computes — the whole field is never resident. Header checks and
 * messages as data::write_snapshots (DataFormatError). */
int dopinf_b200_write_field(dopinf_b200_block* block, const double* tr, size_t r, const double* qtilde,
                            size_t nt_p, const double* means, const double* scales, int scaling, const char* names,
                            const char* path);

#ifdef __cplusplus
}
#endif

#endif /* DOPINF_B200_H */
