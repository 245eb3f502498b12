// capi_internal.h — internals shared by the C ABI's translation units
// (capi.cu: contexts, blocks, Steps II–III, projection, basis, eigensolve;
// capi_io.cu: streamed passes and SNP1 files; capi_post.cu: grid search and
// field reconstruction): status plumbing, grow-only buffers, the per-rank
// context and device block, and the stage helpers the entry points share.
// Nothing here crosses the ABI.
#pragma once

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <functional>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <mutex>
#include <new>
#include <optional>
#include <set>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/dopinf_b200.h"
#include "common.cuh"
#include "eig.h"
#include "field.h"
#include "gram.h"
#include "project.h"
#include "rom.h"
#include "synth.h"
#include "transform.h"

namespace dopinf_b200 {
namespace capi {

// Status + message carrier; thrown only inside the ABI translation units and
// caught by guarded() at every entry point.
struct Fail {
    int status;
    std::string msg;
};

[[noreturn]] inline void fail(int status, std::string msg) { throw Fail{status, std::move(msg)}; }

inline void ck(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        fail(DOPINF_B200_ERR_OUT_OF_MEMORY, std::string(what) + ": out of device memory");
    }
    if (e != cudaSuccess) fail(DOPINF_B200_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

inline void ckn(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        fail(DOPINF_B200_ERR_COLLECTIVE, std::string(what) + ": " + ncclGetErrorString(r));
    }
}

// Guarded device allocations (debug aid; compute-sanitizer is unavailable on
// the B200 pool): with DOPINF_B200_GUARD_BYTES=G set, every library
// allocation gets G bytes of a known pattern before and after it; a kernel
// that writes outside its buffer corrupts a guard, which the release of the
// buffer and dopinf_b200_debug_guard_violations() detect. G = 0 (default): off.
size_t guard_bytes();
cudaError_t dev_alloc(void** p, size_t bytes);
void dev_free(void* p);

// NVTX range over a stage (shows in Nsight Systems / `ncu --nvtx`; header-only
// NVTX v3, a no-op without a tool attached).
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

// Grow-only device buffer.
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    template <class T>
    T* get(size_t count, const char* what) {
        const size_t need = std::max<size_t>(count * sizeof(T), 16);
        if (need > bytes) {
            if (p) dev_free(p);
            p = nullptr;
            bytes = 0;
            ck(dev_alloc(&p, need), what);
            bytes = need;
        }
        return static_cast<T*>(p);
    }
    void release() {
        if (p) dev_free(p);
        p = nullptr;
        bytes = 0;
    }
};

// rows × width doubles between pitched buffers; one linear copy when both
// pitches equal the width (the copy engines stream it at the full link rate).
inline cudaError_t copy_rows(double* dst, size_t dld, const double* src, size_t sld, size_t width, size_t rows,
                      cudaMemcpyKind kind, cudaStream_t stream) {
    if (dld == width && sld == width) {
        return cudaMemcpyAsync(dst, src, rows * width * sizeof(double), kind, stream);
    }
    return cudaMemcpy2DAsync(dst, dld * sizeof(double), src, sld * sizeof(double), width * sizeof(double), rows,
                             kind, stream);
}

inline bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

// Grow-only pinned host staging buffer (pageable D2H through the driver runs
// at a few GB/s; a pinned hop plus a host memcpy is several times faster).
struct PinnedBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
        if (need > bytes) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            bytes = 0;
            ck(cudaMallocHost(&p, need), "pinned staging");
            bytes = need;
        }
        return p;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        bytes = 0;
    }
};

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

// Message of the last failed context-free call (or null-context call) on this thread.
extern thread_local std::string g_thread_err;

}  // namespace capi
}  // namespace dopinf_b200

using namespace dopinf_b200;
using namespace dopinf_b200::capi;

struct dopinf_b200_ctx {
    int device = 0, rank = 0, size = 1;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;    // streamed pass: H2D of chunk c+1 overlaps chunk c
    std::vector<cudaEvent_t> chunk_events;  // one per streamed chunk (grow-only)
    DBuf gv;                                // per-variable packed Grams of the streamed pass
    DBuf ring;                              // synth stream: two chunk slots
    PinnedBuf file_ring;                    // SNP1 reads: two pinned chunk slots
    std::vector<cudaEvent_t> chunk_events2; // field writer: compute-done events
    DBuf field_qt, field_means, field_scales, field_ring;
    std::vector<cudaEvent_t> timing_events; // streamed Gram launches: start/end pairs
    size_t stream_gram_ms_events_used = 0;
    struct EvList {
        std::vector<cudaEvent_t>* pool;
        size_t* used;
        void clear() { *used = 0; }
    } stream_gram_ms_events{&timing_events, &stream_gram_ms_events_used};

    // Record one timing event on the compute stream (pairs bracket Gram launches).
    void gram_event_pair() {
        if (stream_gram_ms_events_used == timing_events.size()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            timing_events.push_back(e);
        }
        ck(cudaEventRecord(timing_events[stream_gram_ms_events_used++], stream), "event");
    }
    // Sum of the bracketed Gram launch times of the last streamed pass (ms).
    double stream_gram_ms() const {
        double total = 0.0;
        for (size_t i = 0; i + 1 < stream_gram_ms_events_used; i += 2) {
            float f = 0.0f;
            if (cudaEventSynchronize(timing_events[i + 1]) == cudaSuccess &&
                cudaEventElapsedTime(&f, timing_events[i], timing_events[i + 1]) == cudaSuccess) {
                total += f;
            }
        }
        return total;
    }
    ncclComm_t comm = nullptr;
    bool owns_comm = true, owns_stream = true;  // false: handed in by dopinf_b200_ctx_create_external
    int gram_reduce = DOPINF_B200_GRAM_REDUCE_NCCL;
    int gram_order = DOPINF_B200_GRAM_ORDER_TENSOR;
    std::string err;

    // Collectives (capi_coll.cu). Every NCCL call goes through coll_*: a
    // poisoned context refuses them, an optional (count, op) agreement check
    // runs first, and sync() waits for a queued collective with a deadline
    // (ncclCommGetAsyncError polled; on expiry ncclCommAbort + poison), the
    // reference's group semantics (comm_inprocess.cpp:41-87).
    double coll_timeout_s = 60.0;    // comm_inprocess.cpp kTimeout
    bool coll_checks = false;        // verify_uniform (comm_inprocess.cpp:139-151) before each collective
    bool coll_pending = false;       // an NCCL op is queued on `stream` since the last completed sync
    bool poisoned = false;
    std::string poison_msg;
    long long coll_seq = 0;          // collectives issued (agreement checks compare it across ranks)
    int inject = 0;                  // dopinf_b200_debug_inject (one-shot)
    int* stall_flag = nullptr;       // host-mapped release flag of an injected stall
    DBuf coll_scratch;

    // Gram state
    int K = 0;                 // nt of the Gram held on the device
    bool have_gram = false;    // dmat holds a Gram (local, reduced or set_gram)
    bool local_valid = false;  // packed holds this rank's local partial (K(K+1)/2 + status slot)
    bool dmat_local = false;   // dmat is the unpacked local partial
    int plan_K = -1;
    long long plan_rows = -1;
    gram::Plan plan;
    int tiles_K = -1;
    DBuf tiles, work, counters, packed, gpacked, gather, dmat, dhost_in, reduce_scratch;
    bool counters_zeroed = false;
    // scratch
    DBuf scales, tr, trt, qhat, sel, rows_out, span;
    PinnedBuf staging;
    // Pinned landing zone for the small results of collectives: a D2H into
    // pageable memory would block the host until the stream drains, i.e.
    // outside sync()'s deadline.
    PinnedBuf coll_host;
    template <class T>
    T* small_pinned(size_t count) {
        return static_cast<T*>(coll_host.get(std::max<size_t>(count * sizeof(T), 64)));
    }
    // device eigensolve (dopinf_b200_eig_sym_desc / dopinf_b200_reduced_map)
    eig::Solver solver;
    DBuf eig_a, eig_w, eig_work, eig_info, eig_v, eig_lambda, tr_dev;
    size_t qhat_r = 0, qhat_nt = 0;  // shape of the device Q̂ of the last projection
    // grid search (dopinf_b200_grid_search)
    DBuf rom_qhat, rom_dhat, rom_q2t, rom_qrows, rom_rhs, rom_g, rom_lhs, rom_rhsb, rom_betas, rom_traj, rom_scores,
        rom_work, rom_info, rom_tiles, rom_gwork, rom_counters, rom_packed, rom_packet;
    int eig_K = 0;      // size of the held eigendecomposition (0: none)
    size_t tr_dev_r = 0;

    // Device → host copy that completes before returning (callers sync anyway).
    void d2h(void* dst, const void* src, size_t bytes, const char* what) {
        if (bytes < (size_t(1) << 20) || is_pinned(dst)) {
            ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream), what);
            ck(cudaStreamSynchronize(stream), what);
            return;
        }
        void* st = staging.get(bytes);
        ck(cudaMemcpyAsync(st, src, bytes, cudaMemcpyDeviceToHost, stream), what);
        ck(cudaStreamSynchronize(stream), what);
        std::memcpy(dst, st, bytes);
    }
    // stage timing
    cudaEvent_t ev[DOPINF_B200_STAGE_COUNT][2] = {};
    bool ev_done[DOPINF_B200_STAGE_COUNT] = {};

    void record(int stage, int which) {
        cudaEventRecord(ev[stage][which], stream);
        if (which == 1) ev_done[stage] = true;
    }
    // Wait for the stream; with a collective queued, poll with the deadline.
    void sync(const char* what);
};

struct dopinf_b200_block {
    dopinf_b200_ctx* ctx = nullptr;
    size_t n_vars = 0, nx_i = 0, row_begin = 0, nt = 0, ld = 0, rows = 0;
    double* q = nullptr;
    DBuf means, varmax, phi, field;
    int phi_ld = 0;
    size_t field_ld = 0;  // pitch of the last reconstructed field (0: none)
    bool pending_center = false;  // means computed, subtraction not yet applied
    bool stats_valid = false;     // varmax describes the current (logical) values
    CUtensorMap gram_map{};
    const double* gram_map_base = nullptr;
};

namespace dopinf_b200 {
namespace capi {

// Context-free entry points: status + message on the calling thread.
template <class F>
int guarded_free(F&& fn) {
    try {
        fn();
        return DOPINF_B200_OK;
    } catch (const Fail& f) {
        g_thread_err = f.msg;
        return f.status;
    } catch (const std::bad_alloc&) {
        g_thread_err = "host allocation failed";
        return DOPINF_B200_ERR_OUT_OF_MEMORY;
    } catch (...) {
        g_thread_err = "unexpected failure";
        return DOPINF_B200_ERR_DEVICE;
    }
}

template <class F>
int guarded(dopinf_b200_ctx* ctx, F&& fn) {
    if (!ctx) {
        g_thread_err = "null context";
        return DOPINF_B200_ERR_INVALID_ARGUMENT;
    }
    try {
        DeviceGuard dg(ctx->device);
        fn();
        ctx->err.clear();
        return DOPINF_B200_OK;
    } catch (const Fail& f) {
        ctx->err = f.msg;
        return f.status;
    } catch (const std::bad_alloc&) {
        ctx->err = "host allocation failed";
        return DOPINF_B200_ERR_OUT_OF_MEMORY;
    } catch (...) {
        ctx->err = "unexpected failure";
        return DOPINF_B200_ERR_DEVICE;
    }
}

inline void require(bool ok, const std::string& msg) {
    if (!ok) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, msg);
}

// ---- SNP1 snapshot files (reference data.hpp:11-15, data.cpp) ----------------
// "SNP1", little-endian u64 n_vars / nx / nt, names as u32 length + bytes,
// then per variable an nx x nt row-major fp64 matrix: a rank's rows of one
// variable are one contiguous byte range.
struct Snp1 {
    uint64_t n_vars = 0, nx = 0, nt = 0, data_offset = 0, file_bytes = 0;
    std::vector<std::string> names;
};

[[noreturn]] inline void format_fail(const std::string& msg) { fail(DOPINF_B200_ERR_DATA_FORMAT, msg); }

struct Fd {
    int fd = -1;
    Fd() = default;
    Fd(const Fd&) = delete;
    Fd& operator=(const Fd&) = delete;
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

// ---- collectives (capi_coll.cu) ------------------------------------------------
// True when the context's collectives run over NCCL (a communicator, or a
// poisoned context whose calls must keep failing).
inline bool coll(const dopinf_b200_ctx* c) { return c->comm != nullptr || c->poisoned; }
void coll_allreduce(dopinf_b200_ctx* c, const void* send, void* recv, size_t count, ncclDataType_t type,
                    ncclRedOp_t op, const char* what);
void coll_allgather(dopinf_b200_ctx* c, const void* send, void* recv, size_t count, ncclDataType_t type,
                    const char* what);
void coll_broadcast(dopinf_b200_ctx* c, void* buf, size_t count, ncclDataType_t type, int root, const char* what);
// Bounded wait on a side stream (a poisoned context must not hang in teardown).
void join_stream(dopinf_b200_ctx* c, cudaStream_t s);
// The rank's own communicator: non-blocking init bounded by the deadline
// (DOPINF_B200_COLLECTIVE_TIMEOUT seconds, default 60); finalize + destroy.
void comm_init(dopinf_b200_ctx* c, int size, const ncclUniqueId& uid, int rank);
void comm_destroy(dopinf_b200_ctx* c);
// The status slot a rank contributes to a SUM-reduced buffer: 2^rank when it
// failed (exact for up to 52 ranks; beyond that every failure reads as rank 52+).
inline double failure_bit(const dopinf_b200_ctx* c, bool failed) {
    return failed ? std::ldexp(1.0, std::min(c->rank, 52)) : 0.0;
}
// Lowest failing rank from a summed status slot, -1 when none failed.
inline int lowest_failed(double bits) {
    if (!(bits > 0.0)) return -1;
    for (int r = 0; r <= 52; ++r) {
        if (std::fmod(std::floor(bits / std::ldexp(1.0, r)), 2.0) == 1.0) return r;
    }
    return 52;
}
// Run a rank-local step whose failure must still let this rank enter the
// collective that follows (so peers learn of it instead of timing out).
template <class F>
std::optional<Fail> attempt(dopinf_b200_ctx* c, F&& fn) {
    if (!coll(c)) {
        fn();
        return std::nullopt;
    }
    try {
        fn();
    } catch (const Fail& f) {
        if (c->poisoned) throw;
        return f;
    } catch (const std::bad_alloc&) {
        return Fail{DOPINF_B200_ERR_OUT_OF_MEMORY, "host allocation failed"};
    }
    return std::nullopt;
}
// After the collective: rethrow this rank's own failure, else report a peer's
// (the reference's peers see CollectiveError "rank r aborted", comm_inprocess.cpp:171).
inline void settle(const std::optional<Fail>& own, int failed_rank) {
    if (own) throw *own;
    if (failed_rank >= 0) fail(DOPINF_B200_ERR_COLLECTIVE, "rank " + std::to_string(failed_rank) + " aborted");
}

// Process-wide pool of host threads for the staged copies (pinned ring fills
// and drains, parallel pread / pwrite): spawning threads per 64 MB chunk cost
// ~20-30% of a staged copy. parallel_for runs fn(0..n-1) on the pool and the
// calling thread and returns when all are done; one job at a time (concurrent
// callers — in-process ranks — take turns; the copies are bandwidth bound).
void parallel_for(int n, const std::function<void(int)>& fn);

// ---- helpers defined in capi.cu / capi_io.cu --------------------------------
void materialize(dopinf_b200_block* b);
void run_stats(dopinf_b200_block* b, bool center);
void do_center(dopinf_b200_block* b, double* means_host, bool side_copy = false);
void do_global_scales(dopinf_b200_block* b, double* scales_host, size_t* degenerate,
                      const std::optional<Fail>& earlier = std::nullopt);
void do_scale(dopinf_b200_block* b, const double* scales_host);
void copy_d_out(dopinf_b200_ctx* c, double* d_host);
void unpack(dopinf_b200_ctx* c, const double* packed);
void ensure_tiles(dopinf_b200_ctx* c, int K);
int* ensure_counters(dopinf_b200_ctx* c);
void do_local_gram(dopinf_b200_block* b, double* d_host);
void do_global_gram(dopinf_b200_ctx* c, double* d_host, const std::optional<Fail>& local_failure = std::nullopt);
bool pread_all(int fd, void* dst, size_t bytes, uint64_t off);
void staged_upload(dopinf_b200_block* b, const double* host, size_t host_ld);
void staged_download(dopinf_b200_block* b, size_t row0, size_t nrows, double* host, size_t host_ld);
void open_snp1(Fd& f, const std::string& path);
void validate_snp1(const Snp1& h);
void check_snp1_payload(const Snp1& h, const std::string& path);
Snp1 read_snp1_header(int fd, const std::string& path);
int file_reader_threads();
bool pread_parallel(int fd, void* dst, size_t bytes, uint64_t off);
const double* tr_operand(dopinf_b200_ctx* c, const double* tr_host, size_t nt, size_t r);
void do_project(dopinf_b200_ctx* c, const double* tr_host, const double* d_dev, size_t nt, size_t r,
                double* qhat_host);
int do_basis(dopinf_b200_block* b, const double* tr, size_t r);
void ensure_events(std::vector<cudaEvent_t>& v, size_t n);
bool pwrite_parallel(int fd, const void* src, size_t bytes, uint64_t off);

}  // namespace capi
}  // namespace dopinf_b200
