// capi.cu — the C ABI (include/dopinf_b200.h): per-rank contexts, device-
// resident LocalBlocks, NCCL collectives and the stage orchestration that the
// reference's pipeline::run_rank (proj/src/pipeline.cpp:270-298) performs on
// the host. Every entry point is synchronous at the boundary, never throws,
// and maps failures onto the reference's exception classes by status code.
#include <nccl.h>

#include <errno.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <limits>
#include <mutex>
#include <new>
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

using namespace dopinf_b200;

namespace dopinf_b200 {

static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        const bool ok = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
                        q == cudaDriverEntryPointSuccess;
        return ok ? reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p) : nullptr;
    }();
    return fn;
}

cudaError_t set_smem_attr_once(const void* func, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({func, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({func, dev});
    return e;
}

}  // namespace dopinf_b200

namespace {

// Status + message carrier; thrown only inside this file.
struct Fail {
    int status;
    std::string msg;
};

[[noreturn]] void fail(int status, std::string msg) { throw Fail{status, std::move(msg)}; }

// Message of the last failed context-free call (or null-context call) on this thread.
thread_local std::string g_thread_err = "null context";

void ck(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        fail(DOPINF_B200_ERR_OUT_OF_MEMORY, std::string(what) + ": out of device memory");
    }
    if (e != cudaSuccess) fail(DOPINF_B200_ERR_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
}

void ckn(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        fail(DOPINF_B200_ERR_COLLECTIVE, std::string(what) + ": " + ncclGetErrorString(r));
    }
}

// Grow-only device buffer.
struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    template <class T>
    T* get(size_t count, const char* what) {
        const size_t need = std::max<size_t>(count * sizeof(T), 16);
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            bytes = 0;
            ck(cudaMalloc(&p, need), what);
            bytes = need;
        }
        return static_cast<T*>(p);
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

// rows × width doubles between pitched buffers; one linear copy when both
// pitches equal the width (the copy engines stream it at the full link rate).
cudaError_t copy_rows(double* dst, size_t dld, const double* src, size_t sld, size_t width, size_t rows,
                      cudaMemcpyKind kind, cudaStream_t stream) {
    if (dld == width && sld == width) {
        return cudaMemcpyAsync(dst, src, rows * width * sizeof(double), kind, stream);
    }
    return cudaMemcpy2DAsync(dst, dld * sizeof(double), src, sld * sizeof(double), width * sizeof(double), rows,
                             kind, stream);
}

bool is_pinned(const void* p) {
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

}  // namespace

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
    int gram_reduce = DOPINF_B200_GRAM_REDUCE_ORDERED;
    std::string err;

    // Gram state
    int K = 0;                 // nt of the Gram held on the device
    bool have_gram = false;
    int plan_K = -1;
    long long plan_rows = -1;
    gram::Plan plan;
    int tiles_K = -1;
    DBuf tiles, work, counters, packed, gather, dmat, dhost_in;
    bool counters_zeroed = false;
    // scratch
    DBuf scales, tr, trt, qhat, sel, rows_out, span;
    PinnedBuf staging;
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
    void sync(const char* what) { ck(cudaStreamSynchronize(stream), what); }
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

namespace {

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

void require(bool ok, const std::string& msg) {
    if (!ok) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, msg);
}

// Apply a pending centering so the device values equal the reference's block.
void materialize(dopinf_b200_block* b) {
    if (!b->pending_center) return;
    auto* c = b->ctx;
    c->record(DOPINF_B200_STAGE_APPLY, 0);
    ck(transform::launch_apply(b->q, b->ld, static_cast<long long>(b->rows), static_cast<int>(b->nt),
                               static_cast<long long>(b->nx_i), b->means.get<double>(b->rows, "means"),
                               nullptr, c->num_sms, c->stream),
       "apply");
    c->record(DOPINF_B200_STAGE_APPLY, 1);
    b->pending_center = false;
}

void run_stats(dopinf_b200_block* b, bool center) {
    auto* c = b->ctx;
    double* vm = b->varmax.get<double>(b->n_vars, "varmax");
    double* mn = b->means.get<double>(b->rows, "means");
    c->record(DOPINF_B200_STAGE_STATS, 0);
    ck(cudaMemsetAsync(vm, 0, b->n_vars * sizeof(double), c->stream), "memset");
    ck(transform::launch_stats(b->q, b->ld, static_cast<long long>(b->rows), static_cast<int>(b->nt),
                               static_cast<long long>(b->nx_i), static_cast<int>(b->n_vars), center,
                               mn, vm, c->num_sms, c->stream),
       "stats");
    c->record(DOPINF_B200_STAGE_STATS, 1);
}

void do_center(dopinf_b200_block* b, double* means_host) {
    materialize(b);  // a second centering acts on centered values, as in the reference
    run_stats(b, true);
    b->pending_center = true;
    b->stats_valid = true;
    if (means_host) {
        ck(cudaMemcpyAsync(means_host, b->means.get<double>(b->rows, "means"), b->rows * sizeof(double),
                           cudaMemcpyDeviceToHost, b->ctx->stream),
           "means D2H");
    }
}

void do_global_scales(dopinf_b200_block* b, double* scales_host, size_t* degenerate) {
    auto* c = b->ctx;
    if (!b->stats_valid) {
        run_stats(b, false);
        b->stats_valid = true;
    }
    double* vm = b->varmax.get<double>(b->n_vars, "varmax");
    double* red = c->scales.get<double>(b->n_vars, "scales");
    c->record(DOPINF_B200_STAGE_SCALES, 0);
    if (c->size > 1) {
        ckn(ncclAllReduce(vm, red, b->n_vars, ncclFloat64, ncclMax, c->comm, c->stream), "allreduce(MAX)");
    } else {
        ck(cudaMemcpyAsync(red, vm, b->n_vars * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "copy");
    }
    c->record(DOPINF_B200_STAGE_SCALES, 1);
    std::vector<double> host(b->n_vars);
    ck(cudaMemcpyAsync(host.data(), red, b->n_vars * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
       "scales D2H");
    c->sync("global_scales");
    if (scales_host) std::memcpy(scales_host, host.data(), b->n_vars * sizeof(double));
    for (size_t j = 0; j < b->n_vars; ++j) {
        if (host[j] == 0.0) {
            if (degenerate) *degenerate = j;
            fail(DOPINF_B200_ERR_DEGENERATE_VARIABLE,
                 "variable " + std::to_string(j) + " is constant in time; max-abs scaling is undefined");
        }
    }
}

void do_scale(dopinf_b200_block* b, const double* scales_host) {
    auto* c = b->ctx;
    double* ds = c->scales.get<double>(b->n_vars, "scales");
    ck(cudaMemcpyAsync(ds, scales_host, b->n_vars * sizeof(double), cudaMemcpyHostToDevice, c->stream),
       "scales H2D");
    c->record(DOPINF_B200_STAGE_APPLY, 0);
    ck(transform::launch_apply(b->q, b->ld, static_cast<long long>(b->rows), static_cast<int>(b->nt),
                               static_cast<long long>(b->nx_i),
                               b->pending_center ? b->means.get<double>(b->rows, "means") : nullptr, ds,
                               c->num_sms, c->stream),
       "apply");
    c->record(DOPINF_B200_STAGE_APPLY, 1);
    b->pending_center = false;
    b->stats_valid = false;
}

void copy_d_out(dopinf_b200_ctx* c, double* d_host) {
    if (!d_host) return;
    c->record(DOPINF_B200_STAGE_DOWNLOAD, 0);
    const size_t n = static_cast<size_t>(c->K) * c->K;
    c->d2h(d_host, c->dmat.get<double>(n, "D"), n * sizeof(double), "D D2H");
    c->record(DOPINF_B200_STAGE_DOWNLOAD, 1);
}

void unpack(dopinf_b200_ctx* c) {
    const int K = c->K;
    c->record(DOPINF_B200_STAGE_UNPACK, 0);
    ck(gram::launch_unpack(c->packed.get<double>(gram::packed_count(K), "packed"), K,
                           c->dmat.get<double>(static_cast<size_t>(K) * K, "D"), c->stream),
       "unpack");
    c->record(DOPINF_B200_STAGE_UNPACK, 1);
}

void ensure_tiles(dopinf_b200_ctx* c, int K) {
    if (c->tiles_K == K) return;
    const std::vector<gram::TileInfo> t = gram::plan_tiles(K);
    ck(cudaMemcpy(c->tiles.get<gram::TileInfo>(t.size(), "tiles"), t.data(), t.size() * sizeof(gram::TileInfo),
                  cudaMemcpyHostToDevice),
       "tiles H2D");
    c->tiles_K = K;
}

int* ensure_counters(dopinf_b200_ctx* c) {
    int* counters = c->counters.get<int>(2, "counters");
    if (!c->counters_zeroed) {
        ck(cudaMemsetAsync(counters, 0, 2 * sizeof(int), c->stream), "memset");
        c->counters_zeroed = true;
    }
    return counters;
}

void do_local_gram(dopinf_b200_block* b, double* d_host) {
    auto* c = b->ctx;
    materialize(b);
    const int K = static_cast<int>(b->nt);
    const long long rows = static_cast<long long>(b->rows);
    c->have_gram = false;
    c->K = K;
    double* packed = c->packed.get<double>(gram::packed_count(K), "packed");
    if (rows == 0) {
        ck(cudaMemsetAsync(packed, 0, gram::packed_count(K) * sizeof(double), c->stream), "memset");
    } else {
        ensure_tiles(c, K);
        if (c->plan_K != K || c->plan_rows != rows) {
            size_t free_b = 0, total_b = 0;
            cudaMemGetInfo(&free_b, &total_b);
            const size_t cap =
                std::min<size_t>(gram::kWorkspaceCapBytes, std::max<size_t>(free_b / 8, size_t(64) << 20));
            c->plan = gram::make_plan(rows, K, c->num_sms, cap);
            c->plan_K = K;
            c->plan_rows = rows;
        }
        if (b->gram_map_base != b->q) {
            ck(gram::make_tensor_map(&b->gram_map, b->q, rows, K, b->ld), "tensor map");
            b->gram_map_base = b->q;
        }
        int* counters = ensure_counters(c);
        double* work = c->work.get<double>(c->plan.workspace_doubles, "workspace");
        const auto* tiles = c->tiles.get<gram::TileInfo>(c->plan.n_tiles, "tiles");
        c->record(DOPINF_B200_STAGE_GRAM, 0);
        ck(gram::launch_gram(c->plan, b->gram_map, tiles, work, counters, c->stream), "gram");
        c->record(DOPINF_B200_STAGE_GRAM, 1);
        c->record(DOPINF_B200_STAGE_GRAM_REDUCE, 0);
        ck(gram::launch_reduce(c->plan, tiles, work, packed, c->stream), "gram reduce");
        c->record(DOPINF_B200_STAGE_GRAM_REDUCE, 1);
    }
    unpack(c);
    c->have_gram = true;
    copy_d_out(c, d_host);
}

void do_global_gram(dopinf_b200_ctx* c, double* d_host) {
    if (!c->have_gram) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "global_gram: no local Gram on this context");
    const int K = c->K;
    const size_t count = gram::packed_count(K);
    if (c->size > 1) {
        double* packed = c->packed.get<double>(count, "packed");
        c->record(DOPINF_B200_STAGE_ALLREDUCE, 0);
        if (c->gram_reduce == DOPINF_B200_GRAM_REDUCE_NCCL) {
            ckn(ncclAllReduce(packed, packed, count, ncclFloat64, ncclSum, c->comm, c->stream),
                "allreduce(SUM)");
        } else {
            double* parts = c->gather.get<double>(count * c->size, "gather");
            ckn(ncclAllGather(packed, parts, count, ncclFloat64, c->comm, c->stream), "allgather");
            ck(gram::launch_ordered_sum(parts, c->size, count, packed, c->stream), "ordered sum");
        }
        c->record(DOPINF_B200_STAGE_ALLREDUCE, 1);
        unpack(c);
    }
    copy_d_out(c, d_host);
}

// ---- streamed Steps II-III ----------------------------------------------------------
// dopinf_b200_snapshot_pass_host: rows arrive from host memory into the
// resident block (H2D on the copy stream overlaps the compute stream).
// dopinf_b200_stream_pass_synth: rows are generated on the device chunk by chunk
// into a two-slot ring — the block is never resident (config 4: 403 GB/GPU).
constexpr long long kStreamChunkRows = 32768;   // rows per H2D chunk (315 MB at K = 1200)
constexpr long long kStreamSplitRows = 2048;    // rows per Gram item inside a host chunk
constexpr long long kSynthChunkRows = 262144;   // rows per generated chunk (3.1 GB at K = 1500)
constexpr long long kSynthSplitRows = 8192;

// ---- SNP1 snapshot files (reference data.hpp:11-15, data.cpp) ----------------
// "SNP1", little-endian u64 n_vars / nx / nt, names as u32 length + bytes,
// then per variable an nx x nt row-major fp64 matrix: a rank's rows of one
// variable are one contiguous byte range.
struct Snp1 {
    uint64_t n_vars = 0, nx = 0, nt = 0, data_offset = 0, file_bytes = 0;
    std::vector<std::string> names;
};

[[noreturn]] void format_fail(const std::string& msg) { fail(DOPINF_B200_ERR_DATA_FORMAT, msg); }

struct Fd {
    int fd = -1;
    Fd() = default;
    Fd(const Fd&) = delete;
    Fd& operator=(const Fd&) = delete;
    ~Fd() {
        if (fd >= 0) close(fd);
    }
};

// Exactly `bytes` at `off`, or false (EOF / error).
bool pread_all(int fd, void* dst, size_t bytes, uint64_t off) {
    auto* p = static_cast<char*>(dst);
    while (bytes > 0) {
        const ssize_t n = pread(fd, p, bytes, static_cast<off_t>(off));
        if (n < 0 && errno == EINTR) continue;
        if (n <= 0) return false;
        p += n;
        bytes -= static_cast<size_t>(n);
        off += static_cast<uint64_t>(n);
    }
    return true;
}

void open_snp1(Fd& f, const std::string& path) {
    f.fd = open(path.c_str(), O_RDONLY | O_CLOEXEC);
    if (f.fd < 0) format_fail("cannot open snapshot file: " + path);  // data.cpp:61-65
}

// data.cpp:35-48 (same checks, same order, same messages).
void validate_snp1(const Snp1& h) {
    if (h.n_vars < 1) format_fail("snapshot header: n_vars must be >= 1");
    if (h.nx < 1) format_fail("snapshot header: nx must be >= 1");
    if (h.nt < 2) format_fail("snapshot header: nt must be >= 2");
    if (h.names.size() != h.n_vars) format_fail("snapshot header: name count does not match n_vars");
    std::set<std::string> seen;
    for (const auto& name : h.names) {
        if (name.empty()) format_fail("snapshot header: empty variable name");
        if (!seen.insert(name).second) format_fail("snapshot header: duplicate variable name '" + name + "'");
    }
}

// data.cpp:69-82: a payload shorter than the header promises names the
// variable the missing bytes belong to.
void check_snp1_payload(const Snp1& h, const std::string& path) {
    const unsigned __int128 per_var = static_cast<unsigned __int128>(h.nx) * h.nt * sizeof(double);
    const unsigned __int128 expected = h.data_offset + h.n_vars * per_var;
    if (h.file_bytes < expected) {
        const uint64_t have = h.file_bytes - std::min(h.file_bytes, h.data_offset);
        const uint64_t var =
            static_cast<uint64_t>(std::min<unsigned __int128>(have / per_var, h.n_vars - 1));
        format_fail("snapshot file truncated in variable '" + h.names[var] + "': " + path);
    }
}

// data::read_header (data.cpp:133-162).
Snp1 read_snp1_header(int fd, const std::string& path) {
    struct stat st;
    if (fstat(fd, &st) != 0) format_fail("cannot open snapshot file: " + path);
    Snp1 h;
    h.file_bytes = static_cast<uint64_t>(st.st_size);
    char magic[4] = {};
    if (!pread_all(fd, magic, 4, 0) || std::memcmp(magic, "SNP1", 4) != 0) {
        format_fail("not a snapshot file (bad magic): " + path);
    }
    uint64_t off = 4;
    auto u64 = [&](const char* field) {
        uint64_t v = 0;
        if (!pread_all(fd, &v, sizeof v, off)) format_fail(std::string("snapshot file truncated in ") + field);
        off += sizeof v;
        return v;
    };
    h.n_vars = u64("n_vars");
    h.nx = u64("nx");
    h.nt = u64("nt");
    if (h.n_vars > (1u << 20)) format_fail("snapshot header: implausible n_vars");
    for (uint64_t j = 0; j < h.n_vars; ++j) {
        const std::string where = "snapshot file truncated in name of variable " + std::to_string(j);
        uint32_t len = 0;
        if (!pread_all(fd, &len, sizeof len, off)) format_fail(where);
        off += sizeof len;
        if (off + len > h.file_bytes) format_fail(where);  // before allocating `len` bytes
        std::string name(len, '\0');
        if (!pread_all(fd, name.data(), len, off)) format_fail(where);
        off += len;
        h.names.push_back(std::move(name));
    }
    h.data_offset = off;  // data.cpp:51-58: 4 + 3*8 + sum(4 + len)
    validate_snp1(h);
    check_snp1_payload(h, path);
    return h;
}

// Reader threads per chunk: a page-cache or NVMe read of a few hundred MB is
// bound by one core's memcpy, so the byte range is split over several.
int file_reader_threads() {
    static const int n = [] {
        const unsigned hw = std::thread::hardware_concurrency();
        return static_cast<int>(std::max(1u, std::min(16u, hw / 2)));
    }();
    return n;
}

// pread `bytes` at `off` into `dst` on up to file_reader_threads() threads.
bool pread_parallel(int fd, void* dst, size_t bytes, uint64_t off) {
    constexpr size_t kPiece = size_t(8) << 20;
    const int n = static_cast<int>(std::min<size_t>(file_reader_threads(), (bytes + kPiece - 1) / kPiece));
    if (n <= 1) return pread_all(fd, dst, bytes, off);
    const size_t per = (bytes / n + 4095) / 4096 * 4096;
    std::vector<std::thread> threads;
    std::vector<char> ok(n, 0);
    for (int i = 0; i < n; ++i) {
        const size_t b0 = std::min(bytes, per * i), b1 = std::min(bytes, per * (i + 1));
        threads.emplace_back([&, i, b0, b1] {
            ok[i] = pread_all(fd, static_cast<char*>(dst) + b0, b1 - b0, off + b0) ? 1 : 0;
        });
    }
    for (auto& t : threads) t.join();
    return std::all_of(ok.begin(), ok.end(), [](char v) { return v != 0; });
}

struct StreamChunk {
    int var;
    long long r0, rows;
    bool first_of_var, last_of_var;
};

struct StreamSource {
    const double* host = nullptr;  // host rows (pitch host_ld) → resident block
    size_t host_ld = 0;
    bool synth = false;            // device-generated rows → ring buffer, block not resident
    uint64_t seed = 0;
    int n_modes = 0;
    double dt = 0.0, noise = 0.0;
    const double* amps = nullptr;  // host [n_vars] or null
    int fd = -1;                   // SNP1 file rows → pinned ring → resident block
    const Snp1* file = nullptr;
    const std::string* path = nullptr;
};

// File source: read chunk k of the block's rows into pinned ring slot k % 2
// and enqueue its H2D on the copy stream; chunk_events[k] marks the copy done
// (the compute stream waits on it; the read of chunk k + 2 into the same slot
// waits on it from the host).
void file_chunk_h2d(dopinf_b200_block* b, const StreamSource& src, const std::vector<StreamChunk>& chunks,
                    size_t k, double* ring, size_t slot_doubles) {
    auto* c = b->ctx;
    const StreamChunk& ch = chunks[k];
    if (k >= 2) ck(cudaEventSynchronize(c->chunk_events[k - 2]), "ring slot");
    double* slot = ring + (k % 2) * slot_doubles;
    const uint64_t local0 = static_cast<uint64_t>(ch.r0) - static_cast<uint64_t>(ch.var) * b->nx_i;
    const uint64_t first = static_cast<uint64_t>(ch.var) * src.file->nx + b->row_begin + local0;
    const size_t bytes = static_cast<size_t>(ch.rows) * b->nt * sizeof(double);
    if (!pread_parallel(src.fd, slot, bytes, src.file->data_offset + first * b->nt * sizeof(double))) {
        format_fail("snapshot file truncated in variable '" + src.file->names[ch.var] + "': " + *src.path);
    }
    ck(copy_rows(b->q + ch.r0 * b->ld, b->ld, slot, b->nt, b->nt, ch.rows, cudaMemcpyHostToDevice, c->copy_stream),
       "chunk H2D");
    ck(cudaEventRecord(c->chunk_events[k], c->copy_stream), "event");
}

std::vector<StreamChunk> stream_chunks(const dopinf_b200_block* b, long long chunk_rows) {
    std::vector<StreamChunk> out;
    for (size_t v = 0; v < b->n_vars; ++v) {
        const long long v0 = static_cast<long long>(v * b->nx_i), v1 = v0 + static_cast<long long>(b->nx_i);
        for (long long r0 = v0; r0 < v1; r0 += chunk_rows) {
            const long long rows = std::min(chunk_rows, v1 - r0);
            out.push_back({static_cast<int>(v), r0, rows, r0 == v0, r0 + rows == v1});
        }
    }
    return out;
}

// On the compute stream each landed chunk gets its row means / max-abs (stats
// pass), is centered in place, and its Gram items accumulate (chunk order)
// into the split slots of its variable. When a variable's last chunk is done
// its slots are reduced into G_v, its MAX goes over the ranks and (resident
// block) its rows are scaled. D = Σ_v G_v / s_v².
void do_stream_pass(dopinf_b200_block* b, const StreamSource& src, bool scaling, double* means_host,
                    double* scales_host) {
    auto* c = b->ctx;
    const int K = static_cast<int>(b->nt);
    const size_t count = gram::packed_count(K);
    const long long chunk_rows = src.synth ? kSynthChunkRows : kStreamChunkRows;
    const long long split_rows = src.synth ? kSynthSplitRows : kStreamSplitRows;
    b->pending_center = false;
    b->stats_valid = false;
    c->have_gram = false;
    c->K = K;
    const std::vector<StreamChunk> chunks = stream_chunks(b, chunk_rows);
    while (c->chunk_events.size() < chunks.size() + 1) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        c->chunk_events.push_back(e);
    }
    ensure_tiles(c, K);
    int* counters = ensure_counters(c);
    const auto* tiles = c->tiles.get<gram::TileInfo>(gram::plan_tiles(K).size(), "tiles");
    const long long first_rows = std::min<long long>(chunk_rows, static_cast<long long>(b->nx_i));
    const gram::Plan full =
        gram::make_stream_plan(std::max<long long>(first_rows, 1), K, c->num_sms, split_rows);
    double* work = c->work.get<double>(full.workspace_doubles, "workspace");
    double* gv = c->gv.get<double>(count * b->n_vars, "per-variable Grams");
    double* vm = b->varmax.get<double>(b->n_vars, "varmax");
    double* ds = c->scales.get<double>(b->n_vars, "scales");
    double* mn = b->means.get<double>(std::max<size_t>(b->rows, 1), "means");
    double* packed = c->packed.get<double>(count, "packed");
    double* ring = src.synth ? c->ring.get<double>(2 * static_cast<size_t>(first_rows) * b->ld, "chunk ring")
                             : nullptr;
    const bool from_file = src.fd >= 0;
    const size_t slot_doubles = static_cast<size_t>(first_rows) * b->nt;
    double* fring = from_file && !chunks.empty()
                        ? static_cast<double*>(c->file_ring.get(2 * slot_doubles * sizeof(double)))
                        : nullptr;
    std::vector<double> amps_v;  // per-variable amplitude slice for the generator
    if (src.synth && src.amps) amps_v.assign(src.amps, src.amps + b->n_vars);
    c->stream_gram_ms_events.clear();

    c->record(DOPINF_B200_STAGE_STREAM, 0);
    ck(cudaMemsetAsync(vm, 0, b->n_vars * sizeof(double), c->stream), "memset");
    ck(cudaMemsetAsync(gv, 0, count * b->n_vars * sizeof(double), c->stream), "memset");
    if (!src.synth) {
        // The copy stream must not overwrite the block before earlier work on it is done.
        cudaEvent_t ready = c->chunk_events[chunks.size()];
        ck(cudaEventRecord(ready, c->stream), "event");
        ck(cudaStreamWaitEvent(c->copy_stream, ready, 0), "event wait");
        if (from_file && !chunks.empty()) file_chunk_h2d(b, src, chunks, 0, fring, slot_doubles);
        for (size_t k = 0; !from_file && k < chunks.size(); ++k) {
            const StreamChunk& ch = chunks[k];
            ck(copy_rows(b->q + ch.r0 * b->ld, b->ld, src.host + ch.r0 * src.host_ld, src.host_ld, b->nt, ch.rows,
                         cudaMemcpyHostToDevice, c->copy_stream),
               "chunk H2D");
            ck(cudaEventRecord(c->chunk_events[k], c->copy_stream), "event");
        }
    }
    gram::Plan first_plan = full;
    for (size_t k = 0; k < chunks.size(); ++k) {
        const StreamChunk& ch = chunks[k];
        double* qk;
        if (src.synth) {
            qk = ring + (k % 2) * static_cast<size_t>(first_rows) * b->ld;
            const long long local0 = ch.r0 - static_cast<long long>(ch.var) * static_cast<long long>(b->nx_i);
            ck(synth::oscillator(qk, b->ld, ch.rows, K, ch.rows, static_cast<long long>(b->row_begin) + local0, 1,
                                 src.seed, src.n_modes, src.dt, src.noise, src.amps ? &amps_v[ch.var] : nullptr,
                                 c->num_sms, c->stream, ch.var),
               "synth chunk");
        } else {
            ck(cudaStreamWaitEvent(c->stream, c->chunk_events[k], 0), "event wait");
            qk = b->q + ch.r0 * b->ld;
        }
        // chunk = one variable's rows: present it to the kernels as a 1-variable block
        ck(transform::launch_stats(qk, b->ld, ch.rows, K, ch.rows, 1, true, mn + ch.r0, vm + ch.var, c->num_sms,
                                   c->stream),
           "stats");
        ck(transform::launch_apply(qk, b->ld, ch.rows, K, ch.rows, mn + ch.r0, nullptr, c->num_sms, c->stream),
           "center");
        CUtensorMap map;
        ck(gram::make_tensor_map(&map, qk, ch.rows, K, b->ld), "tensor map");
        const gram::Plan plan = gram::make_stream_plan(ch.rows, K, c->num_sms, split_rows);
        if (ch.first_of_var) first_plan = plan;
        c->gram_event_pair();
        ck(gram::launch_gram(plan, map, tiles, work, counters, c->stream, !ch.first_of_var), "gram");
        c->gram_event_pair();
        if (ch.last_of_var) {
            ck(gram::launch_reduce(first_plan, tiles, work, gv + static_cast<size_t>(ch.var) * count, c->stream),
               "gram reduce");
            if (scaling) {
                if (c->size > 1) {
                    ckn(ncclAllReduce(vm + ch.var, ds + ch.var, 1, ncclFloat64, ncclMax, c->comm, c->stream),
                        "allreduce(MAX)");
                } else {
                    ck(cudaMemcpyAsync(ds + ch.var, vm + ch.var, sizeof(double), cudaMemcpyDeviceToDevice,
                                       c->stream),
                       "copy");
                }
                if (!src.synth) {
                    const long long v0 = static_cast<long long>(ch.var) * static_cast<long long>(b->nx_i);
                    ck(transform::launch_apply(b->q + v0 * b->ld, b->ld, static_cast<long long>(b->nx_i), K,
                                               static_cast<long long>(b->nx_i), nullptr, ds + ch.var, c->num_sms,
                                               c->stream),
                       "scale");
                }
            }
        }
        // the host reads chunk k + 1 while the device copies and reduces chunk k
        if (from_file && k + 1 < chunks.size()) file_chunk_h2d(b, src, chunks, k + 1, fring, slot_doubles);
    }
    // the pinned ring is free for the next call once the last copy has landed
    if (from_file && !chunks.empty()) ck(cudaEventSynchronize(c->chunk_events[chunks.size() - 1]), "ring");
    if (b->rows == 0 && scaling) {  // an empty rank still joins the MAX collectives
        for (size_t v = 0; v < b->n_vars; ++v) {
            if (c->size > 1) {
                ckn(ncclAllReduce(vm + v, ds + v, 1, ncclFloat64, ncclMax, c->comm, c->stream), "allreduce(MAX)");
            } else {
                ck(cudaMemcpyAsync(ds + v, vm + v, sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "copy");
            }
        }
    }
    ck(gram::launch_combine_vars(gv, static_cast<int>(b->n_vars), count, scaling ? ds : nullptr, packed,
                                 c->stream),
       "combine");
    c->record(DOPINF_B200_STAGE_STREAM, 1);
    c->have_gram = true;
    if (means_host && b->rows > 0) c->d2h(means_host, mn, b->rows * sizeof(double), "means D2H");
    if (scaling) {
        std::vector<double> s(b->n_vars);
        c->d2h(s.data(), ds, b->n_vars * sizeof(double), "scales D2H");
        if (scales_host) std::memcpy(scales_host, s.data(), s.size() * sizeof(double));
        for (size_t j = 0; j < b->n_vars; ++j) {
            if (s[j] == 0.0) {
                fail(DOPINF_B200_ERR_DEGENERATE_VARIABLE,
                     "variable " + std::to_string(j) + " is constant in time; max-abs scaling is undefined");
            }
        }
    }
}

// data::read_block (data.cpp:164-202) into the device block: the file rows go
// through the pinned ring, each H2D overlapping the next chunk's read.
void do_block_read(dopinf_b200_block* b, const StreamSource& src) {
    auto* c = b->ctx;
    b->pending_center = false;
    b->stats_valid = false;
    const std::vector<StreamChunk> chunks = stream_chunks(b, kStreamChunkRows);
    if (chunks.empty()) return;
    while (c->chunk_events.size() < chunks.size() + 1) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        c->chunk_events.push_back(e);
    }
    const size_t slot_doubles = static_cast<size_t>(std::min<long long>(kStreamChunkRows, b->nx_i)) * b->nt;
    auto* fring = static_cast<double*>(c->file_ring.get(2 * slot_doubles * sizeof(double)));
    c->record(DOPINF_B200_STAGE_UPLOAD, 0);
    cudaEvent_t ready = c->chunk_events[chunks.size()];
    ck(cudaEventRecord(ready, c->stream), "event");
    ck(cudaStreamWaitEvent(c->copy_stream, ready, 0), "event wait");
    for (size_t k = 0; k < chunks.size(); ++k) file_chunk_h2d(b, src, chunks, k, fring, slot_doubles);
    ck(cudaStreamWaitEvent(c->stream, c->chunk_events[chunks.size() - 1], 0), "event wait");
    c->record(DOPINF_B200_STAGE_UPLOAD, 1);
    ck(cudaEventSynchronize(c->chunk_events[chunks.size() - 1]), "ring");
}

// ---- Step IV: OpInf grid search (rom_search.cpp:185-262) --------------------
// Host span all-reduce over NCCL (comm::allreduce_scalar's role).
void host_allreduce(dopinf_b200_ctx* c, double* data, size_t count, ncclRedOp_t op) {
    double* buf = c->span.get<double>(count, "span");
    ck(cudaMemcpyAsync(buf, data, count * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
    ckn(ncclAllReduce(buf, buf, count, ncclFloat64, op, c->comm, c->stream), "allreduce");
    ck(cudaMemcpyAsync(data, buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    c->sync("allreduce");
}

// rom_search::distribute_pairs (rom_search.cpp:147-160).
std::pair<size_t, size_t> distribute_pairs(size_t n_reg, int rank, int size) {
    const size_t ranks = static_cast<size_t>(size), rk = static_cast<size_t>(rank);
    if (ranks > n_reg) return rk < n_reg ? std::make_pair(rk, rk + 1) : std::make_pair(n_reg, n_reg);
    const size_t base = n_reg / ranks;
    return {rk * base, (rk + 1 == ranks) ? n_reg : (rk + 1) * base};
}

// G = DhatᵀDhat (d × d, full, bitwise symmetric) with the Gram kernel on the
// grid search's own plan/tiles (the snapshot pass's cached plan stays intact).
void rom_gram(dopinf_b200_ctx* c, const double* dhat, size_t ldd, int K, int d, double* g) {
    const std::vector<gram::TileInfo> t = gram::plan_tiles(d);
    auto* tiles = c->rom_tiles.get<gram::TileInfo>(t.size(), "rom tiles");
    ck(cudaMemcpyAsync(tiles, t.data(), t.size() * sizeof(gram::TileInfo), cudaMemcpyHostToDevice, c->stream),
       "tiles H2D");
    const gram::Plan plan = gram::make_plan(K, d, c->num_sms, size_t(256) << 20);
    int* counters = c->rom_counters.get<int>(2, "rom counters");
    ck(cudaMemsetAsync(counters, 0, 2 * sizeof(int), c->stream), "memset");
    double* work = c->rom_gwork.get<double>(plan.workspace_doubles, "rom gram workspace");
    double* packed = c->rom_packed.get<double>(gram::packed_count(d), "rom packed");
    CUtensorMap map;
    ck(gram::make_tensor_map(&map, dhat, K, d, ldd), "tensor map");
    ck(gram::launch_gram(plan, map, tiles, work, counters, c->stream), "gram");
    ck(gram::launch_reduce(plan, tiles, work, packed, c->stream), "gram reduce");
    ck(gram::launch_unpack(packed, d, g, c->stream), "unpack");
    c->sync("rom gram");  // the host tile table must outlive its copy
}

struct GridOutcome {
    double beta1 = 0.0, beta2 = 0.0, train_err = 0.0, rom_seconds = 0.0;
    int owner = -1;
};

GridOutcome do_grid_search(dopinf_b200_ctx* c, const double* qhat_host, size_t r, size_t nt, const double* b1,
                           size_t n1, const double* b2, size_t n2, double max_growth, size_t nt_p,
                           double* traj_host) {
    // rom_search.cpp:187-203 (same checks, same order, same messages)
    if (n1 == 0 || n2 == 0) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "grid_search: empty candidate grid");
    require(b1 && b2, "grid_search: null candidate arrays");
    for (size_t i = 0; i < n1; ++i) {
        if (!(b1[i] > 0.0)) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "grid_search: b1 candidates must be positive");
    }
    for (size_t i = 0; i < n2; ++i) {
        if (!(b2[i] > 0.0)) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "grid_search: b2 candidates must be positive");
    }
    if (!(max_growth > 0.0)) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "grid_search: max_growth must be positive");
    if (nt_p < nt) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "grid_search: trial horizon shorter than training");
    if (nt < 2) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "assemble_data: need at least 2 snapshots");
    require(r >= 1 && r <= 180, "grid_search: r must lie in [1, 180]");
    const int R = static_cast<int>(r), NT = static_cast<int>(nt), NTP = static_cast<int>(nt_p);
    const int S = R * (R + 1) / 2, D = R + S + 1, KK = NT - 1;
    const size_t ldd = (static_cast<size_t>(D) + 1) / 2 * 2;

    // Q̂ (r × nt) on the device
    const double* dq;
    if (qhat_host) {
        double* q = c->rom_qhat.get<double>(r * nt, "rom qhat");
        ck(cudaMemcpyAsync(q, qhat_host, r * nt * sizeof(double), cudaMemcpyHostToDevice, c->stream), "qhat H2D");
        dq = q;
    } else {
        require(c->qhat_r == r && c->qhat_nt == nt, "grid_search: no device Q-hat of this shape on the context");
        dq = c->qhat.get<double>(r * nt, "qhat");
    }
    // pair-independent data: Dhat, Qhat2ᵀ, qhat_rows, G = DhatᵀDhat, Dhatᵀ Qhat2ᵀ
    double* dhat = c->rom_dhat.get<double>(static_cast<size_t>(KK) * ldd, "dhat");
    double* q2t = c->rom_q2t.get<double>(static_cast<size_t>(KK) * r, "qhat2t");
    double* qrows = c->rom_qrows.get<double>(nt * r, "qhat rows");
    double* g = c->rom_g.get<double>(static_cast<size_t>(D) * D, "dhat gram");
    double* rhs = c->rom_rhs.get<double>(static_cast<size_t>(D) * r, "rhs");
    ck(rom::launch_assemble(dq, R, NT, dhat, ldd, q2t, c->stream), "assemble");
    ck(rom::launch_transpose(dq, R, NT, qrows, c->stream), "transpose");
    rom_gram(c, dhat, ldd, KK, D, g);
    ck(rom::launch_rhs(dhat, ldd, q2t, KK, D, R, rhs, c->stream), "rhs");

    // this rank's candidates, solved / integrated / scored in batches that fit
    const size_t n_reg = n1 * n2;
    const auto mine = distribute_pairs(n_reg, c->rank, c->size);
    const size_t np = mine.second - mine.first;
    const size_t per_pair = static_cast<size_t>(D) * D + static_cast<size_t>(D) * r + nt_p * r;
    const size_t batch = std::max<size_t>(1, std::min<size_t>(std::max<size_t>(np, 1),
                                                               (size_t(8) << 30) / (per_pair * sizeof(double))));
    std::string err;
    int* info = c->rom_info.get<int>(2 * batch, "potrf info");
    double* betas = c->rom_betas.get<double>(2 * batch, "betas");
    double* lhs = c->rom_lhs.get<double>(batch * D * D, "lhs");
    double* rhsb = c->rom_rhsb.get<double>(batch * D * r, "rhs batch");
    double* traj = c->rom_traj.get<double>(batch * nt_p * r, "trajectories");
    double* scores = c->rom_scores.get<double>(batch * rom::kScoreFields, "scores");
    cudaEvent_t ev[2];
    ck(cudaEventCreate(&ev[0]), "event");
    ck(cudaEventCreate(&ev[1]), "event");
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            cudaEventDestroy(e[0]);
            cudaEventDestroy(e[1]);
        }
    } evg{ev};

    double best_err = std::numeric_limits<double>::infinity();
    size_t best = n_reg;
    double n_diverged = 0.0, n_growth = 0.0, rom_ms = 0.0;
    std::vector<double> best_traj;
    for (size_t p0 = mine.first; p0 < mine.second; p0 += batch) {
        const size_t nb = std::min(batch, mine.second - p0);
        std::vector<double> hb(2 * nb);
        for (size_t k = 0; k < nb; ++k) {
            hb[k] = b1[(p0 + k) / n2];
            hb[nb + k] = b2[(p0 + k) % n2];
        }
        ck(cudaMemcpyAsync(betas, hb.data(), 2 * nb * sizeof(double), cudaMemcpyHostToDevice, c->stream), "betas");
        ck(rom::launch_systems(g, D, R, betas, betas + nb, static_cast<int>(nb), rhs, lhs, rhsb, c->stream),
           "systems");
        ck(cudaMemsetAsync(info, 0, 2 * nb * sizeof(int), c->stream), "memset");
        if (c->solver.spd_solve(lhs, D, static_cast<int>(nb), rhsb, R, info, c->stream, &err) != cudaSuccess) {
            fail(DOPINF_B200_ERR_DEVICE, err);
        }
        ck(cudaEventRecord(ev[0], c->stream), "event");
        ck(rom::launch_integrate(rhsb, R, qrows, NTP, static_cast<int>(nb), traj, c->stream), "integrate");
        ck(cudaEventRecord(ev[1], c->stream), "event");
        ck(rom::launch_score(traj, NTP, R, qrows, NT, static_cast<int>(nb), scores, c->stream), "score");
        std::vector<int> hinfo(2 * nb);
        std::vector<double> sc(nb * rom::kScoreFields);
        ck(cudaMemcpyAsync(hinfo.data(), info, hinfo.size() * sizeof(int), cudaMemcpyDeviceToHost, c->stream),
           "info D2H");
        ck(cudaMemcpyAsync(sc.data(), scores, sc.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
           "scores D2H");
        c->sync("grid search");
        float f = 0.0f;
        cudaEventElapsedTime(&f, ev[0], ev[1]);
        rom_ms += f;
        // pairs in index order, as the reference's loop (rom_search.cpp:214-225)
        for (size_t k = 0; k < nb; ++k) {
            if (hinfo[k] != 0 || hinfo[nb + k] != 0) {
                fail(DOPINF_B200_ERR_SOLVE, "positive definite solve failed (dposv info=" +
                                                std::to_string(hinfo[k] != 0 ? hinfo[k] : hinfo[nb + k]) + ")");
            }
            const double* o = &sc[k * rom::kScoreFields];
            double score = std::numeric_limits<double>::infinity();
            if (o[0] == 0.0) {
                n_diverged += 1.0;
            } else {
                if (o[3] >= 0.0) {
                    fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "training_error: reference row " +
                                                               std::to_string(static_cast<long long>(o[3])) +
                                                               " has zero norm");
                }
                if (o[4] != 0.0) {
                    fail(DOPINF_B200_ERR_INVALID_ARGUMENT,
                         "growth_ratio: training data is constant; deviation ratio undefined");
                }
                if (o[2] < max_growth) {
                    score = o[1];
                } else {
                    n_growth += 1.0;
                }
            }
            if (score < best_err) {
                best_err = score;
                best = p0 + k;
                best_traj.resize(nt_p * r);
                ck(cudaMemcpy(best_traj.data(), traj + k * nt_p * r, nt_p * r * sizeof(double),
                              cudaMemcpyDeviceToHost),
                   "trajectory D2H");
            }
        }
    }

    // agree on the winner across ranks (rom_search.cpp:227-261)
    GridOutcome out;
    double global_min = best_err;
    if (c->size > 1) {
        std::vector<double> v = {best_err};
        host_allreduce(c, v.data(), 1, ncclMin);
        global_min = v[0];
    }
    if (global_min == std::numeric_limits<double>::infinity()) {
        std::vector<double> counts = {n_diverged, n_growth};
        if (c->size > 1) host_allreduce(c, counts.data(), 2, ncclSum);
        fail(DOPINF_B200_ERR_NO_ADMISSIBLE_PAIR,
             "no admissible regularization pair among " + std::to_string(n_reg) + " candidates (" +
                 std::to_string(static_cast<long>(counts[0])) + " diverged, " +
                 std::to_string(static_cast<long>(counts[1])) + " exceeded growth bound " +
                 std::to_string(max_growth) + ")");
    }
    int owner = 0;
    if (c->size > 1) {
        std::vector<double> claim = {best_err == global_min ? static_cast<double>(c->rank)
                                                            : static_cast<double>(c->size)};
        host_allreduce(c, claim.data(), 1, ncclMin);
        owner = static_cast<int>(claim[0]);
    }
    std::vector<double> packet(3 + nt_p * r, 0.0);
    if (c->rank == owner) {
        packet[0] = b1[best / n2];
        packet[1] = b2[best % n2];
        packet[2] = rom_ms * 1e-3;
        std::copy(best_traj.begin(), best_traj.end(), packet.begin() + 3);
    }
    if (c->size > 1) {
        double* dp = c->rom_packet.get<double>(packet.size(), "packet");
        ck(cudaMemcpyAsync(dp, packet.data(), packet.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream),
           "packet H2D");
        ckn(ncclBroadcast(dp, dp, packet.size(), ncclFloat64, owner, c->comm, c->stream), "broadcast");
        ck(cudaMemcpyAsync(packet.data(), dp, packet.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
           "packet D2H");
        c->sync("broadcast");
    }
    out.beta1 = packet[0];
    out.beta2 = packet[1];
    out.rom_seconds = packet[2];
    out.train_err = global_min;
    out.owner = owner;
    if (traj_host) std::memcpy(traj_host, packet.data() + 3, nt_p * r * sizeof(double));
    return out;
}

// T_r operand: the caller's host T_r (uploaded) or, for tr_host == nullptr,
// the context's device T_r from dopinf_b200_reduced_map.
const double* tr_operand(dopinf_b200_ctx* c, const double* tr_host, size_t nt, size_t r) {
    if (!tr_host) {
        require(c->tr_dev_r > 0 && c->tr_dev_r == r && static_cast<size_t>(c->K) == nt,
                "no device T_r of this shape on the context (call dopinf_b200_reduced_map)");
        return c->tr_dev.get<double>(nt * r, "tr");
    }
    double* dtr = c->tr.get<double>(nt * r, "tr");
    ck(cudaMemcpyAsync(dtr, tr_host, nt * r * sizeof(double), cudaMemcpyHostToDevice, c->stream), "tr H2D");
    return dtr;
}

void do_project(dopinf_b200_ctx* c, const double* tr_host, const double* d_dev, size_t nt, size_t r,
                double* qhat_host) {
    require(r >= 1 && r <= nt, "project: r must lie in [1, nt]");
    const double* dtr = tr_operand(c, tr_host, nt, r);
    double* dq = c->qhat.get<double>(nt * r, "qhat");
    c->record(DOPINF_B200_STAGE_PROJECT, 0);
    ck(project::launch_project(dtr, d_dev, static_cast<int>(nt), static_cast<int>(r), dq, c->stream),
       "project");
    c->record(DOPINF_B200_STAGE_PROJECT, 1);
    c->qhat_r = r;
    c->qhat_nt = nt;
    if (qhat_host) c->d2h(qhat_host, dq, nt * r * sizeof(double), "qhat D2H");
}

// Φ_r = Q·T_r into b->phi (pitch basis_cols_pad(r), columns ≥ r zero);
// returns the pitch. T_r from the host, or the context's device T_r (NULL).
int do_basis(dopinf_b200_block* b, const double* tr, size_t r) {
    auto* c = b->ctx;
    require(r >= 1, "basis: bad map");
    materialize(b);
    const int r_pad = project::basis_cols_pad(static_cast<int>(r));
    // T_rᵀ, zero padded to r_pad rows, pitch = block pitch
    const double* dtr = tr_operand(c, tr, b->nt, r);
    double* dtrt = c->trt.get<double>(static_cast<size_t>(r_pad) * b->ld, "trt");
    ck(eig::launch_transpose_pad(dtr, static_cast<int>(b->nt), static_cast<int>(r), r_pad, b->ld, dtrt,
                                 c->stream),
       "T_r transpose");
    double* dphi = b->phi.get<double>(std::max<size_t>(b->rows, 1) * r_pad, "phi");
    b->phi_ld = r_pad;
    c->record(DOPINF_B200_STAGE_BASIS, 0);
    if (b->rows > 0) {
        ck(project::launch_basis(b->q, b->ld, static_cast<long long>(b->rows), static_cast<int>(b->nt), dtrt,
                                 b->ld, r_pad, dphi, c->num_sms, c->stream),
           "basis");
    }
    c->record(DOPINF_B200_STAGE_BASIS, 1);
    return r_pad;
}

// Field operands on the device: Q̃ (nt_p × r) padded to the Φ_r pitch with
// zeros, the means and (scaling) the scales of the transform.
struct FieldOperands {
    const double* qt = nullptr;
    const double* means = nullptr;
    const double* scales = nullptr;
    size_t nt_p = 0;
    int r_pad = 0;
};

FieldOperands field_operands(dopinf_b200_block* b, const double* qtilde, size_t r, size_t nt_p, int r_pad,
                             const double* means, const double* scales, bool scaling) {
    auto* c = b->ctx;
    FieldOperands f;
    f.nt_p = nt_p;
    f.r_pad = r_pad;
    double* dqt = c->field_qt.get<double>(nt_p * r_pad, "qtilde");
    ck(cudaMemsetAsync(dqt, 0, nt_p * r_pad * sizeof(double), c->stream), "memset");
    ck(cudaMemcpy2DAsync(dqt, r_pad * sizeof(double), qtilde, r * sizeof(double), r * sizeof(double), nt_p,
                         cudaMemcpyHostToDevice, c->stream),
       "qtilde H2D");
    f.qt = dqt;
    if (b->rows > 0) {
        double* dm = c->field_means.get<double>(b->rows, "field means");
        ck(cudaMemcpyAsync(dm, means, b->rows * sizeof(double), cudaMemcpyHostToDevice, c->stream), "means H2D");
        f.means = dm;
    }
    if (scaling) {
        double* ds = c->field_scales.get<double>(b->n_vars, "field scales");
        ck(cudaMemcpyAsync(ds, scales, b->n_vars * sizeof(double), cudaMemcpyHostToDevice, c->stream),
           "scales H2D");
        f.scales = ds;
    }
    return f;
}

// Field rows [row0, row0 + nrows) → out (pitch ldo). Widths beyond the
// kernel's resident Φ_r tile run as k-slabs accumulated in `out`, the inverse
// transform applied with the last one.
void do_field_rows(dopinf_b200_block* b, const FieldOperands& f, long long row0, long long nrows, double* out,
                   size_t ldo) {
    auto* c = b->ctx;
    const int slab = field::max_r_pad();
    const double* phi = static_cast<const double*>(b->phi.p) + static_cast<size_t>(row0) * f.r_pad;
    for (int k0 = 0; k0 < f.r_pad; k0 += slab) {
        const int w = std::min(slab, f.r_pad - k0);
        const bool last = k0 + w == f.r_pad;
        ck(field::launch_field(phi + k0, f.r_pad, f.qt + k0, f.r_pad, nrows, static_cast<int>(f.nt_p), w,
                               last && f.means ? f.means + row0 : nullptr, last ? f.scales : nullptr,
                               static_cast<long long>(b->nx_i), row0, out, ldo, k0 > 0 ? 1 : 0, c->num_sms,
                               c->stream),
           "field");
    }
}

void ensure_events(std::vector<cudaEvent_t>& v, size_t n) {
    while (v.size() < n) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        v.push_back(e);
    }
}

// rows × cols doubles, device pitch dev_ld → host pitch host_ld. Pinned
// destinations take one copy; pageable ones go through two pinned slots, the
// host copy of one slot overlapping the D2H of the next. Synchronous.
void d2h_2d(dopinf_b200_ctx* c, double* host, size_t host_ld, const double* dev, size_t dev_ld, size_t rows,
            size_t cols, const char* what) {
    if (rows == 0) return;
    if (is_pinned(host)) {
        ck(cudaMemcpy2DAsync(host, host_ld * sizeof(double), dev, dev_ld * sizeof(double), cols * sizeof(double),
                             rows, cudaMemcpyDeviceToHost, c->stream),
           what);
        ck(cudaStreamSynchronize(c->stream), what);
        return;
    }
    const size_t slot_rows = std::max<size_t>(1, (size_t(64) << 20) / (cols * sizeof(double)));
    auto* st = static_cast<double*>(c->staging.get(2 * slot_rows * cols * sizeof(double)));
    const size_t n = (rows + slot_rows - 1) / slot_rows;
    ensure_events(c->chunk_events2, 2);
    auto drain = [&](size_t k) {
        const size_t r0 = k * slot_rows, nr = std::min(slot_rows, rows - r0);
        ck(cudaEventSynchronize(c->chunk_events2[k % 2]), what);
        const double* src = st + (k % 2) * slot_rows * cols;
        if (host_ld == cols) {
            std::memcpy(host + r0 * cols, src, nr * cols * sizeof(double));
        } else {
            for (size_t i = 0; i < nr; ++i) std::memcpy(host + (r0 + i) * host_ld, src + i * cols, cols * sizeof(double));
        }
    };
    for (size_t k = 0; k < n; ++k) {
        const size_t r0 = k * slot_rows, nr = std::min(slot_rows, rows - r0);
        ck(cudaMemcpy2DAsync(st + (k % 2) * slot_rows * cols, cols * sizeof(double), dev + r0 * dev_ld,
                             dev_ld * sizeof(double), cols * sizeof(double), nr, cudaMemcpyDeviceToHost, c->stream),
           what);
        ck(cudaEventRecord(c->chunk_events2[k % 2], c->stream), "event");
        if (k > 0) drain(k - 1);
    }
    drain(n - 1);
}

// pwrite `bytes` at `off` from `src` on up to file_reader_threads() threads.
bool pwrite_parallel(int fd, const void* src, size_t bytes, uint64_t off) {
    auto write_all = [fd](const char* p, size_t n, uint64_t o) {
        while (n > 0) {
            const ssize_t w = pwrite(fd, p, n, static_cast<off_t>(o));
            if (w < 0 && errno == EINTR) continue;
            if (w <= 0) return false;
            p += w;
            n -= static_cast<size_t>(w);
            o += static_cast<uint64_t>(w);
        }
        return true;
    };
    constexpr size_t kPiece = size_t(8) << 20;
    const int n = static_cast<int>(std::min<size_t>(file_reader_threads(), (bytes + kPiece - 1) / kPiece));
    if (n <= 1) return write_all(static_cast<const char*>(src), bytes, off);
    const size_t per = (bytes / n + 4095) / 4096 * 4096;
    std::vector<std::thread> threads;
    std::vector<char> ok(n, 0);
    for (int i = 0; i < n; ++i) {
        const size_t b0 = std::min(bytes, per * i), b1 = std::min(bytes, per * (i + 1));
        threads.emplace_back([&, i, b0, b1] {
            ok[i] = write_all(static_cast<const char*>(src) + b0, b1 - b0, off + b0) ? 1 : 0;
        });
    }
    for (auto& t : threads) t.join();
    return std::all_of(ok.begin(), ok.end(), [](char v) { return v != 0; });
}

// Stream the field into an SNP1 file: chunk k is computed into device slot
// k % 2, copied (copy stream) into pinned slot k % 2, and written by the host
// while chunk k + 1 computes. Layout = data::write_snapshots (data.cpp:118-129):
// the field's rows are the variables' rows in order.
void write_field_file(dopinf_b200_block* b, const FieldOperands& f, const Snp1& h, const std::string& path) {
    auto* c = b->ctx;
    Fd fd;
    fd.fd = open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0644);
    if (fd.fd < 0) format_fail("cannot create snapshot file: " + path);
    std::string head("SNP1");
    for (uint64_t v : {h.n_vars, h.nx, h.nt}) head.append(reinterpret_cast<const char*>(&v), sizeof v);
    for (const auto& n : h.names) {
        const uint32_t len = static_cast<uint32_t>(n.size());
        head.append(reinterpret_cast<const char*>(&len), sizeof len);
        head += n;
    }
    if (!pwrite_parallel(fd.fd, head.data(), head.size(), 0)) format_fail("write failed: " + path);
    const uint64_t data_off = head.size();
    const size_t nt_p = f.nt_p, ldo = (nt_p + 1) / 2 * 2, rows = b->rows;
    size_t ch = std::max<size_t>(128, (size_t(256) << 20) / (nt_p * sizeof(double))) / 128 * 128;
    ch = std::min(ch, (rows + 127) / 128 * 128);
    const size_t n = (rows + ch - 1) / ch;
    double* dring = c->field_ring.get<double>(2 * ch * ldo, "field ring");
    auto* hring = static_cast<double*>(c->file_ring.get(2 * ch * nt_p * sizeof(double)));
    ensure_events(c->chunk_events, n + 1);
    ensure_events(c->chunk_events2, n + 1);
    cudaEvent_t* computed = c->chunk_events2.data();
    cudaEvent_t* copied = c->chunk_events.data();
    auto flush = [&](size_t k) {  // host: write chunk k from pinned slot k % 2
        const size_t r0 = k * ch, nr = std::min(ch, rows - r0);
        ck(cudaEventSynchronize(copied[k]), "field D2H");
        if (!pwrite_parallel(fd.fd, hring + (k % 2) * ch * nt_p, nr * nt_p * sizeof(double),
                             data_off + r0 * nt_p * sizeof(double))) {
            format_fail("write failed: " + path);
        }
    };
    c->record(DOPINF_B200_STAGE_FIELD, 0);
    for (size_t k = 0; k < n; ++k) {
        const size_t r0 = k * ch, nr = std::min(ch, rows - r0);
        double* dslot = dring + (k % 2) * ch * ldo;
        if (k >= 2) ck(cudaStreamWaitEvent(c->stream, copied[k - 2], 0), "event wait");  // slot drained
        do_field_rows(b, f, static_cast<long long>(r0), static_cast<long long>(nr), dslot, ldo);
        ck(cudaEventRecord(computed[k], c->stream), "event");
        ck(cudaStreamWaitEvent(c->copy_stream, computed[k], 0), "event wait");
        ck(cudaMemcpy2DAsync(hring + (k % 2) * ch * nt_p, nt_p * sizeof(double), dslot, ldo * sizeof(double),
                             nt_p * sizeof(double), nr, cudaMemcpyDeviceToHost, c->copy_stream),
           "field D2H");
        ck(cudaEventRecord(copied[k], c->copy_stream), "event");
        if (k > 0) flush(k - 1);  // pinned slot (k-1) % 2 is reused by chunk k + 1
    }
    if (n > 0) flush(n - 1);
    c->record(DOPINF_B200_STAGE_FIELD, 1);
    if (close(fd.fd) != 0) {
        fd.fd = -1;
        format_fail("write failed: " + path);
    }
    fd.fd = -1;
}


}  // namespace

extern "C" {

int dopinf_b200_abi_version(void) { return DOPINF_B200_ABI_VERSION; }

uint64_t dopinf_b200_kernel_launches(void) { return g_launches.load(); }

const char* dopinf_b200_status_string(int status) {
    switch (status) {
        case DOPINF_B200_OK: return "ok";
        case DOPINF_B200_ERR_INVALID_ARGUMENT: return "InvalidArgumentError";
        case DOPINF_B200_ERR_PARTITION: return "PartitionError";
        case DOPINF_B200_ERR_COLLECTIVE: return "CollectiveError";
        case DOPINF_B200_ERR_DEGENERATE_VARIABLE: return "DegenerateVariableError";
        case DOPINF_B200_ERR_DEVICE: return "DeviceError";
        case DOPINF_B200_ERR_OUT_OF_MEMORY: return "OutOfMemoryError";
        case DOPINF_B200_ERR_NOT_PSD: return "NotPsdError";
        case DOPINF_B200_ERR_RANK_DEFICIENCY: return "RankDeficiencyError";
        case DOPINF_B200_ERR_SOLVE: return "SolveError";
        case DOPINF_B200_ERR_DATA_FORMAT: return "DataFormatError";
        case DOPINF_B200_ERR_NO_ADMISSIBLE_PAIR: return "NoAdmissiblePairError";
        default: return "unknown status";
    }
}

int dopinf_b200_get_unique_id(unsigned char* id) {
    if (!id) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    static_assert(sizeof(ncclUniqueId) == DOPINF_B200_UNIQUE_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId uid;
    if (ncclGetUniqueId(&uid) != ncclSuccess) return DOPINF_B200_ERR_COLLECTIVE;
    std::memcpy(id, &uid, sizeof uid);
    return DOPINF_B200_OK;
}

int dopinf_b200_ctx_create(int device, int rank, int size, const unsigned char* id,
                           dopinf_b200_ctx** out) {
    if (!out || size < 1 || rank < 0 || rank >= size || (size > 1 && !id)) {
        return DOPINF_B200_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    auto* c = new (std::nothrow) dopinf_b200_ctx;
    if (!c) return DOPINF_B200_ERR_OUT_OF_MEMORY;
    c->device = device;
    c->rank = rank;
    c->size = size;
    const int rc = guarded(c, [&] {
        int ndev = 0;
        ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
        if (device < 0 || device >= ndev) {
            fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "device " + std::to_string(device) + " not present");
        }
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10 || prop.minor != 0) {
            fail(DOPINF_B200_ERR_DEVICE, std::string("device is ") + prop.name +
                                             " (sm_" + std::to_string(prop.major) + std::to_string(prop.minor) +
                                             "); this build targets sm_100a (B200) only");
        }
        c->num_sms = prop.multiProcessorCount;
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
        for (auto& pair : c->ev) {
            ck(cudaEventCreate(&pair[0]), "cudaEventCreate");
            ck(cudaEventCreate(&pair[1]), "cudaEventCreate");
        }
        if (size > 1) {
            ncclUniqueId uid;
            std::memcpy(&uid, id, sizeof uid);
            ckn(ncclCommInitRank(&c->comm, size, uid, rank), "ncclCommInitRank");
        }
    });
    if (rc != DOPINF_B200_OK) {
        std::fprintf(stderr, "dopinf_b200_ctx_create: %s\n", c->err.c_str());
        dopinf_b200_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return DOPINF_B200_OK;
}

void dopinf_b200_ctx_destroy(dopinf_b200_ctx* c) {
    if (!c) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm) ncclCommDestroy(c->comm);
    for (auto& pair : c->ev) {
        if (pair[0]) cudaEventDestroy(pair[0]);
        if (pair[1]) cudaEventDestroy(pair[1]);
    }
    for (DBuf* b : {&c->tiles, &c->work, &c->counters, &c->packed, &c->gather, &c->dmat, &c->dhost_in,
                    &c->scales, &c->tr, &c->trt, &c->qhat, &c->sel, &c->rows_out, &c->span, &c->eig_a,
                    &c->eig_w, &c->eig_work, &c->eig_info, &c->eig_v, &c->eig_lambda, &c->tr_dev, &c->field_qt,
                    &c->field_means, &c->field_scales, &c->field_ring, &c->rom_qhat, &c->rom_dhat, &c->rom_q2t,
                    &c->rom_qrows, &c->rom_rhs, &c->rom_g, &c->rom_lhs, &c->rom_rhsb, &c->rom_betas, &c->rom_traj,
                    &c->rom_scores, &c->rom_work, &c->rom_info, &c->rom_tiles, &c->rom_gwork, &c->rom_counters,
                    &c->rom_packed, &c->rom_packet}) {
        b->release();
    }
    c->staging.release();
    c->file_ring.release();
    c->gv.release();
    c->ring.release();
    for (cudaEvent_t e : c->chunk_events) cudaEventDestroy(e);
    for (cudaEvent_t e : c->chunk_events2) cudaEventDestroy(e);
    for (cudaEvent_t e : c->timing_events) cudaEventDestroy(e);
    if (c->copy_stream) {
        cudaStreamSynchronize(c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    if (c->stream) cudaStreamDestroy(c->stream);
    cudaSetDevice(prev);
    delete c;
}

int dopinf_b200_ctx_rank(const dopinf_b200_ctx* c) { return c ? c->rank : -1; }
int dopinf_b200_ctx_size(const dopinf_b200_ctx* c) { return c ? c->size : -1; }
const char* dopinf_b200_last_error(const dopinf_b200_ctx* c) { return c ? c->err.c_str() : g_thread_err.c_str(); }
void* dopinf_b200_ctx_stream(dopinf_b200_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int dopinf_b200_set_gram_reduce(dopinf_b200_ctx* c, int mode) {
    return guarded(c, [&] {
        require(mode == DOPINF_B200_GRAM_REDUCE_ORDERED || mode == DOPINF_B200_GRAM_REDUCE_NCCL,
                "set_gram_reduce: unknown mode");
        c->gram_reduce = mode;
    });
}

int dopinf_b200_allreduce(dopinf_b200_ctx* c, double* data, size_t count, int op) {
    return guarded(c, [&] {
        require(op >= DOPINF_B200_SUM && op <= DOPINF_B200_MIN, "allreduce: unknown op");
        require(count == 0 || data, "allreduce: null data");
        if (c->size == 1 || count == 0) return;
        double* buf = c->span.get<double>(count * (op == DOPINF_B200_SUM ? c->size + 1 : 1), "span");
        ck(cudaMemcpyAsync(buf, data, count * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
        if (op == DOPINF_B200_SUM) {
            // Ascending-rank order, as the reference's in-process backend sums.
            double* parts = buf + count;
            ckn(ncclAllGather(buf, parts, count, ncclFloat64, c->comm, c->stream), "allgather");
            ck(gram::launch_ordered_sum(parts, c->size, count, buf, c->stream), "ordered sum");
        } else {
            ckn(ncclAllReduce(buf, buf, count, ncclFloat64, op == DOPINF_B200_MAX ? ncclMax : ncclMin,
                              c->comm, c->stream),
                "allreduce");
        }
        ck(cudaMemcpyAsync(data, buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
        c->sync("allreduce");
    });
}

int dopinf_b200_barrier(dopinf_b200_ctx* c) {
    double one = 1.0;
    return dopinf_b200_allreduce(c, &one, 1, DOPINF_B200_MAX);
}

int dopinf_b200_stage_ms(const dopinf_b200_ctx* c, int stage, double* ms) {
    if (!c || !ms || stage < 0 || stage >= DOPINF_B200_STAGE_COUNT) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    *ms = 0.0;
    if (stage == DOPINF_B200_STAGE_STREAM_GRAM) {
        *ms = c->stream_gram_ms();
        return DOPINF_B200_OK;
    }
    if (!c->ev_done[stage]) return DOPINF_B200_OK;
    float f = 0.0f;
    if (cudaEventSynchronize(c->ev[stage][1]) != cudaSuccess ||
        cudaEventElapsedTime(&f, c->ev[stage][0], c->ev[stage][1]) != cudaSuccess) {
        return DOPINF_B200_ERR_DEVICE;
    }
    *ms = f;
    return DOPINF_B200_OK;
}

int dopinf_b200_partition_rows(size_t nx, int p, size_t* begin, size_t* end) {
    // data.cpp:86-103
    if (p < 1 || static_cast<size_t>(p) > nx) return DOPINF_B200_ERR_PARTITION;
    if (!begin || !end) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    const size_t ranks = static_cast<size_t>(p);
    const size_t base = nx / ranks;
    for (size_t r = 0; r < ranks; ++r) {
        begin[r] = r * base;
        end[r] = (r + 1 == ranks) ? nx : (r + 1) * base;
    }
    return DOPINF_B200_OK;
}

int dopinf_b200_block_create(dopinf_b200_ctx* c, size_t n_vars, size_t nx_i, size_t row_begin, size_t nt,
                             dopinf_b200_block** out) {
    if (!out) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    auto* b = new (std::nothrow) dopinf_b200_block;
    if (!b) return DOPINF_B200_ERR_OUT_OF_MEMORY;
    const int rc = guarded(c, [&] {
        require(n_vars >= 1 && nt >= 1, "block_create: n_vars and nt must be >= 1");
        require(nt <= (1u << 20), "block_create: nt too large");
        b->ctx = c;
        b->n_vars = n_vars;
        b->nx_i = nx_i;
        b->row_begin = row_begin;
        b->nt = nt;
        b->ld = (nt + 1) / 2 * 2;  // 16-byte rows for TMA and 128-bit accesses
        b->rows = n_vars * nx_i;
        if (b->rows > 0) {
            ck(cudaMalloc(&b->q, b->rows * b->ld * sizeof(double)), "block values");
            if (b->ld != nt) {
                ck(cudaMemsetAsync(b->q, 0, b->rows * b->ld * sizeof(double), c->stream), "memset");
            }
        }
        b->varmax.get<double>(n_vars, "varmax");
        c->sync("block_create");
    });
    if (rc != DOPINF_B200_OK) {
        if (b->q) cudaFree(b->q);
        delete b;
        return rc;
    }
    *out = b;
    return DOPINF_B200_OK;
}

void dopinf_b200_block_destroy(dopinf_b200_block* b) {
    if (!b) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(b->ctx->device);
    cudaStreamSynchronize(b->ctx->stream);
    if (b->q) cudaFree(b->q);
    b->means.release();
    b->varmax.release();
    b->phi.release();
    b->field.release();
    cudaSetDevice(prev);
    delete b;
}

int dopinf_b200_block_upload(dopinf_b200_block* b, const double* host, size_t host_ld) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(host_ld >= b->nt && (b->rows == 0 || host), "block_upload: bad host buffer");
        c->record(DOPINF_B200_STAGE_UPLOAD, 0);
        if (b->rows > 0) {
            if (host_ld == b->ld) {
                ck(cudaMemcpyAsync(b->q, host, b->rows * b->ld * sizeof(double), cudaMemcpyHostToDevice,
                                   c->stream),
                   "upload");
            } else {
                ck(cudaMemcpy2DAsync(b->q, b->ld * sizeof(double), host, host_ld * sizeof(double),
                                     b->nt * sizeof(double), b->rows, cudaMemcpyHostToDevice, c->stream),
                   "upload");
            }
        }
        c->record(DOPINF_B200_STAGE_UPLOAD, 1);
        b->pending_center = false;
        b->stats_valid = false;
        c->sync("block_upload");
    });
}

int dopinf_b200_block_download(dopinf_b200_block* b, double* host, size_t host_ld) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(host_ld >= b->nt && (b->rows == 0 || host), "block_download: bad host buffer");
        materialize(b);
        c->record(DOPINF_B200_STAGE_DOWNLOAD, 0);
        if (b->rows > 0) {
            ck(cudaMemcpy2DAsync(host, host_ld * sizeof(double), b->q, b->ld * sizeof(double),
                                 b->nt * sizeof(double), b->rows, cudaMemcpyDeviceToHost, c->stream),
               "download");
        }
        c->record(DOPINF_B200_STAGE_DOWNLOAD, 1);
        c->sync("block_download");
    });
}

int dopinf_b200_block_device(dopinf_b200_block* b, double** values, size_t* ld) {
    if (!b || !values || !ld) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    return guarded(b->ctx, [&] {
        materialize(b);
        b->ctx->sync("block_device");
        b->stats_valid = false;  // the caller may write through the pointer
        *values = b->q;
        *ld = b->ld;
    });
}

int dopinf_b200_block_synth_oscillator(dopinf_b200_block* b, uint64_t seed, int n_modes, double dt,
                                       double noise, const double* amps) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        if (b->rows == 0) return;
        ck(synth::oscillator(b->q, b->ld, static_cast<long long>(b->rows), static_cast<int>(b->nt),
                             static_cast<long long>(b->nx_i), static_cast<long long>(b->row_begin),
                             static_cast<int>(b->n_vars), seed, n_modes, dt, noise, amps, c->num_sms,
                             c->stream),
           "synth");
        b->pending_center = false;
        b->stats_valid = false;
        c->sync("synth");
    });
}

int dopinf_b200_block_synth_lowrank(dopinf_b200_block* b, uint64_t seed, int rank, double amplitude) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        if (b->rows == 0) return;
        ck(synth::lowrank(b->q, b->ld, static_cast<long long>(b->rows), static_cast<int>(b->nt),
                          static_cast<long long>(b->nx_i), static_cast<long long>(b->row_begin), seed, rank,
                          amplitude, c->num_sms, c->stream),
           "synth");
        b->pending_center = false;
        b->stats_valid = false;
        c->sync("synth");
    });
}

int dopinf_b200_center(dopinf_b200_block* b, double* means) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    return guarded(b->ctx, [&] {
        if (b->rows > 0) do_center(b, means);
        b->ctx->sync("center");
    });
}

int dopinf_b200_global_scales(dopinf_b200_block* b, double* scales, size_t* degenerate_var) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    return guarded(b->ctx, [&] { do_global_scales(b, scales, degenerate_var); });
}

int dopinf_b200_scale(dopinf_b200_block* b, const double* scales) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    return guarded(b->ctx, [&] {
        require(scales != nullptr, "scale: null scales");
        if (b->rows > 0) do_scale(b, scales);
        b->ctx->sync("scale");
    });
}

int dopinf_b200_local_gram(dopinf_b200_block* b, double* d) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    return guarded(b->ctx, [&] {
        do_local_gram(b, d);
        b->ctx->sync("local_gram");
    });
}

int dopinf_b200_global_gram(dopinf_b200_ctx* c, double* d) {
    return guarded(c, [&] {
        do_global_gram(c, d);
        c->sync("global_gram");
    });
}

int dopinf_b200_project(dopinf_b200_ctx* c, const double* tr, size_t nt, size_t r, double* qhat) {
    return guarded(c, [&] {
        require(qhat != nullptr, "project: null buffers");
        require(c->have_gram && static_cast<size_t>(c->K) == nt,
                "project: no Gram of matching size on this context");
        do_project(c, tr, c->dmat.get<double>(nt * nt, "D"), nt, r, qhat);
        c->sync("project");
    });
}

int dopinf_b200_project_host(dopinf_b200_ctx* c, const double* tr, const double* d, size_t nt, size_t r,
                             double* qhat) {
    return guarded(c, [&] {
        require(tr && d && qhat, "project: null buffers");
        double* dd = c->dhost_in.get<double>(nt * nt, "D in");
        ck(cudaMemcpyAsync(dd, d, nt * nt * sizeof(double), cudaMemcpyHostToDevice, c->stream), "D H2D");
        do_project(c, tr, dd, nt, r, qhat);
        c->sync("project");
    });
}

int dopinf_b200_set_gram(dopinf_b200_ctx* c, const double* d, size_t nt) {
    return guarded(c, [&] {
        require(d != nullptr && nt >= 1 && nt <= (1u << 16), "set_gram: bad matrix");
        const size_t nn = nt * nt;
        ck(cudaMemcpyAsync(c->dmat.get<double>(nn, "D"), d, nn * sizeof(double), cudaMemcpyHostToDevice, c->stream),
           "D H2D");
        c->K = static_cast<int>(nt);
        c->have_gram = true;
        c->eig_K = 0;
        c->tr_dev_r = 0;
        c->sync("set_gram");
    });
}

int dopinf_b200_eig_sym_desc(dopinf_b200_ctx* c, double* lambda, double* vectors) {
    return guarded(c, [&] {
        require(c->have_gram && c->K > 0, "eig_sym_desc: no Gram on this context");
        const int n = c->K;
        const size_t nn = static_cast<size_t>(n) * n;
        std::string err;
        const size_t lwork = c->solver.workspace_doubles(n, &err);
        if (!err.empty()) fail(DOPINF_B200_ERR_DEVICE, "eig_sym_desc: " + err);
        double* a = c->eig_a.get<double>(nn, "eig scratch");
        double* w = c->eig_w.get<double>(n, "eig w");
        double* work = c->eig_work.get<double>(std::max<size_t>(lwork, 1), "eig work");
        int* info = c->eig_info.get<int>(1, "eig info");
        double* v = c->eig_v.get<double>(nn, "eig vectors");
        double* lam = c->eig_lambda.get<double>(n, "eig lambda");
        c->eig_K = 0;
        c->tr_dev_r = 0;
        if (c->solver.run(c->dmat.get<double>(nn, "D"), n, a, w, work, lwork, info, v, lam, c->stream, &err) !=
            cudaSuccess) {
            fail(DOPINF_B200_ERR_DEVICE, "eig_sym_desc: " + (err.empty() ? std::string("cuSOLVER failure") : err));
        }
        int hinfo = 0;
        std::vector<double> hl(n);
        c->d2h(&hinfo, info, sizeof(int), "info D2H");
        c->d2h(hl.data(), lam, n * sizeof(double), "lambda D2H");
        if (hinfo != 0) fail(DOPINF_B200_ERR_SOLVE, "symmetric eigendecomposition failed (dsyevd info=" +
                                                         std::to_string(hinfo) + ")");
        // pod.cpp:35-48: clamp round-off negatives, reject real ones.
        const double lambda1 = hl.empty() ? 0.0 : hl.front();
        if (lambda1 < 0.0) {
            fail(DOPINF_B200_ERR_NOT_PSD, "Gram matrix is not positive semidefinite (largest eigenvalue is negative)");
        }
        const double clamp = 1e-10 * lambda1;
        bool changed = false;
        for (double& l : hl) {
            if (l < -clamp) {
                fail(DOPINF_B200_ERR_NOT_PSD, "Gram matrix has eigenvalue " + std::to_string(l) +
                                                  " below the round-off clamp; data is corrupted");
            }
            if (l < 0.0) {
                l = 0.0;
                changed = true;
            }
        }
        if (changed) {
            ck(cudaMemcpyAsync(lam, hl.data(), n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "lambda H2D");
        }
        if (lambda) std::memcpy(lambda, hl.data(), n * sizeof(double));
        if (vectors) c->d2h(vectors, v, nn * sizeof(double), "vectors D2H");
        c->sync("eig_sym_desc");
        c->eig_K = n;
    });
}

int dopinf_b200_reduced_map(dopinf_b200_ctx* c, size_t r, double* tr) {
    return guarded(c, [&] {
        require(c->eig_K > 0 && c->eig_K == c->K, "reduced_map: no eigendecomposition on this context");
        const size_t n = static_cast<size_t>(c->eig_K);
        require(r >= 1 && r <= n, "reduced_map: r must lie in [1, nt]");
        double lam_r = 0.0;
        c->d2h(&lam_r, c->eig_lambda.get<double>(n, "eig lambda") + (r - 1), sizeof(double), "lambda D2H");
        if (!(lam_r > 0.0)) {
            fail(DOPINF_B200_ERR_RANK_DEFICIENCY,
                 "reduced dimension " + std::to_string(r) + " exceeds the numerical rank of the data");
        }
        double* dtr = c->tr_dev.get<double>(n * r, "device T_r");
        ck(eig::launch_reduced_map(c->eig_v.get<double>(n * n, "eig vectors"), c->eig_lambda.get<double>(n, "lambda"),
                                   static_cast<int>(n), static_cast<int>(r), dtr, c->stream),
           "reduced_map");
        c->tr_dev_r = r;
        if (tr) c->d2h(tr, dtr, n * r * sizeof(double), "T_r D2H");
        c->sync("reduced_map");
    });
}

int dopinf_b200_basis(dopinf_b200_block* b, const double* tr, size_t r, double* phi) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        const int r_pad = do_basis(b, tr, r);
        if (phi && b->rows > 0) {
            c->record(DOPINF_B200_STAGE_DOWNLOAD, 0);
            ck(cudaMemcpy2DAsync(phi, r * sizeof(double), b->phi.p, r_pad * sizeof(double), r * sizeof(double),
                                 b->rows, cudaMemcpyDeviceToHost, c->stream),
               "phi D2H");
            c->record(DOPINF_B200_STAGE_DOWNLOAD, 1);
        }
        c->sync("basis");  // trt host staging must outlive the copy
    });
}

int dopinf_b200_basis_device(dopinf_b200_block* b, double** phi, size_t* ld) {
    if (!b || !phi || !ld) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    return guarded(b->ctx, [&] {
        require(b->phi_ld > 0, "basis_device: no basis computed");
        *phi = static_cast<double*>(b->phi.p);
        *ld = static_cast<size_t>(b->phi_ld);
    });
}

int dopinf_b200_grid_search(dopinf_b200_ctx* c, const double* qhat, size_t r, size_t nt, const double* b1,
                            size_t n1, const double* b2, size_t n2, double max_growth, size_t nt_p,
                            double* pair_opt, double* train_err, int* owner, double* rom_seconds,
                            double* trajectory) {
    return guarded(c, [&] {
        const GridOutcome o = do_grid_search(c, qhat, r, nt, b1, n1, b2, n2, max_growth, nt_p, trajectory);
        if (pair_opt) {
            pair_opt[0] = o.beta1;
            pair_opt[1] = o.beta2;
        }
        if (train_err) *train_err = o.train_err;
        if (owner) *owner = o.owner;
        if (rom_seconds) *rom_seconds = o.rom_seconds;
    });
}

int dopinf_b200_rom_integrate(dopinf_b200_ctx* c, const double* a, const double* f, const double* cvec, size_t r,
                              const double* q0, size_t n_steps, double* traj, int* finite) {
    return guarded(c, [&] {
        if (n_steps < 1) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "integrate: need at least one step");
        require(r >= 1 && r <= 180, "integrate: r must lie in [1, 180]");
        require(a && f && cvec && q0, "integrate: null operator");
        const size_t s = r * (r + 1) / 2, d = r + s + 1;
        // the solve's layout: column i = [A_i, F_i, c_i] (column-major d × r)
        std::vector<double> x(d * r);
        for (size_t i = 0; i < r; ++i) {
            std::memcpy(&x[i * d], a + i * r, r * sizeof(double));
            std::memcpy(&x[i * d + r], f + i * s, s * sizeof(double));
            x[i * d + r + s] = cvec[i];
        }
        double* dx = c->rom_rhsb.get<double>(d * r, "operators");
        double* dq0 = c->rom_qrows.get<double>(r, "q0");
        double* dt = c->rom_traj.get<double>(n_steps * r, "trajectory");
        ck(cudaMemcpyAsync(dx, x.data(), x.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream), "ops H2D");
        ck(cudaMemcpyAsync(dq0, q0, r * sizeof(double), cudaMemcpyHostToDevice, c->stream), "q0 H2D");
        ck(rom::launch_integrate(dx, static_cast<int>(r), dq0, static_cast<int>(n_steps), 1, dt, c->stream),
           "integrate");
        std::vector<double> h(n_steps * r);
        ck(cudaMemcpyAsync(h.data(), dt, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
        c->sync("integrate");
        if (traj) std::memcpy(traj, h.data(), h.size() * sizeof(double));
        if (finite) *finite = std::all_of(h.begin(), h.end(), [](double v) { return std::isfinite(v); }) ? 1 : 0;
    });
}

int dopinf_b200_reconstruct_field(dopinf_b200_block* b, const double* tr, size_t r, const double* qtilde,
                                  size_t nt_p, const double* means, const double* scales, int scaling,
                                  double* field) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(qtilde != nullptr && nt_p >= 1, "reconstruct_field: null or empty trajectory");
        require(b->rows == 0 || means != nullptr, "reconstruct_field: null means");
        require(!scaling || scales != nullptr, "reconstruct_field: null scales");
        const int r_pad = do_basis(b, tr, r);
        const FieldOperands f = field_operands(b, qtilde, r, nt_p, r_pad, means, scales, scaling != 0);
        const size_t ldo = (nt_p + 1) / 2 * 2;
        double* out = b->field.get<double>(std::max<size_t>(b->rows, 1) * ldo, "field");
        b->field_ld = ldo;
        c->record(DOPINF_B200_STAGE_FIELD, 0);
        if (b->rows > 0) do_field_rows(b, f, 0, static_cast<long long>(b->rows), out, ldo);
        c->record(DOPINF_B200_STAGE_FIELD, 1);
        if (field && b->rows > 0) {
            c->record(DOPINF_B200_STAGE_DOWNLOAD, 0);
            d2h_2d(c, field, nt_p, out, ldo, b->rows, nt_p, "field D2H");
            c->record(DOPINF_B200_STAGE_DOWNLOAD, 1);
        }
        c->sync("reconstruct_field");
    });
}

int dopinf_b200_field_device(dopinf_b200_block* b, double** field, size_t* ld) {
    if (!b || !field || !ld) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    return guarded(b->ctx, [&] {
        require(b->field_ld > 0, "field_device: no field reconstructed");
        *field = static_cast<double*>(b->field.p);
        *ld = b->field_ld;
    });
}

int dopinf_b200_write_field(dopinf_b200_block* b, const double* tr, size_t r, const double* qtilde, size_t nt_p,
                            const double* means, const double* scales, int scaling, const char* names,
                            const char* path) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(names != nullptr && path != nullptr, "write_field: null names or path");
        require(qtilde != nullptr, "write_field: null trajectory");
        require(b->rows == 0 || means != nullptr, "write_field: null means");
        require(!scaling || scales != nullptr, "write_field: null scales");
        // the header write_snapshots would write (pipeline.cpp:333-337), same checks (data.cpp:105-107)
        Snp1 h;
        h.n_vars = b->n_vars;
        h.nx = b->nx_i;
        h.nt = nt_p;
        for (const char* p = names; h.names.size() < b->n_vars; p += h.names.back().size() + 1) {
            h.names.emplace_back(p);
        }
        validate_snp1(h);
        const int r_pad = do_basis(b, tr, r);
        const FieldOperands f = field_operands(b, qtilde, r, nt_p, r_pad, means, scales, scaling != 0);
        write_field_file(b, f, h, path);
    });
}

int dopinf_b200_basis_rows(dopinf_b200_block* b, const double* tr, size_t r, const size_t* rows, size_t nsel,
                           double* out) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(tr != nullptr && r >= 1, "basis_rows: bad map");
        require(nsel == 0 || (rows && out), "basis_rows: null buffers");
        std::vector<long long> sel(nsel);
        for (size_t k = 0; k < nsel; ++k) {
            if (rows[k] >= b->rows) {
                fail(DOPINF_B200_ERR_INVALID_ARGUMENT,
                     "basis_rows: row " + std::to_string(rows[k]) + " outside the local block");
            }
            sel[k] = static_cast<long long>(rows[k]);
        }
        if (nsel == 0) return;
        materialize(b);
        double* dtr = c->tr.get<double>(b->nt * r, "tr");
        long long* dsel = c->sel.get<long long>(nsel, "sel");
        double* dout = c->rows_out.get<double>(nsel * r, "rows out");
        ck(cudaMemcpyAsync(dtr, tr, b->nt * r * sizeof(double), cudaMemcpyHostToDevice, c->stream), "tr H2D");
        ck(cudaMemcpyAsync(dsel, sel.data(), nsel * sizeof(long long), cudaMemcpyHostToDevice, c->stream),
           "rows H2D");
        ck(project::launch_basis_rows(b->q, b->ld, static_cast<int>(b->nt), dtr, static_cast<int>(r), dsel,
                                      static_cast<int>(nsel), dout, c->stream),
           "basis_rows");
        ck(cudaMemcpyAsync(out, dout, nsel * r * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
        c->sync("basis_rows");
    });
}

int dopinf_b200_snapshot_pass(dopinf_b200_block* b, int scaling, double* means, double* scales, double* d) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        if (b->rows > 0) do_center(b, means);
        if (scaling) {
            std::vector<double> s(b->n_vars);
            do_global_scales(b, s.data(), nullptr);
            if (scales) std::memcpy(scales, s.data(), s.size() * sizeof(double));
            if (b->rows > 0) do_scale(b, s.data());
            c->sync("snapshot_pass");  // host scales must outlive the async upload
        }
        do_local_gram(b, nullptr);
        do_global_gram(c, d);
        c->sync("snapshot_pass");
    });
}

int dopinf_b200_snapshot_pass_host(dopinf_b200_block* b, const double* host, size_t host_ld, int scaling,
                                   double* means, double* scales, double* d) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(host_ld >= b->nt && (b->rows == 0 || host), "snapshot_pass_host: bad host buffer");
        StreamSource src;
        src.host = host;
        src.host_ld = host_ld;
        do_stream_pass(b, src, scaling != 0, means, scales);
        unpack(c);
        do_global_gram(c, d);
        c->sync("snapshot_pass_host");
    });
}

int dopinf_b200_snp1_header(const char* path, uint64_t* dims, char* names, size_t names_cap,
                            size_t* names_len) {
    return guarded_free([&] {
        require(path && dims, "snp1_header: null path or dims");
        Fd f;
        open_snp1(f, path);
        const Snp1 h = read_snp1_header(f.fd, path);
        dims[0] = h.n_vars;
        dims[1] = h.nx;
        dims[2] = h.nt;
        dims[3] = h.data_offset;
        size_t need = 0;
        for (const auto& n : h.names) need += n.size() + 1;
        if (names_len) *names_len = need;
        if (names) {
            require(names_cap >= need, "snp1_header: names buffer too small");
            size_t at = 0;
            for (const auto& n : h.names) {
                std::memcpy(names + at, n.c_str(), n.size() + 1);
                at += n.size() + 1;
            }
        }
    });
}

}  // extern "C"

namespace {

// Open + validate the file and create the device block of rows
// [row_begin, row_end) of every variable (pipeline.cpp:254-258).
dopinf_b200_block* open_file_block(dopinf_b200_ctx* c, const char* path, size_t row_begin, size_t row_end,
                                   Fd& f, Snp1& h) {
    require(path != nullptr, "null path");
    open_snp1(f, path);
    h = read_snp1_header(f.fd, path);
    if (row_begin > row_end || row_end > h.nx) {
        fail(DOPINF_B200_ERR_PARTITION, "read_block: rows [" + std::to_string(row_begin) + ", " +
                                            std::to_string(row_end) + ") outside the file's " +
                                            std::to_string(h.nx) + " rows");
    }
    require(h.nt <= (1u << 20), "snapshot file: nt too large");
    dopinf_b200_block* b = nullptr;
    const int rc = dopinf_b200_block_create(c, h.n_vars, row_end - row_begin, row_begin, h.nt, &b);
    if (rc != DOPINF_B200_OK) fail(rc, c->err);
    return b;
}

}  // namespace

extern "C" {

int dopinf_b200_block_read(dopinf_b200_ctx* c, const char* path, size_t row_begin, size_t row_end,
                           dopinf_b200_block** out) {
    if (!out) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    dopinf_b200_block* b = nullptr;
    const int rc = guarded(c, [&] {
        Fd f;
        Snp1 h;
        b = open_file_block(c, path, row_begin, row_end, f, h);
        StreamSource src;
        src.fd = f.fd;
        src.file = &h;
        const std::string p(path);
        src.path = &p;
        do_block_read(b, src);
        c->sync("block_read");
    });
    if (rc != DOPINF_B200_OK) {
        dopinf_b200_block_destroy(b);
        return rc;
    }
    *out = b;
    return DOPINF_B200_OK;
}

int dopinf_b200_snapshot_pass_file(dopinf_b200_ctx* c, const char* path, size_t row_begin, size_t row_end,
                                   int scaling, dopinf_b200_block** out, double* means, double* scales,
                                   double* d) {
    if (!out) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    dopinf_b200_block* b = nullptr;
    const int rc = guarded(c, [&] {
        Fd f;
        Snp1 h;
        b = open_file_block(c, path, row_begin, row_end, f, h);
        StreamSource src;
        src.fd = f.fd;
        src.file = &h;
        const std::string p(path);
        src.path = &p;
        do_stream_pass(b, src, scaling != 0, means, scales);
        unpack(c);
        do_global_gram(c, d);
        c->sync("snapshot_pass_file");
    });
    if (rc != DOPINF_B200_OK) {
        dopinf_b200_block_destroy(b);
        return rc;
    }
    *out = b;
    return DOPINF_B200_OK;
}

int dopinf_b200_stream_pass_synth(dopinf_b200_ctx* c, size_t n_vars, size_t nx_i, size_t row_begin, size_t nt,
                                  uint64_t seed, int n_modes, double dt, double noise, const double* amps,
                                  int scaling, double* means, double* scales, double* d) {
    return guarded(c, [&] {
        require(n_vars >= 1 && nt >= 1 && nt <= (1u << 20), "stream_pass_synth: bad shape");
        require(n_modes >= 1 && n_modes <= 128, "stream_pass_synth: n_modes must lie in [1, 128]");
        // A block that is never resident: means/varmax live on the device, values stream through a ring.
        dopinf_b200_block view;
        view.ctx = c;
        view.n_vars = n_vars;
        view.nx_i = nx_i;
        view.row_begin = row_begin;
        view.nt = nt;
        view.ld = (nt + 1) / 2 * 2;
        view.rows = n_vars * nx_i;
        struct Release {
            dopinf_b200_block& b;
            ~Release() {
                cudaStreamSynchronize(b.ctx->stream);
                b.means.release();
                b.varmax.release();
            }
        } release{view};
        StreamSource src;
        src.synth = true;
        src.seed = seed;
        src.n_modes = n_modes;
        src.dt = dt;
        src.noise = noise;
        src.amps = amps;
        do_stream_pass(&view, src, scaling != 0, means, scales);
        unpack(c);
        do_global_gram(c, d);
        c->sync("stream_pass_synth");
    });
}

}  // extern "C"
