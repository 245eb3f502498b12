// capi_coll.cu — the collective layer of the C ABI: every NCCL call of the
// library goes through here, so the reference group semantics hold for all of
// them (paths relative to /root/reference/proj):
//
//   * a deadline on every wait for a queued collective (comm_inprocess.cpp:
//     50-63, kTimeout = 60 s): while the stream holds an unfinished
//     collective, sync() polls it together with ncclCommGetAsyncError; an
//     asynchronous NCCL error or the deadline aborts the communicator
//     (ncclCommAbort) and poisons the context, so this and every later
//     collective call fails with CollectiveError (comm_inprocess.cpp:66-78);
//   * optional (count, op) agreement before each collective
//     (verify_uniform, comm_inprocess.cpp:139-151): the ranks all-gather
//     (sequence, count, tag) and every rank reaches the same verdict and
//     message;
//   * rank-local failures ahead of a collective ride in a status slot of the
//     collective's own buffer (attempt/settle in capi_internal.h), so peers
//     raise CollectiveError "rank r aborted" instead of waiting out the
//     deadline (comm_inprocess.cpp:171).
#include "capi_internal.h"

#include <chrono>
#include <map>

namespace dopinf_b200 {
namespace capi {

namespace {

using Clock = std::chrono::steady_clock;

// Debug stall behind an injected collective: spins until the host releases
// the flag (the abort path does) or `max_ns` passes, so it can never outlive
// its test by more than the bound.
__global__ void stall_kernel(volatile int* flag, unsigned long long max_ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        __nanosleep(20000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (*flag == 0 && t - t0 < max_ns);
}

// Positive control of the guarded allocations: one store just past a buffer.
__global__ void poke_kernel(double* p) { *p = 1.0; }

// Tags of verify_uniform: the op for an all-reduce, the root for a broadcast.
constexpr long long kTagAllgather = 100, kTagBroadcast = 200;

long long reduce_tag(ncclRedOp_t op, ncclDataType_t type) {
    return static_cast<long long>(op) + 16LL * static_cast<long long>(type);
}

[[noreturn]] void poison_and_fail(dopinf_b200_ctx* c, const std::string& msg) {
    if (!c->poisoned) {
        c->poisoned = true;
        c->poison_msg = msg;
    }
    fail(DOPINF_B200_ERR_COLLECTIVE, msg);
}

// ncclCommAbort: NCCL kernels waiting on absent peers exit, the communicator
// is gone (also one handed in by ctx_create_external — it is unusable after a
// hang); the stream then drains (bounded wait).
void abort_comm(dopinf_b200_ctx* c) {
    // an injected stall is not an NCCL kernel: release it first, since the
    // abort waits for the device work NCCL cannot flag
    if (c->stall_flag) *reinterpret_cast<volatile int*>(c->stall_flag) = 1;
    if (c->comm) {
        ncclCommAbort(c->comm);
        c->comm = nullptr;
    }
    const auto t0 = Clock::now();
    while (cudaStreamQuery(c->stream) == cudaErrorNotReady &&
           Clock::now() - t0 < std::chrono::seconds(20)) {
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    cudaGetLastError();
    c->coll_pending = false;
}

void before(dopinf_b200_ctx* c, size_t count, long long tag, const char* what);

// An NCCL call on a non-blocking communicator may return ncclInProgress: its
// host-side work (connection setup, the init itself) completes in the
// background and must be polled; a peer that never arrives leaves it in
// progress, so the poll has the collective deadline.
void settle_call(dopinf_b200_ctx* c, ncclResult_t r, const std::string& what) {
    if (r == ncclSuccess) return;
    if (r != ncclInProgress) poison_and_fail(c, what + ": " + ncclGetErrorString(r));
    const auto t0 = Clock::now();
    for (;;) {
        ncclResult_t st = ncclInProgress;
        if (ncclCommGetAsyncError(c->comm, &st) != ncclSuccess) st = ncclInternalError;
        if (st == ncclSuccess) return;
        if (st != ncclInProgress) {
            abort_comm(c);
            poison_and_fail(c, what + ": " + ncclGetErrorString(st));
        }
        if (std::chrono::duration<double>(Clock::now() - t0).count() > c->coll_timeout_s) {
            abort_comm(c);
            poison_and_fail(c, "collective timed out waiting for peer ranks");
        }
        std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
}

void issued(dopinf_b200_ctx* c) {
    c->coll_pending = true;
    ++c->coll_seq;
    if (c->inject == DOPINF_B200_INJECT_STALL) {
        c->inject = 0;
        if (!c->stall_flag) {
            void* p = nullptr;
            ck(cudaHostAlloc(&p, sizeof(int), cudaHostAllocMapped), "stall flag");
            c->stall_flag = static_cast<int*>(p);
        }
        *reinterpret_cast<volatile int*>(c->stall_flag) = 0;
        int* dflag = nullptr;
        ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dflag), c->stall_flag, 0), "stall flag");
        const double bound_s = c->coll_timeout_s + 30.0;
        stall_kernel<<<1, 1, 0, c->stream>>>(dflag, static_cast<unsigned long long>(bound_s * 1e9));
        note_launch();
        ck(cudaGetLastError(), "stall");
    }
}

// comm_inprocess.cpp:139-151 over NCCL: all-gather (sequence, count, tag).
void before(dopinf_b200_ctx* c, size_t count, long long tag, const char* what) {
    if (c->poisoned) fail(DOPINF_B200_ERR_COLLECTIVE, c->poison_msg);
    if (!c->coll_checks) return;
    const int p = c->size;
    long long mine[3] = {c->coll_seq, static_cast<long long>(count), tag};
    auto* dev = c->coll_scratch.get<long long>(3 * (static_cast<size_t>(p) + 1), "collective check");
    long long* pin = c->small_pinned<long long>(3 * static_cast<size_t>(p) + 3);
    std::memcpy(pin, mine, sizeof mine);
    ck(cudaMemcpyAsync(dev, pin, sizeof mine, cudaMemcpyHostToDevice, c->stream), "check H2D");
    settle_call(c, ncclAllGather(dev, dev + 3, 3, ncclInt64, c->comm, c->stream), what);
    c->coll_pending = true;
    ck(cudaMemcpyAsync(pin + 3, dev + 3, 3 * static_cast<size_t>(p) * sizeof(long long), cudaMemcpyDeviceToHost,
                       c->stream),
       "check D2H");
    c->sync(what);
    const std::vector<long long> table(pin + 3, pin + 3 + 3 * static_cast<size_t>(p));
    char msg[512];
    if (dopinf_b200_check_uniform(table.data(), p, c->rank, what, msg, sizeof msg) != DOPINF_B200_OK) {
        // every rank holds the same table, so every rank poisons with the same verdict
        if (!c->poisoned) {
            c->poisoned = true;
            c->poison_msg = std::string(what) + ": ranks disagree on buffer shape or operation";
        }
        fail(DOPINF_B200_ERR_COLLECTIVE, msg);
    }
}

}  // namespace

void coll_allreduce(dopinf_b200_ctx* c, const void* send, void* recv, size_t count, ncclDataType_t type,
                    ncclRedOp_t op, const char* what) {
    before(c, count, reduce_tag(op, type), what);
    settle_call(c, ncclAllReduce(send, recv, count, type, op, c->comm, c->stream), what);
    issued(c);
}

void coll_allgather(dopinf_b200_ctx* c, const void* send, void* recv, size_t count, ncclDataType_t type,
                    const char* what) {
    before(c, count, kTagAllgather, what);
    settle_call(c, ncclAllGather(send, recv, count, type, c->comm, c->stream), what);
    issued(c);
}

void coll_broadcast(dopinf_b200_ctx* c, void* buf, size_t count, ncclDataType_t type, int root, const char* what) {
    before(c, count, kTagBroadcast + root, what);
    settle_call(c, ncclBroadcast(buf, buf, count, type, root, c->comm, c->stream), what);
    issued(c);
}

void join_stream(dopinf_b200_ctx* c, cudaStream_t s) {
    if (!c->poisoned) {
        cudaStreamSynchronize(s);
        return;
    }
    const auto t0 = Clock::now();
    while (cudaStreamQuery(s) == cudaErrorNotReady && Clock::now() - t0 < std::chrono::seconds(20)) {
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    cudaGetLastError();
}

// ---- guarded allocations ----------------------------------------------------------
namespace {
constexpr unsigned char kGuardByte = 0xA5;
std::mutex g_guard_mu;
std::map<void*, size_t> g_guarded;  // user pointer -> user bytes
std::atomic<long long> g_guard_violations{0};

bool guard_intact(void* user, size_t bytes) {
    const size_t g = guard_bytes();
    std::vector<unsigned char> h(2 * g);
    char* base = static_cast<char*>(user) - g;
    if (cudaMemcpy(h.data(), base, g, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(h.data() + g, static_cast<char*>(user) + bytes, g, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return true;  // a device fault is reported by the call that caused it
    }
    for (unsigned char v : h) {
        if (v != kGuardByte) return false;
    }
    return true;
}
}  // namespace

size_t guard_bytes() {
    static const size_t g = [] {
        const char* e = std::getenv("DOPINF_B200_GUARD_BYTES");
        const long long v = e ? std::atoll(e) : 0;
        return v > 0 ? (static_cast<size_t>(v) + 255) / 256 * 256 : size_t(0);
    }();
    return g;
}

cudaError_t dev_alloc(void** p, size_t bytes) {
    const size_t g = guard_bytes();
    if (g == 0) return cudaMalloc(p, bytes);
    char* base = nullptr;
    cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&base), bytes + 2 * g);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemset(base, kGuardByte, g)) != cudaSuccess) return e;
    if ((e = cudaMemset(base + g + bytes, kGuardByte, g)) != cudaSuccess) return e;
    *p = base + g;
    std::lock_guard<std::mutex> lock(g_guard_mu);
    g_guarded[*p] = bytes;
    return cudaSuccess;
}

void dev_free(void* p) {
    const size_t g = guard_bytes();
    if (g == 0) {
        cudaFree(p);
        return;
    }
    size_t bytes = 0;
    {
        std::lock_guard<std::mutex> lock(g_guard_mu);
        auto it = g_guarded.find(p);
        if (it == g_guarded.end()) {
            cudaFree(p);
            return;
        }
        bytes = it->second;
        g_guarded.erase(it);
    }
    cudaDeviceSynchronize();
    if (!guard_intact(p, bytes)) {
        ++g_guard_violations;
        std::fprintf(stderr, "dopinf_b200: guard region of a %zu-byte device buffer overwritten\n", bytes);
    }
    cudaFree(static_cast<char*>(p) - g);
}

// Create the rank's communicator as a non-blocking one and wait for the init
// with the collective deadline: a peer that never joins (it failed before the
// init) ends in CollectiveError instead of a hang in ncclCommInitRank.
void comm_init(dopinf_b200_ctx* c, int size, const ncclUniqueId& uid, int rank) {
    if (const char* e = std::getenv("DOPINF_B200_COLLECTIVE_TIMEOUT")) {
        const double v = std::atof(e);
        if (v > 0.0) c->coll_timeout_s = v;
    }
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    cfg.blocking = 0;
    ncclComm_t comm = nullptr;
    const ncclResult_t r = ncclCommInitRankConfig(&comm, size, uid, rank, &cfg);
    c->comm = comm;
    if (r != ncclSuccess && r != ncclInProgress) {
        c->comm = nullptr;
        fail(DOPINF_B200_ERR_COLLECTIVE, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    settle_call(c, r, "ncclCommInitRank");
}

// Finalize (non-blocking: polled, bounded) and destroy an owned communicator.
void comm_destroy(dopinf_b200_ctx* c) {
    if (!c->comm) return;
    ncclResult_t r = ncclCommFinalize(c->comm);
    const auto t0 = Clock::now();
    while (r == ncclInProgress && Clock::now() - t0 < std::chrono::seconds(20)) {
        std::this_thread::sleep_for(std::chrono::microseconds(100));
        if (ncclCommGetAsyncError(c->comm, &r) != ncclSuccess) break;
    }
    if (r == ncclSuccess) {
        ncclCommDestroy(c->comm);
    } else {
        ncclCommAbort(c->comm);
    }
    c->comm = nullptr;
}

}  // namespace capi
}  // namespace dopinf_b200

void dopinf_b200_ctx::sync(const char* what) {
    if (!coll_pending) {
        ck(cudaStreamSynchronize(stream), what);
        return;
    }
    // A collective is queued: poll the stream and the communicator until the
    // deadline (spin briefly first: most collectives finish within microseconds).
    const auto t0 = Clock::now();
    const auto deadline = t0 + std::chrono::duration_cast<Clock::duration>(std::chrono::duration<double>(coll_timeout_s));
    for (long long it = 0;; ++it) {
        const cudaError_t e = cudaStreamQuery(stream);
        if (e == cudaSuccess) {
            coll_pending = false;
            return;
        }
        if (e != cudaErrorNotReady) ck(e, what);
        if (comm) {
            ncclResult_t st = ncclSuccess;
            if (ncclCommGetAsyncError(comm, &st) == ncclSuccess && st != ncclSuccess && st != ncclInProgress) {
                const std::string msg = std::string(what) + ": NCCL asynchronous error: " + ncclGetErrorString(st);
                abort_comm(this);
                poison_and_fail(this, msg);
            }
        }
        const auto now = Clock::now();
        if (now >= deadline) {
            abort_comm(this);
            poison_and_fail(this, "collective timed out waiting for peer ranks");
        }
        if (now - t0 < std::chrono::milliseconds(2)) {
            std::this_thread::yield();
        } else {
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
}

extern "C" {

int dopinf_b200_check_uniform(const long long* table, int p, int rank, const char* what, char* msg,
                              size_t msg_cap) {
    if (!table || p < 1 || rank < 0 || rank >= p) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    const std::string w = what ? what : "collective";
    const long long* mine = table + 3 * static_cast<size_t>(rank);
    std::string m;
    for (int r = 0; r < p && m.empty(); ++r) {
        const long long* t = table + 3 * static_cast<size_t>(r);
        if (t[0] != mine[0]) {
            m = w + ": ranks are out of step (rank " + std::to_string(rank) + " is at collective " +
                std::to_string(mine[0]) + ", rank " + std::to_string(r) + " at " + std::to_string(t[0]) + ")";
        } else if (t[1] != mine[1] || t[2] != mine[2]) {
            // comm_inprocess.cpp:145-148
            m = w + ": rank " + std::to_string(rank) + " passed count " + std::to_string(mine[1]) + ", rank " +
                std::to_string(r) + " passed count " + std::to_string(t[1]);
            if (t[1] == mine[1]) m += " (operations differ)";
        }
    }
    if (m.empty()) return DOPINF_B200_OK;
    if (msg && msg_cap > 0) {
        const size_t n = std::min(m.size(), msg_cap - 1);
        std::memcpy(msg, m.data(), n);
        msg[n] = '\0';
    }
    return DOPINF_B200_ERR_COLLECTIVE;
}

int dopinf_b200_debug_gram_coverage(int K, long long* entries, long long* covered, long long* duplicates,
                                    long long* mma_tiles) {
    if (K < 1 || !entries || !covered || !duplicates || !mma_tiles) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    try {
        const gram::CoverageReport r = gram::coverage(K);
        *entries = r.entries;
        *covered = r.covered;
        *duplicates = r.duplicates;
        *mma_tiles = r.mma_tiles;
        return DOPINF_B200_OK;
    } catch (const std::bad_alloc&) {
        return DOPINF_B200_ERR_OUT_OF_MEMORY;
    } catch (...) {
        return DOPINF_B200_ERR_DEVICE;
    }
}

long long dopinf_b200_debug_guard_violations(void) {
    if (guard_bytes() == 0) return -1;
    cudaDeviceSynchronize();
    std::vector<std::pair<void*, size_t>> live;
    {
        std::lock_guard<std::mutex> lock(g_guard_mu);
        live.assign(g_guarded.begin(), g_guarded.end());
    }
    long long bad = g_guard_violations.load();
    for (const auto& [p, n] : live) bad += guard_intact(p, n) ? 0 : 1;
    return bad;
}

int dopinf_b200_set_collective_timeout(dopinf_b200_ctx* c, double seconds) {
    return guarded(c, [&] {
        require(seconds > 0.0, "set_collective_timeout: seconds must be positive");
        c->coll_timeout_s = seconds;
    });
}

int dopinf_b200_set_collective_checks(dopinf_b200_ctx* c, int enabled) {
    return guarded(c, [&] { c->coll_checks = enabled != 0; });
}

int dopinf_b200_ctx_poisoned(const dopinf_b200_ctx* c) { return c && c->poisoned ? 1 : 0; }

int dopinf_b200_debug_inject(dopinf_b200_ctx* c, int what) {
    return guarded(c, [&] {
        require(what == 0 || what == DOPINF_B200_INJECT_STALL || what == DOPINF_B200_INJECT_OOB_STORE,
                "debug_inject: unknown fault");
        if (what == DOPINF_B200_INJECT_OOB_STORE) {
            require(guard_bytes() >= 8, "debug_inject: out-of-bounds store needs DOPINF_B200_GUARD_BYTES");
            double* p = c->span.get<double>(2, "span");
            poke_kernel<<<1, 1, 0, c->stream>>>(p + c->span.bytes / sizeof(double));
            note_launch();
            ck(cudaGetLastError(), "poke");
            c->sync("debug_inject");
            return;
        }
        require(what == 0 || c->comm, "debug_inject: the context has no NCCL communicator");
        c->inject = what;
    });
}

int dopinf_b200_ordered_sum(dopinf_b200_ctx* c, const double* parts, int p, size_t count, double* out) {
    return guarded(c, [&] {
        require(p >= 1 && (count == 0 || (parts && out)), "ordered_sum: bad arguments");
        if (count == 0) return;
        const size_t n = static_cast<size_t>(p) * count;
        double* dev = c->span.get<double>(n + count, "span");
        ck(cudaMemcpyAsync(dev, parts, n * sizeof(double), cudaMemcpyHostToDevice, c->stream), "parts H2D");
        ck(gram::launch_ordered_sum(dev, p, count, count, dev + n, c->stream), "ordered sum");
        ck(cudaMemcpyAsync(out, dev + n, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
        c->sync("ordered_sum");
    });
}

}  // extern "C"
