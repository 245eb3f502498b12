// capi.cu — the C ABI (include/dopinf_b200.h): per-rank contexts, device-
// resident LocalBlocks, NCCL collectives and the stage orchestration that the
// reference's pipeline::run_rank (proj/src/pipeline.cpp:270-298) performs on
// the host. Every entry point is synchronous at the boundary, never throws,
// and maps failures onto the reference's exception classes by status code.
#include "capi_internal.h"

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

namespace dopinf_b200 {
namespace capi {

thread_local std::string g_thread_err = "null context";

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
    double* vm = b->varmax.get<double>(b->n_vars + 1, "varmax");
    double* mn = b->means.get<double>(b->rows, "means");
    c->record(DOPINF_B200_STAGE_STATS, 0);
    ck(cudaMemsetAsync(vm, 0, b->n_vars * sizeof(double), c->stream), "memset");
    ck(transform::launch_stats(b->q, b->ld, static_cast<long long>(b->rows), static_cast<int>(b->nt),
                               static_cast<long long>(b->nx_i), static_cast<int>(b->n_vars), center,
                               mn, vm, c->num_sms, c->stream),
       "stats");
    c->record(DOPINF_B200_STAGE_STATS, 1);
}

void do_center(dopinf_b200_block* b, double* means_host, bool side_copy) {
    Nvtx nvtx_range("dopinf_b200 center_in_place");
    materialize(b);  // a second centering acts on centered values, as in the reference
    run_stats(b, true);
    b->pending_center = true;
    b->stats_valid = true;
    if (means_host && side_copy && is_pinned(means_host)) {
        // the means leave on the copy stream while the scales, apply and Gram
        // run; the caller joins the copy stream before returning
        auto* c = b->ctx;
        ck(cudaStreamWaitEvent(c->copy_stream, c->ev[DOPINF_B200_STAGE_STATS][1], 0), "wait stats");
        ck(cudaMemcpyAsync(means_host, b->means.get<double>(b->rows, "means"), b->rows * sizeof(double),
                           cudaMemcpyDeviceToHost, c->copy_stream),
           "means D2H");
    } else if (means_host) {
        ck(cudaMemcpyAsync(means_host, b->means.get<double>(b->rows, "means"), b->rows * sizeof(double),
                           cudaMemcpyDeviceToHost, b->ctx->stream),
           "means D2H");
    }
}

void do_global_scales(dopinf_b200_block* b, double* scales_host, size_t* degenerate,
                      const std::optional<Fail>& earlier) {
    Nvtx nvtx_range("dopinf_b200 compute_global_scales");
    auto* c = b->ctx;
    const size_t nv = b->n_vars;
    // varmax carries one status slot after the n_vars maxima: MAX of
    // (size - rank) over the failed ranks, so the lowest failed rank is size - max
    double* vm = b->varmax.get<double>(nv + 1, "varmax");
    double* red = c->scales.get<double>(nv + 1, "scales");
    std::optional<Fail> own = earlier;
    if (!own) {
        own = attempt(c, [&] {
            if (!b->stats_valid) {
                run_stats(b, false);
                b->stats_valid = true;
            }
        });
    }
    c->record(DOPINF_B200_STAGE_SCALES, 0);
    if (coll(c)) {
        const double flag = own ? static_cast<double>(c->size - c->rank) : 0.0;
        ck(cudaMemcpyAsync(vm + nv, &flag, sizeof(double), cudaMemcpyHostToDevice, c->stream), "status H2D");
        coll_allreduce(c, vm, red, nv + 1, ncclFloat64, ncclMax, "allreduce(MAX)");
    } else {
        ck(cudaMemcpyAsync(red, vm, nv * sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "copy");
    }
    c->record(DOPINF_B200_STAGE_SCALES, 1);
    double* pin = c->small_pinned<double>(nv + 1);
    pin[nv] = 0.0;
    ck(cudaMemcpyAsync(pin, red, (coll(c) ? nv + 1 : nv) * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
       "scales D2H");
    c->sync("global_scales");
    const std::vector<double> host(pin, pin + nv + 1);
    settle(own, host[nv] > 0.0 ? c->size - static_cast<int>(host[nv]) : -1);
    if (scales_host) std::memcpy(scales_host, host.data(), nv * sizeof(double));
    for (size_t j = 0; j < b->n_vars; ++j) {
        if (host[j] == 0.0) {
            if (degenerate) *degenerate = j;
            fail(DOPINF_B200_ERR_DEGENERATE_VARIABLE,
                 "variable " + std::to_string(j) + " is constant in time; max-abs scaling is undefined");
        }
    }
}

void do_scale(dopinf_b200_block* b, const double* scales_host) {
    Nvtx nvtx_range("dopinf_b200 scale_in_place");
    auto* c = b->ctx;
    double* ds = c->scales.get<double>(b->n_vars + 1, "scales");
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

void unpack(dopinf_b200_ctx* c, const double* packed) {
    const int K = c->K;
    c->record(DOPINF_B200_STAGE_UNPACK, 0);
    ck(gram::launch_unpack(packed, K, c->dmat.get<double>(static_cast<size_t>(K) * K, "D"), c->stream),
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
    Nvtx nvtx_range("dopinf_b200 local_gram");
    auto* c = b->ctx;
    materialize(b);
    const int K = static_cast<int>(b->nt);
    const long long rows = static_cast<long long>(b->rows);
    require(rows < (1LL << 31), "local_gram: blocks of 2^31 rows or more are not supported (TMA row coordinate)");
    c->have_gram = false;
    c->local_valid = false;
    c->K = K;
    // packed triangle + one status slot (0: this rank's partial is valid)
    double* packed = c->packed.get<double>(gram::packed_count(K) + 1, "packed");
    ck(cudaMemsetAsync(packed + gram::packed_count(K), 0, sizeof(double), c->stream), "memset");
    if (rows == 0) {
        ck(cudaMemsetAsync(packed, 0, gram::packed_count(K) * sizeof(double), c->stream), "memset");
    } else if (c->gram_order == DOPINF_B200_GRAM_ORDER_REFERENCE) {
        c->record(DOPINF_B200_STAGE_GRAM, 0);
        ck(gram::launch_gram_reference_order(b->q, b->ld, rows, K, packed, false, c->stream), "gram (reference order)");
        c->record(DOPINF_B200_STAGE_GRAM, 1);
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
        const int groups = gram::reduce_groups(c->plan, c->num_sms);
        double* scratch = groups > 1 ? c->reduce_scratch.get<double>(gram::reduce_scratch_doubles(c->plan, groups),
                                                                     "reduce scratch")
                                     : nullptr;
        ck(gram::launch_reduce(c->plan, tiles, work, packed, c->stream, groups, scratch), "gram reduce");
        c->record(DOPINF_B200_STAGE_GRAM_REDUCE, 1);
    }
    unpack(c, packed);
    c->have_gram = true;
    c->dmat_local = true;
    c->local_valid = true;
    copy_d_out(c, d_host);
}

// pod::global_gram: SUM over the ranks of the local partial in `packed` into
// `gpacked` (the partial stays, so a repeated call gives the same D). A rank
// whose local step failed (local_failure) still enters the reduction with its
// status slot set: every rank learns the lowest failed rank from the summed
// slot and raises (settle) instead of leaving its peers to the deadline.
void do_global_gram(dopinf_b200_ctx* c, double* d_host, const std::optional<Fail>& local_failure) {
    Nvtx nvtx_range("dopinf_b200 global_gram");
    if (!local_failure && !c->local_valid) {
        fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "global_gram: no local Gram on this context");
    }
    const int K = c->K;
    const size_t count = gram::packed_count(K);
    if (!coll(c)) {
        if (local_failure) throw *local_failure;
        if (!c->dmat_local) unpack(c, c->packed.get<double>(count + 1, "packed"));
        c->have_gram = true;
        c->dmat_local = true;
        copy_d_out(c, d_host);
        return;
    }
    double* packed = c->packed.get<double>(count + 1, "packed");
    if (local_failure) {  // else the status slot is 0 (do_local_gram / the streamed pass set it)
        double* bit = c->small_pinned<double>(1);
        *bit = failure_bit(c, true);
        ck(cudaMemsetAsync(packed, 0, count * sizeof(double), c->stream), "memset");
        ck(cudaMemcpyAsync(packed + count, bit, sizeof(double), cudaMemcpyHostToDevice, c->stream), "status H2D");
    }
    double* out = c->gpacked.get<double>(count + 1, "reduced Gram");
    c->record(DOPINF_B200_STAGE_ALLREDUCE, 0);
    if (c->gram_reduce == DOPINF_B200_GRAM_REDUCE_NCCL) {
        coll_allreduce(c, packed, out, count + 1, ncclFloat64, ncclSum, "allreduce(SUM)");
    } else {
        double* parts = c->gather.get<double>((count + 1) * static_cast<size_t>(c->size), "gather");
        coll_allgather(c, packed, parts, count + 1, ncclFloat64, "allgather");
        ck(gram::launch_ordered_sum(parts, c->size, count + 1, count + 1, out, c->stream), "ordered sum");
    }
    c->record(DOPINF_B200_STAGE_ALLREDUCE, 1);
    double* pin = c->small_pinned<double>(1);
    ck(cudaMemcpyAsync(pin, out + count, sizeof(double), cudaMemcpyDeviceToHost, c->stream), "status D2H");
    c->sync("global_gram");
    const double status = *pin;
    c->have_gram = false;
    settle(local_failure, lowest_failed(status));
    unpack(c, out);
    c->have_gram = true;
    c->dmat_local = false;
    copy_d_out(c, d_host);
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
    Nvtx nvtx_range("dopinf_b200 project");
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
    Nvtx nvtx_range("dopinf_b200 basis");
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

void ensure_events(std::vector<cudaEvent_t>& v, size_t n) {
    while (v.size() < n) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        v.push_back(e);
    }
}

}  // namespace capi
}  // namespace dopinf_b200

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

}  // extern "C"

namespace {

// Device checks, streams and stage events of a new context (stream: the
// caller's, or null to create one).
void init_ctx(dopinf_b200_ctx* c, int device, cudaStream_t stream) {
    int ndev = 0;
    ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    if (device < 0 || device >= ndev) {
        fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "device " + std::to_string(device) + " not present");
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop;
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0) {
        fail(DOPINF_B200_ERR_DEVICE, std::string("device is ") + prop.name + " (sm_" + std::to_string(prop.major) +
                                         std::to_string(prop.minor) + "); this build targets sm_100a (B200) only");
    }
    c->num_sms = prop.multiProcessorCount;
    if (stream) {
        c->stream = stream;
        c->owns_stream = false;
    } else {
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    ck(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    for (auto& pair : c->ev) {
        ck(cudaEventCreate(&pair[0]), "cudaEventCreate");
        ck(cudaEventCreate(&pair[1]), "cudaEventCreate");
    }
}

int finish_create(dopinf_b200_ctx* c, int rc, dopinf_b200_ctx** out) {
    if (rc != DOPINF_B200_OK) {
        std::fprintf(stderr, "dopinf_b200_ctx_create: %s\n", c->err.c_str());
        dopinf_b200_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return DOPINF_B200_OK;
}

}  // namespace

extern "C" {

int dopinf_b200_ctx_create(int device, int rank, int size, const unsigned char* id,
                           dopinf_b200_ctx** out) {
    return dopinf_b200_ctx_create_ex(device, rank, size, id, 0u, out);
}

int dopinf_b200_ctx_create_ex(int device, int rank, int size, const unsigned char* id, unsigned flags,
                              dopinf_b200_ctx** out) {
    const bool nccl = size > 1 || (flags & DOPINF_B200_CTX_NCCL) != 0;
    if (!out || size < 1 || rank < 0 || rank >= size || (nccl && !id) || (flags & ~DOPINF_B200_CTX_NCCL)) {
        return DOPINF_B200_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    auto* c = new (std::nothrow) dopinf_b200_ctx;
    if (!c) return DOPINF_B200_ERR_OUT_OF_MEMORY;
    c->device = device;
    c->rank = rank;
    c->size = size;
    const int rc = guarded(c, [&] {
        init_ctx(c, device, nullptr);
        if (nccl) {
            ncclUniqueId uid;
            std::memcpy(&uid, id, sizeof uid);
            comm_init(c, size, uid, rank);
        }
    });
    return finish_create(c, rc, out);
}

int dopinf_b200_ctx_create_external(int device, void* nccl_comm, void* stream, dopinf_b200_ctx** out) {
    if (!out) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    auto* c = new (std::nothrow) dopinf_b200_ctx;
    if (!c) return DOPINF_B200_ERR_OUT_OF_MEMORY;
    c->device = device;
    const int rc = guarded(c, [&] {
        init_ctx(c, device, static_cast<cudaStream_t>(stream));
        if (nccl_comm) {
            c->comm = static_cast<ncclComm_t>(nccl_comm);
            c->owns_comm = false;
            ckn(ncclCommUserRank(c->comm, &c->rank), "ncclCommUserRank");
            ckn(ncclCommCount(c->comm, &c->size), "ncclCommCount");
        }
    });
    return finish_create(c, rc, out);
}

void dopinf_b200_ctx_destroy(dopinf_b200_ctx* c) {
    if (!c) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(c->device);
    if (c->stream) join_stream(c, c->stream);
    if (c->comm && c->owns_comm) comm_destroy(c);
    if (c->stall_flag) cudaFreeHost(c->stall_flag);
    for (auto& pair : c->ev) {
        if (pair[0]) cudaEventDestroy(pair[0]);
        if (pair[1]) cudaEventDestroy(pair[1]);
    }
    for (DBuf* b : {&c->tiles, &c->work, &c->counters, &c->packed, &c->gpacked, &c->coll_scratch, &c->gather,
                    &c->dmat, &c->dhost_in, &c->scales, &c->tr, &c->trt, &c->qhat, &c->sel, &c->rows_out, &c->span, &c->eig_a,
                    &c->eig_w, &c->eig_work, &c->eig_info, &c->eig_v, &c->eig_lambda, &c->tr_dev, &c->field_qt,
                    &c->field_means, &c->field_scales, &c->field_ring, &c->rom_qhat, &c->rom_dhat, &c->rom_q2t,
                    &c->rom_qrows, &c->rom_rhs, &c->rom_g, &c->rom_lhs, &c->rom_rhsb, &c->rom_betas, &c->rom_traj,
                    &c->rom_scores, &c->rom_work, &c->rom_info, &c->rom_tiles, &c->rom_gwork, &c->rom_counters,
                    &c->rom_packed, &c->rom_packet}) {
        b->release();
    }
    c->staging.release();
    c->coll_host.release();
    c->file_ring.release();
    c->gv.release();
    c->ring.release();
    for (cudaEvent_t e : c->chunk_events) cudaEventDestroy(e);
    for (cudaEvent_t e : c->chunk_events2) cudaEventDestroy(e);
    for (cudaEvent_t e : c->timing_events) cudaEventDestroy(e);
    if (c->copy_stream) {
        join_stream(c, c->copy_stream);
        cudaStreamDestroy(c->copy_stream);
    }
    if (c->stream && c->owns_stream) cudaStreamDestroy(c->stream);
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

int dopinf_b200_set_gram_order(dopinf_b200_ctx* c, int order) {
    return guarded(c, [&] {
        require(order == DOPINF_B200_GRAM_ORDER_TENSOR || order == DOPINF_B200_GRAM_ORDER_REFERENCE,
                "set_gram_order: unknown order");
        c->gram_order = order;
        if (order == DOPINF_B200_GRAM_ORDER_REFERENCE) c->gram_reduce = DOPINF_B200_GRAM_REDUCE_ORDERED;
    });
}

int dopinf_b200_allreduce(dopinf_b200_ctx* c, double* data, size_t count, int op) {
    return guarded(c, [&] {
        require(op >= DOPINF_B200_SUM && op <= DOPINF_B200_MIN, "allreduce: unknown op");
        require(count == 0 || data, "allreduce: null data");
        if (!coll(c) || count == 0) return;
        double* buf = c->span.get<double>(count * (op == DOPINF_B200_SUM ? c->size + 1 : 1), "span");
        ck(cudaMemcpyAsync(buf, data, count * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
        if (op == DOPINF_B200_SUM) {
            // Ascending-rank order, as the reference's in-process backend sums.
            double* parts = buf + count;
            coll_allgather(c, buf, parts, count, ncclFloat64, "allreduce");
            ck(gram::launch_ordered_sum(parts, c->size, count, count, buf, c->stream), "ordered sum");
        } else {
            coll_allreduce(c, buf, buf, count, ncclFloat64, op == DOPINF_B200_MAX ? ncclMax : ncclMin,
                           "allreduce");
        }
        double* pin = c->small_pinned<double>(count);
        ck(cudaMemcpyAsync(pin, buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
        c->sync("allreduce");
        std::memcpy(data, pin, count * sizeof(double));
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
        require(b->rows < (size_t(1) << 31), "block_create: blocks of 2^31 rows or more are not supported "
                                             "(TMA row coordinates are 32-bit); shard over more ranks");
        if (b->rows > 0) {
            ck(dev_alloc(reinterpret_cast<void**>(&b->q), b->rows * b->ld * sizeof(double)), "block values");
            if (b->ld != nt) {
                ck(cudaMemsetAsync(b->q, 0, b->rows * b->ld * sizeof(double), c->stream), "memset");
            }
        }
        b->varmax.get<double>(n_vars + 1, "varmax");  // + the status slot of the MAX collective
        c->sync("block_create");
    });
    if (rc != DOPINF_B200_OK) {
        if (b->q) dev_free(b->q);
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
    if (b->q) dev_free(b->q);
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
        if (b->rows > 0 && b->rows * b->nt * sizeof(double) >= (size_t(64) << 20) && !is_pinned(host)) {
            staged_upload(b, host, host_ld);  // records the UPLOAD stage itself
            b->pending_center = false;
            b->stats_valid = false;
            return;
        }
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
        if (b->rows > 0 && b->rows * b->nt * sizeof(double) >= (size_t(64) << 20) && !is_pinned(host)) {
            staged_download(b, 0, b->rows, host, host_ld);
        } else if (b->rows > 0) {
            ck(cudaMemcpy2DAsync(host, host_ld * sizeof(double), b->q, b->ld * sizeof(double),
                                 b->nt * sizeof(double), b->rows, cudaMemcpyDeviceToHost, c->stream),
               "download");
        }
        c->record(DOPINF_B200_STAGE_DOWNLOAD, 1);
        c->sync("block_download");
    });
}

int dopinf_b200_block_download_rows(dopinf_b200_block* b, size_t row0, size_t nrows, double* host,
                                    size_t host_ld) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(host_ld >= b->nt && (nrows == 0 || host), "block_download_rows: bad host buffer");
        require(row0 <= b->rows && nrows <= b->rows - row0, "block_download_rows: rows outside the block");
        materialize(b);
        if (nrows * b->nt * sizeof(double) >= (size_t(64) << 20) && !is_pinned(host)) {
            staged_download(b, row0, nrows, host, host_ld);
        } else if (nrows > 0) {
            ck(cudaMemcpy2DAsync(host, host_ld * sizeof(double), b->q + row0 * b->ld, b->ld * sizeof(double),
                                 b->nt * sizeof(double), nrows, cudaMemcpyDeviceToHost, c->stream),
               "download");
        }
        c->sync("block_download_rows");
    });
}

int dopinf_b200_block_shape(const dopinf_b200_block* b, size_t* dims) {
    if (!b || !dims) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    dims[0] = b->n_vars;
    dims[1] = b->nx_i;
    dims[2] = b->row_begin;
    dims[3] = b->nt;
    return DOPINF_B200_OK;
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
    return dopinf_b200_block_synth_oscillator_vars(b, 0, seed, n_modes, dt, noise, amps);
}

int dopinf_b200_block_synth_oscillator_vars(dopinf_b200_block* b, int var0, uint64_t seed, int n_modes, double dt,
                                            double noise, const double* amps) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(var0 >= 0, "synth: var0 must be >= 0");
        if (b->rows == 0) return;
        ck(synth::oscillator(b->q, b->ld, static_cast<long long>(b->rows), static_cast<int>(b->nt),
                             static_cast<long long>(b->nx_i), static_cast<long long>(b->row_begin),
                             static_cast<int>(b->n_vars), seed, n_modes, dt, noise, amps, c->num_sms,
                             c->stream, var0),
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

int dopinf_b200_local_maxabs(dopinf_b200_block* b, double* maxabs) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    return guarded(b->ctx, [&] {
        require(maxabs != nullptr, "local_maxabs: null output");
        if (!b->stats_valid) {
            run_stats(b, false);
            b->stats_valid = true;
        }
        auto* c = b->ctx;
        std::vector<double> host(b->n_vars);
        ck(cudaMemcpyAsync(host.data(), b->varmax.get<double>(b->n_vars + 1, "varmax"), b->n_vars * sizeof(double),
                           cudaMemcpyDeviceToHost, c->stream),
           "maxabs D2H");
        c->sync("local_maxabs");
        std::memcpy(maxabs, host.data(), host.size() * sizeof(double));
    });
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

int dopinf_b200_global_gram(dopinf_b200_ctx* c, double* d, size_t nt) {
    return guarded(c, [&] {
        require(c->local_valid, "global_gram: no local Gram on this context");
        require(nt == static_cast<size_t>(c->K),
                "global_gram: local Gram is " + std::to_string(c->K) + " x " + std::to_string(c->K) +
                    ", caller passed nt = " + std::to_string(nt));
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
        c->local_valid = false;  // D is the caller's: no local partial to reduce
        c->dmat_local = false;
        c->eig_K = 0;
        c->tr_dev_r = 0;
        c->sync("set_gram");
    });
}

int dopinf_b200_eig_sym_desc(dopinf_b200_ctx* c, double* lambda, double* vectors) {
    return guarded(c, [&] {
        Nvtx nvtx_range("dopinf_b200 eig_sym_desc");
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
        struct JoinCopies {  // also on failure: no copy into the caller's means outlives the call
            dopinf_b200_ctx* c;
            ~JoinCopies() { join_stream(c, c->copy_stream); }
        } join{c};
        // Rank-local steps that fail still enter the collective that follows,
        // whose status slot tells the peers (attempt / settle).
        std::optional<Fail> own = attempt(c, [&] {
            if (b->rows > 0) do_center(b, means, true);
        });
        std::vector<double> s(b->n_vars);  // outlives the async scales upload (synced below)
        if (scaling) {
            do_global_scales(b, s.data(), nullptr, own);  // settles `own` across the ranks
            if (scales) std::memcpy(scales, s.data(), s.size() * sizeof(double));
            own.reset();
        }
        if (!own) {
            own = attempt(c, [&] {
                if (scaling && b->rows > 0) do_scale(b, s.data());
                do_local_gram(b, nullptr);
            });
        }
        do_global_gram(c, d, own);
        c->sync("snapshot_pass");
    });
}

}  // extern "C"
