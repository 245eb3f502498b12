// capi_io.cu — the C ABI's streamed passes (host rows, SNP1 files, device-
// generated rows) and the SNP1 container (reference data.hpp / data.cpp):
// header parsing with the reference's checks and messages, the pinned-ring
// file reader, and Steps II–III over chunks whose H2D / read overlaps the
// compute of the chunk before.
#include "capi_internal.h"

namespace dopinf_b200 {
namespace capi {

namespace {

// ---- streamed Steps II-III ----------------------------------------------------------
// dopinf_b200_snapshot_pass_host: rows arrive from host memory into the
// resident block (H2D on the copy stream overlaps the compute stream).
// dopinf_b200_stream_pass_synth: rows are generated on the device chunk by chunk
// into a two-slot ring — the block is never resident (config 4: 403 GB/GPU).
constexpr long long kStreamChunkRows = 32768;   // rows per H2D chunk (315 MB at K = 1200)
constexpr size_t kStagedSlotBytes = size_t(64) << 20;  // pinned ring slot of staged (file / pageable) copies

// Rows per chunk of a staged copy: ~64 MB slots, so the pinned ring a context
// allocates on first use is ~128 MB (page-locking costs ~0.1 s per 100 MB) and
// the first copy starts early.
long long staged_rows(size_t nt) {
    const long long r = static_cast<long long>(kStagedSlotBytes / (nt * sizeof(double)));
    return std::max<long long>(256, std::min<long long>(kStreamChunkRows, r));
}

constexpr long long kTailChunkRows = 8192;     // the pass's final chunk is cut to this size
constexpr long long kStreamSplitRows = 2048;    // rows per Gram item inside a host chunk

constexpr long long kSynthChunkRows = 262144;   // rows per generated chunk (3.1 GB at K = 1500)

constexpr long long kSynthSplitRows = 8192;

struct StreamChunk {
    int var;
    long long r0, rows;
    bool first_of_var, last_of_var;
};

// Joins the copy stream when an entry point leaves (also on failure): work a
// streamed pass left there (the last variable's scaling) is done by then.
struct SideJoin {
    dopinf_b200_ctx* c;
    ~SideJoin() { join_stream(c, c->copy_stream); }
};

struct StreamSource {
    const double* host = nullptr;  // host rows (pitch host_ld) → resident block
    size_t host_ld = 0;
    bool synth = false;            // device-generated rows → ring buffer, block not resident
    uint64_t seed = 0;
    int n_modes = 0;
    double dt = 0.0, noise = 0.0;
    const double* amps = nullptr;  // host [n_vars] or null
    bool pageable = false;         // host rows not pinned: staged through the pinned ring
    int fd = -1;                   // SNP1 file rows → pinned ring → resident block
    const Snp1* file = nullptr;
    const std::string* path = nullptr;
};

// Pageable host rows [r0, r0 + rows) (pitch sld) → dense pinned slot (pitch
// nt) on up to file_reader_threads() threads: a pageable H2D runs through the
// driver's staging at ~10 GB/s; parallel host copies into pinned memory plus a
// pinned H2D run at the link rate.
void copy_rows_parallel(double* dst, const double* src, size_t sld, size_t nt, long long rows) {
    const size_t total = static_cast<size_t>(rows) * nt;
    const int n = static_cast<int>(std::min<size_t>(file_reader_threads(), std::max<size_t>(1, total >> 20)));
    auto part = [&](int i) {
        const long long a = rows * i / n, e = rows * (i + 1) / n;
        if (sld == nt) {
            std::memcpy(dst + a * nt, src + a * nt, static_cast<size_t>(e - a) * nt * sizeof(double));
        } else {
            for (long long r = a; r < e; ++r) std::memcpy(dst + r * nt, src + r * sld, nt * sizeof(double));
        }
    };
    parallel_for(n, part);
}

// Staged source (SNP1 file or pageable host rows): fill pinned ring slot k % 2
// with chunk k of the block's rows and enqueue its H2D on the copy stream;
// chunk_events[k] marks the copy done (the compute stream waits on it; filling
// chunk k + 2 into the same slot waits on it from the host).
void staged_chunk_h2d(dopinf_b200_block* b, const StreamSource& src, const std::vector<StreamChunk>& chunks,
                      size_t k, double* ring, size_t slot_doubles) {
    auto* c = b->ctx;
    const StreamChunk& ch = chunks[k];
    if (k >= 2) ck(cudaEventSynchronize(c->chunk_events[k - 2]), "ring slot");
    double* slot = ring + (k % 2) * slot_doubles;
    if (src.fd >= 0) {
        const uint64_t local0 = static_cast<uint64_t>(ch.r0) - static_cast<uint64_t>(ch.var) * b->nx_i;
        const uint64_t first = static_cast<uint64_t>(ch.var) * src.file->nx + b->row_begin + local0;
        const size_t bytes = static_cast<size_t>(ch.rows) * b->nt * sizeof(double);
        if (!pread_parallel(src.fd, slot, bytes, src.file->data_offset + first * b->nt * sizeof(double))) {
            format_fail("snapshot file truncated in variable '" + src.file->names[ch.var] + "': " + *src.path);
        }
    } else {
        copy_rows_parallel(slot, src.host + static_cast<size_t>(ch.r0) * src.host_ld, src.host_ld, b->nt, ch.rows);
    }
    ck(copy_rows(b->q + ch.r0 * b->ld, b->ld, slot, b->nt, b->nt, ch.rows, cudaMemcpyHostToDevice, c->copy_stream),
       "chunk H2D");
    ck(cudaEventRecord(c->chunk_events[k], c->copy_stream), "event");
}

std::vector<StreamChunk> stream_chunks(const dopinf_b200_block* b, long long chunk_rows, bool split_tail) {
    std::vector<StreamChunk> out;
    for (size_t v = 0; v < b->n_vars; ++v) {
        const long long v0 = static_cast<long long>(v * b->nx_i), v1 = v0 + static_cast<long long>(b->nx_i);
        for (long long r0 = v0; r0 < v1; r0 += chunk_rows) {
            const long long rows = std::min(chunk_rows, v1 - r0);
            out.push_back({static_cast<int>(v), r0, rows, r0 == v0, r0 + rows == v1});
        }
    }
    // A copied pass cannot finish before the last chunk has landed and been
    // processed: cut the final chunk finer so little work trails the last copy.
    if (split_tail && !out.empty() && out.back().rows > kTailChunkRows) {
        const StreamChunk last = out.back();
        out.pop_back();
        for (long long r0 = last.r0; r0 < last.r0 + last.rows; r0 += kTailChunkRows) {
            const long long rows = std::min(kTailChunkRows, last.r0 + last.rows - r0);
            out.push_back({last.var, r0, rows, last.first_of_var && r0 == last.r0,
                           last.last_of_var && r0 + rows == last.r0 + last.rows});
        }
    }
    return out;
}

// On the compute stream each landed chunk gets its row means / max-abs (stats
// pass), is centered in place, and its Gram items accumulate (chunk order)
// into the split slots of its variable. When a variable's last chunk is done
// its slots are reduced into G_v, its MAX goes over the ranks and (resident
// block) its rows are scaled. D = Σ_v G_v / s_v². In the reference-order
// mode the chunks are only centered; once a variable is scaled, its rows'
// Gram continues the reference's FMA chains (gram_ref.cu) in block-row order.
void do_stream_pass(dopinf_b200_block* b, const StreamSource& src, bool scaling, double* means_host,
                    double* scales_host) {
    Nvtx nvtx_range("dopinf_b200 streamed snapshot pass");
    auto* c = b->ctx;
    const int K = static_cast<int>(b->nt);
    const size_t count = gram::packed_count(K);
    const long long chunk_rows =
        src.synth ? kSynthChunkRows : (src.fd >= 0 || src.pageable) ? staged_rows(b->nt) : kStreamChunkRows;
    const long long split_rows = src.synth ? kSynthSplitRows : kStreamSplitRows;
    const bool ref_order = c->gram_order == DOPINF_B200_GRAM_ORDER_REFERENCE;
    require(!(ref_order && src.synth),
            "stream_pass_synth: the reference-order Gram needs the rows resident (use the tensor order)");
    b->pending_center = false;
    b->stats_valid = false;
    c->have_gram = false;
    c->local_valid = false;
    c->dmat_local = false;
    c->K = K;
    const std::vector<StreamChunk> chunks = stream_chunks(b, chunk_rows, !src.synth);
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
    double* vm = b->varmax.get<double>(b->n_vars + 1, "varmax");
    double* ds = c->scales.get<double>(b->n_vars + 1, "scales");
    double* mn = b->means.get<double>(std::max<size_t>(b->rows, 1), "means");
    double* packed = c->packed.get<double>(count + 1, "packed");  // + status slot (0)
    double* ring = src.synth ? c->ring.get<double>(2 * static_cast<size_t>(first_rows) * b->ld, "chunk ring")
                             : nullptr;
    const bool staged = src.fd >= 0 || src.pageable;  // through the pinned ring
    const size_t slot_doubles = static_cast<size_t>(first_rows) * b->nt;
    double* fring = staged && !chunks.empty()
                        ? static_cast<double*>(c->file_ring.get(2 * slot_doubles * sizeof(double)))
                        : nullptr;
    std::vector<double> amps_v;  // per-variable amplitude slice for the generator
    if (src.synth && src.amps) amps_v.assign(src.amps, src.amps + b->n_vars);
    c->stream_gram_ms_events.clear();

    c->record(DOPINF_B200_STAGE_STREAM, 0);
    ck(cudaMemsetAsync(vm, 0, b->n_vars * sizeof(double), c->stream), "memset");
    if (ref_order) ck(cudaMemsetAsync(packed, 0, (count + 1) * sizeof(double), c->stream), "memset");
    ck(cudaMemsetAsync(gv, 0, count * b->n_vars * sizeof(double), c->stream), "memset");
    if (!src.synth) {
        // The copy stream must not overwrite the block before earlier work on it is done.
        cudaEvent_t ready = c->chunk_events[chunks.size()];
        ck(cudaEventRecord(ready, c->stream), "event");
        ck(cudaStreamWaitEvent(c->copy_stream, ready, 0), "event wait");
        if (staged && !chunks.empty()) staged_chunk_h2d(b, src, chunks, 0, fring, slot_doubles);
        for (size_t k = 0; !staged && k < chunks.size(); ++k) {
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
        if (!ref_order) {
            CUtensorMap map;
            ck(gram::make_tensor_map(&map, qk, ch.rows, K, b->ld), "tensor map");
            const gram::Plan plan = gram::make_stream_plan(ch.rows, K, c->num_sms, split_rows);
            if (ch.first_of_var) first_plan = plan;
            c->gram_event_pair();
            ck(gram::launch_gram(plan, map, tiles, work, counters, c->stream, !ch.first_of_var), "gram");
            c->gram_event_pair();
        }
        if (ch.last_of_var && ref_order) {
            const long long v0 = static_cast<long long>(ch.var) * static_cast<long long>(b->nx_i);
            if (scaling) {
                if (coll(c)) {
                    coll_allreduce(c, vm + ch.var, ds + ch.var, 1, ncclFloat64, ncclMax, "allreduce(MAX)");
                } else {
                    ck(cudaMemcpyAsync(ds + ch.var, vm + ch.var, sizeof(double), cudaMemcpyDeviceToDevice,
                                       c->stream),
                       "copy");
                }
                ck(transform::launch_apply(b->q + v0 * b->ld, b->ld, static_cast<long long>(b->nx_i), K,
                                           static_cast<long long>(b->nx_i), nullptr, ds + ch.var, c->num_sms,
                                           c->stream, /*skip_zero_scale=*/true),
                   "scale");
            }
            c->gram_event_pair();
            ck(gram::launch_gram_reference_order(b->q + v0 * b->ld, b->ld, static_cast<long long>(b->nx_i), K,
                                                 packed, ch.var > 0, c->stream),
               "gram (reference order)");
            c->gram_event_pair();
        } else if (ch.last_of_var) {
            const int groups = gram::reduce_groups(first_plan, c->num_sms);
            double* scratch =
                groups > 1 ? c->reduce_scratch.get<double>(gram::reduce_scratch_doubles(first_plan, groups),
                                                           "reduce scratch")
                           : nullptr;
            ck(gram::launch_reduce(first_plan, tiles, work, gv + static_cast<size_t>(ch.var) * count, c->stream,
                                   groups, scratch),
               "gram reduce");
            if (scaling) {
                if (coll(c)) {
                    coll_allreduce(c, vm + ch.var, ds + ch.var, 1, ncclFloat64, ncclMax, "allreduce(MAX)");
                } else {
                    ck(cudaMemcpyAsync(ds + ch.var, vm + ch.var, sizeof(double), cudaMemcpyDeviceToDevice,
                                       c->stream),
                       "copy");
                }
                if (!src.synth) {
                    const long long v0 = static_cast<long long>(ch.var) * static_cast<long long>(b->nx_i);
                    // the last variable's scaling runs on the copy stream (its copies are all
                    // done) beside the Gram combine and the downloads; the entry point joins it
                    cudaStream_t s = c->stream;
                    if (ch.var + 1 == static_cast<int>(b->n_vars)) {
                        cudaEvent_t ev = c->chunk_events[chunks.size()];
                        ck(cudaEventRecord(ev, c->stream), "event");
                        ck(cudaStreamWaitEvent(c->copy_stream, ev, 0), "event wait");
                        s = c->copy_stream;
                    }
                    ck(transform::launch_apply(b->q + v0 * b->ld, b->ld, static_cast<long long>(b->nx_i), K,
                                               static_cast<long long>(b->nx_i), nullptr, ds + ch.var, c->num_sms,
                                               s, /*skip_zero_scale=*/true),
                       "scale");
                }
            }
        }
        // the host reads chunk k + 1 while the device copies and reduces chunk k
        if (staged && k + 1 < chunks.size()) staged_chunk_h2d(b, src, chunks, k + 1, fring, slot_doubles);
    }
    // the pinned ring is free for the next call once the last copy has landed
    if (staged && !chunks.empty()) ck(cudaEventSynchronize(c->chunk_events[chunks.size() - 1]), "ring");
    if (b->rows == 0 && scaling) {  // an empty rank still joins the MAX collectives
        for (size_t v = 0; v < b->n_vars; ++v) {
            if (coll(c)) {
                coll_allreduce(c, vm + v, ds + v, 1, ncclFloat64, ncclMax, "allreduce(MAX)");
            } else {
                ck(cudaMemcpyAsync(ds + v, vm + v, sizeof(double), cudaMemcpyDeviceToDevice, c->stream), "copy");
            }
        }
    }
    if (!ref_order) {
        ck(gram::launch_combine_vars(gv, static_cast<int>(b->n_vars), count, scaling ? ds : nullptr, packed,
                                     c->stream),
           "combine");
    }
    ck(cudaMemsetAsync(packed + count, 0, sizeof(double), c->stream), "memset");
    c->record(DOPINF_B200_STAGE_STREAM, 1);
    c->local_valid = true;
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
    Nvtx nvtx_range("dopinf_b200 read_block");
    auto* c = b->ctx;
    b->pending_center = false;
    b->stats_valid = false;
    const long long chunk_rows = staged_rows(b->nt);
    const std::vector<StreamChunk> chunks = stream_chunks(b, chunk_rows, false);
    if (chunks.empty()) return;
    while (c->chunk_events.size() < chunks.size() + 1) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        c->chunk_events.push_back(e);
    }
    const size_t slot_doubles = static_cast<size_t>(std::min<long long>(chunk_rows, b->nx_i)) * b->nt;
    auto* fring = static_cast<double*>(c->file_ring.get(2 * slot_doubles * sizeof(double)));
    c->record(DOPINF_B200_STAGE_UPLOAD, 0);
    cudaEvent_t ready = c->chunk_events[chunks.size()];
    ck(cudaEventRecord(ready, c->stream), "event");
    ck(cudaStreamWaitEvent(c->copy_stream, ready, 0), "event wait");
    for (size_t k = 0; k < chunks.size(); ++k) staged_chunk_h2d(b, src, chunks, k, fring, slot_doubles);
    ck(cudaStreamWaitEvent(c->stream, c->chunk_events[chunks.size() - 1], 0), "event wait");
    c->record(DOPINF_B200_STAGE_UPLOAD, 1);
    ck(cudaEventSynchronize(c->chunk_events[chunks.size() - 1]), "ring");
}

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

// Rows [row0, row0 + nrows) of the materialised block to pageable host memory
// through the pinned ring: the D2H of one slot overlaps the parallel copy out
// of the other.
void staged_download(dopinf_b200_block* b, size_t row0, size_t nrows, double* host, size_t host_ld) {
    auto* c = b->ctx;
    const size_t chunk = static_cast<size_t>(staged_rows(b->nt));
    const size_t slot_doubles = std::min(chunk, nrows) * b->nt;
    auto* ring = static_cast<double*>(c->file_ring.get(2 * slot_doubles * sizeof(double)));
    const size_t n = (nrows + chunk - 1) / chunk;
    ensure_events(c->chunk_events, 2);
    auto d2h = [&](size_t k) {
        const size_t r0 = k * chunk, rows = std::min(chunk, nrows - r0);
        ck(copy_rows(ring + (k % 2) * slot_doubles, b->nt, b->q + (row0 + r0) * b->ld, b->ld, b->nt, rows,
                     cudaMemcpyDeviceToHost, c->stream),
           "download");
        ck(cudaEventRecord(c->chunk_events[k % 2], c->stream), "event");
    };
    if (n > 0) d2h(0);
    for (size_t k = 0; k < n; ++k) {
        if (k + 1 < n) d2h(k + 1);
        ck(cudaEventSynchronize(c->chunk_events[k % 2]), "download");
        const size_t r0 = k * chunk, rows = std::min(chunk, nrows - r0);
        const double* slot = ring + (k % 2) * slot_doubles;
        // slot (pitch nt) -> host rows (pitch host_ld): the same parallel copy, mirrored
        const int th = static_cast<int>(std::min<size_t>(file_reader_threads(), std::max<size_t>(1, rows * b->nt >> 20)));
        auto part = [&](int i) {
            const size_t a = rows * i / th, e = rows * (i + 1) / th;
            if (host_ld == b->nt) {
                std::memcpy(host + (r0 + a) * host_ld, slot + a * b->nt, (e - a) * b->nt * sizeof(double));
            } else {
                for (size_t r = a; r < e; ++r)
                    std::memcpy(host + (r0 + r) * host_ld, slot + r * b->nt, b->nt * sizeof(double));
            }
        };
        parallel_for(th, part);
    }
}

// Block upload from pageable host rows through the pinned ring (parallel host
// copies ‖ pinned H2D): several times the driver's pageable copy rate.
void staged_upload(dopinf_b200_block* b, const double* host, size_t host_ld) {
    StreamSource src;
    src.host = host;
    src.host_ld = host_ld;
    src.pageable = true;
    do_block_read(b, src);
}


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
    constexpr size_t kPiece = size_t(4) << 20;
    const int n = static_cast<int>(std::min<size_t>(file_reader_threads(), (bytes + kPiece - 1) / kPiece));
    if (n <= 1) return pread_all(fd, dst, bytes, off);
    const size_t per = (bytes / n + 4095) / 4096 * 4096;
    std::vector<char> ok(n, 0);
    parallel_for(n, [&](int i) {
        const size_t b0 = std::min(bytes, per * i), b1 = std::min(bytes, per * (i + 1));
        ok[i] = pread_all(fd, static_cast<char*>(dst) + b0, b1 - b0, off + b0) ? 1 : 0;
    });
    return std::all_of(ok.begin(), ok.end(), [](char v) { return v != 0; });
}

namespace {
class HostPool {
public:
    explicit HostPool(int workers) {
        for (int i = 0; i < workers; ++i) std::thread([this] { loop(); }).detach();  // live until exit
    }
    void run(int n, const std::function<void(int)>& fn) {
        std::lock_guard<std::mutex> job(job_mu_);
        {
            std::lock_guard<std::mutex> lock(mu_);
            fn_ = &fn;
            n_ = n;
            next_ = 0;
            pending_ = n;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lock(mu_);
        done_.wait(lock, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }

private:
    void work() {
        for (;;) {
            int i;
            const std::function<void(int)>* fn;
            {
                std::lock_guard<std::mutex> lock(mu_);
                if (!fn_ || next_ >= n_) return;
                i = next_++;
                fn = fn_;
            }
            (*fn)(i);
            std::lock_guard<std::mutex> lock(mu_);
            if (--pending_ == 0) done_.notify_all();
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lock(mu_);
                cv_.wait(lock, [&] { return gen_ != seen; });
                seen = gen_;
            }
            work();
        }
    }
    std::mutex job_mu_, mu_;
    std::condition_variable cv_, done_;
    const std::function<void(int)>* fn_ = nullptr;
    int n_ = 0, next_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
};
}  // namespace

void parallel_for(int n, const std::function<void(int)>& fn) {
    if (n <= 1) {
        if (n == 1) fn(0);
        return;
    }
    static HostPool* pool = new HostPool(std::max(1, file_reader_threads() - 1));  // + the caller
    pool->run(n, fn);
}

}  // namespace capi
}  // namespace dopinf_b200

extern "C" {

int dopinf_b200_snapshot_pass_host(dopinf_b200_block* b, const double* host, size_t host_ld, int scaling,
                                   double* means, double* scales, double* d) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(host_ld >= b->nt && (b->rows == 0 || host), "snapshot_pass_host: bad host buffer");
        SideJoin join{c};
        StreamSource src;
        src.host = host;
        src.host_ld = host_ld;
        src.pageable = b->rows > 0 && !is_pinned(host);
        do_stream_pass(b, src, scaling != 0, means, scales);
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

int dopinf_b200_block_read(dopinf_b200_ctx* c, const char* path, size_t row_begin, size_t row_end,
                           dopinf_b200_block** out) {
    if (!out) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    dopinf_b200_block* b = nullptr;
    const int rc = guarded(c, [&] {
        SideJoin join{c};
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
        SideJoin join{c};
        Fd f;
        Snp1 h;
        b = open_file_block(c, path, row_begin, row_end, f, h);
        StreamSource src;
        src.fd = f.fd;
        src.file = &h;
        const std::string p(path);
        src.path = &p;
        do_stream_pass(b, src, scaling != 0, means, scales);
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
                join_stream(b.ctx, b.ctx->stream);
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
        do_global_gram(c, d);
        c->sync("stream_pass_synth");
    });
}

}  // extern "C"
