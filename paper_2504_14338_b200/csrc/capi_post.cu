// capi_post.cu — the C ABI after the projection: the OpInf grid search
// (reference rom_search.cpp / opinf.cpp) and Step V field reconstruction with
// its streamed SNP1 field writer (postprocess.cpp, pipeline.cpp:330-350).
#include "capi_internal.h"

namespace dopinf_b200 {
namespace capi {

namespace {

// ---- Step IV: OpInf grid search (rom_search.cpp:185-262) --------------------
// Host span all-reduce over NCCL (comm::allreduce_scalar's role).
void host_allreduce(dopinf_b200_ctx* c, double* data, size_t count, ncclRedOp_t op) {
    double* buf = c->span.get<double>(count, "span");
    ck(cudaMemcpyAsync(buf, data, count * sizeof(double), cudaMemcpyHostToDevice, c->stream), "H2D");
    coll_allreduce(c, buf, buf, count, ncclFloat64, op, "allreduce");
    double* pin = c->small_pinned<double>(count);
    ck(cudaMemcpyAsync(pin, buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
    c->sync("allreduce");
    std::memcpy(data, pin, count * sizeof(double));
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
    Nvtx nvtx_range("dopinf_b200 grid_search");
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

    const size_t n_reg = n1 * n2;
    double best_err = std::numeric_limits<double>::infinity();
    size_t best = n_reg;
    double n_diverged = 0.0, n_growth = 0.0, rom_ms = 0.0;
    std::vector<double> best_traj;
    // This rank's share; a failure here still reaches the first collective
    // below, so the peers raise "rank r aborted" rather than wait out the deadline.
    const std::optional<Fail> own = attempt(c, [&] {
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
        // DhatᵀDhat: bit-identical to linalg::gram (FMA chains) up to d = 2048;
        // larger systems on the tensor-pipe Gram kernel
        if (D <= 2048) {
            ck(rom::launch_gram_exact(dhat, ldd, KK, D, g, c->stream), "dhat gram");
        } else {
            rom_gram(c, dhat, ldd, KK, D, g);
        }
        ck(rom::launch_rhs(dhat, ldd, q2t, KK, D, R, rhs, c->stream), "rhs");

        // this rank's candidates, solved / integrated / scored in batches that fit
        size_t pb = 0, pe = 0;
        if (dopinf_b200_distribute_pairs(n_reg, c->rank, c->size, &pb, &pe) != DOPINF_B200_OK) {
            fail(DOPINF_B200_ERR_INVALID_ARGUMENT, g_thread_err);
        }
        const std::pair<size_t, size_t> mine(pb, pe);
        const size_t np = mine.second - mine.first;
        const size_t per_pair = static_cast<size_t>(D) * D + static_cast<size_t>(D) * r + nt_p * r;
        size_t batch = std::max<size_t>(1, std::min<size_t>(std::max<size_t>(np, 1),
                                                             (size_t(8) << 30) / (per_pair * sizeof(double))));
        if (const char* env = std::getenv("DOPINF_B200_GRID_BATCH")) {  // test knob: pairs per batch
            const long long v = std::atoll(env);
            if (v > 0) batch = std::min<size_t>(batch, static_cast<size_t>(v));
        }
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
            // Cholesky factors over concurrent cuSOLVER lanes, then every pair's
            // triangular solves in one launch (shared-memory substitution); systems
            // beyond the shared-memory solve use cuSOLVER's potrs per pair
            if (D <= 1760) {
                if (c->solver.cholesky(lhs, D, static_cast<int>(nb), info, c->stream, &err) != cudaSuccess) {
                    fail(DOPINF_B200_ERR_DEVICE, err);
                }
                ck(rom::launch_chol_solve(lhs, D, static_cast<int>(nb), rhsb, R, c->stream), "cholesky solve");
            } else if (c->solver.spd_solve(lhs, D, static_cast<int>(nb), rhsb, R, info, c->stream, &err) != cudaSuccess) {
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

    });

    // agree on the winner across ranks (rom_search.cpp:227-261)
    GridOutcome out;
    double global_min = best_err;
    if (coll(c)) {
        // MIN of the errors, and of (failed ? rank : size): the lowest failed rank
        std::vector<double> v = {own ? std::numeric_limits<double>::infinity() : best_err,
                                 static_cast<double>(own ? c->rank : c->size)};
        host_allreduce(c, v.data(), 2, ncclMin);
        global_min = v[0];
        settle(own, v[1] < c->size ? static_cast<int>(v[1]) : -1);
    }
    if (global_min == std::numeric_limits<double>::infinity()) {
        std::vector<double> counts = {n_diverged, n_growth};
        if (coll(c)) host_allreduce(c, counts.data(), 2, ncclSum);
        fail(DOPINF_B200_ERR_NO_ADMISSIBLE_PAIR,
             "no admissible regularization pair among " + std::to_string(n_reg) + " candidates (" +
                 std::to_string(static_cast<long>(counts[0])) + " diverged, " +
                 std::to_string(static_cast<long>(counts[1])) + " exceeded growth bound " +
                 std::to_string(max_growth) + ")");
    }
    int owner = 0;
    if (coll(c)) {
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
    if (coll(c)) {
        double* dp = c->rom_packet.get<double>(packet.size(), "packet");
        ck(cudaMemcpyAsync(dp, packet.data(), packet.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream),
           "packet H2D");
        coll_broadcast(c, dp, packet.size(), ncclFloat64, owner, "broadcast");
        double* pin = c->small_pinned<double>(packet.size());
        ck(cudaMemcpyAsync(pin, dp, packet.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream),
           "packet D2H");
        c->sync("broadcast");
        std::memcpy(packet.data(), pin, packet.size() * sizeof(double));
    }
    out.beta1 = packet[0];
    out.beta2 = packet[1];
    out.rom_seconds = packet[2];
    out.train_err = global_min;
    out.owner = owner;
    if (traj_host) std::memcpy(traj_host, packet.data() + 3, nt_p * r * sizeof(double));
    return out;
}

// Field operands on the device: Q̃ (nt_p × r) padded to the Φ_r pitch with
// zeros, the means and (scaling) the scales of the transform.
struct FieldOperands {
    const double* qt = nullptr;
    const double* means = nullptr;
    const double* scales = nullptr;
    size_t nt_p = 0;
    int r_pad = 0;  // pitch of Φ_r and Q̃ on the device
    int k_ext = 0;  // contraction extent: r rounded up to the DMMA k-step of 4 (columns ≥ r are zero)
};

FieldOperands field_operands(dopinf_b200_block* b, const double* qtilde, size_t r, size_t nt_p, int r_pad,
                             const double* means, const double* scales, bool scaling) {
    auto* c = b->ctx;
    FieldOperands f;
    f.nt_p = nt_p;
    f.r_pad = r_pad;
    f.k_ext = static_cast<int>((r + 3) / 4 * 4);
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
    for (int k0 = 0; k0 < f.k_ext; k0 += slab) {
        const int w = std::min(slab, f.k_ext - k0);
        const bool last = k0 + w == f.k_ext;
        ck(field::launch_field(phi + k0, f.r_pad, f.qt + k0, f.r_pad, nrows, static_cast<int>(f.nt_p), w,
                               last && f.means ? f.means + row0 : nullptr, last ? f.scales : nullptr,
                               static_cast<long long>(b->nx_i), row0, out, ldo, k0 > 0 ? 1 : 0, c->num_sms,
                               c->stream),
           "field");
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

// Stream the field into an SNP1 file: chunk k is computed into device slot
// k % 2, copied (copy stream) into pinned slot k % 2, and written by the host
// while chunk k + 1 computes. Layout = data::write_snapshots (data.cpp:118-129):
// the field's rows are the variables' rows in order.
void write_field_file(dopinf_b200_block* b, const FieldOperands& f, const Snp1& h, const std::string& path) {
    Nvtx nvtx_range("dopinf_b200 write_field");
    auto* c = b->ctx;
    Fd fd;
    // No O_TRUNC: rewriting a field file of the previous run in place (then
    // ftruncate to the exact size) spares ext4 freeing every block at open and
    // flushing the replaced file at close; the bytes are the same.
    fd.fd = open(path.c_str(), O_WRONLY | O_CREAT | O_CLOEXEC, 0644);
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
    // 32 MB row chunks: the host's parallel writes of chunk k overlap chunk k+1's
    // compute and D2H, the first write starts early, and the pinned ring (2 slots,
    // shared with the file reads) stays small — page-locking is ~0.1 s per 100 MB
    size_t ch = std::max<size_t>(128, (size_t(32) << 20) / (nt_p * sizeof(double))) / 128 * 128;
    // reuse the pinned ring a file pass left if its slots hold >= 1024 rows
    // (re-pinning a larger ring costs more than the smaller chunks do)
    const size_t have = c->file_ring.bytes / (2 * nt_p * sizeof(double)) / 128 * 128;
    if (have >= 1024) ch = std::min(ch, have);
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
    if (ftruncate(fd.fd, static_cast<off_t>(data_off + rows * nt_p * sizeof(double))) != 0) {
        format_fail("write failed: " + path);
    }
    c->record(DOPINF_B200_STAGE_FIELD, 1);
    if (close(fd.fd) != 0) {
        fd.fd = -1;
        format_fail("write failed: " + path);
    }
    fd.fd = -1;
}

}  // namespace

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
    constexpr size_t kPiece = size_t(4) << 20;
    const int n = static_cast<int>(std::min<size_t>(file_reader_threads(), (bytes + kPiece - 1) / kPiece));
    if (n <= 1) return write_all(static_cast<const char*>(src), bytes, off);
    const size_t per = (bytes / n + 4095) / 4096 * 4096;
    std::vector<char> ok(n, 0);
    parallel_for(n, [&](int i) {
        const size_t b0 = std::min(bytes, per * i), b1 = std::min(bytes, per * (i + 1));
        ok[i] = write_all(static_cast<const char*>(src) + b0, b1 - b0, off + b0) ? 1 : 0;
    });
    return std::all_of(ok.begin(), ok.end(), [](char v) { return v != 0; });
}

}  // namespace capi
}  // namespace dopinf_b200

extern "C" {

int dopinf_b200_distribute_pairs(size_t n_reg, int rank, int size, size_t* begin, size_t* end) {
    return guarded_free([&] {
        if (n_reg < 1) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "distribute_pairs: no candidates");
        if (size < 1 || rank < 0 || rank >= size) fail(DOPINF_B200_ERR_INVALID_ARGUMENT, "distribute_pairs: bad rank/size");
        require(begin && end, "distribute_pairs: null outputs");
        const size_t ranks = static_cast<size_t>(size), rk = static_cast<size_t>(rank);
        if (ranks > n_reg) {
            *begin = rk < n_reg ? rk : n_reg;
            *end = rk < n_reg ? rk + 1 : n_reg;
            return;
        }
        const size_t base = n_reg / ranks;
        *begin = rk * base;
        *end = (rk + 1 == ranks) ? n_reg : (rk + 1) * base;
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

int dopinf_b200_reconstruct_probes(dopinf_b200_block* b, const double* tr, size_t r, const double* qtilde,
                                   size_t nt_p, const size_t* var, const size_t* index, size_t n_probes,
                                   const double* means, const double* scales, int scaling, double* series,
                                   int* owned) {
    if (!b) return DOPINF_B200_ERR_INVALID_ARGUMENT;
    auto* c = b->ctx;
    return guarded(c, [&] {
        require(n_probes == 0 || (var && index), "reconstruct_probes: null probe arrays");
        require(qtilde != nullptr && r >= 1, "reconstruct_probes: null trajectory");
        require(b->rows == 0 || means != nullptr, "reconstruct_probes: null means");
        require(!scaling || scales != nullptr, "reconstruct_probes: null scales");
        // the owned probes' local rows, in probe order (postprocess.cpp:42-48)
        std::vector<long long> rows;
        std::vector<size_t> which;
        for (size_t i = 0; i < n_probes; ++i) {
            const bool mine = index[i] >= b->row_begin && index[i] < b->row_begin + b->nx_i;
            if (owned) owned[i] = mine ? 1 : 0;
            if (!mine) continue;
            const size_t row = var[i] * b->nx_i + (index[i] - b->row_begin);
            if (row >= b->rows) {  // basis_rows' check (postprocess.cpp:20-23)
                fail(DOPINF_B200_ERR_INVALID_ARGUMENT,
                     "basis_rows: row " + std::to_string(row) + " outside the local block");
            }
            rows.push_back(static_cast<long long>(row));
            which.push_back(i);
        }
        if (rows.empty()) return;
        materialize(b);
        const int nsel = static_cast<int>(rows.size());
        const double* dtr = tr_operand(c, tr, b->nt, r);
        long long* dsel = c->sel.get<long long>(rows.size(), "sel");
        double* dbasis = c->rows_out.get<double>(rows.size() * r, "probe basis");
        double* dqt = c->field_qt.get<double>(nt_p * r, "qtilde");
        double* dm = c->field_means.get<double>(b->rows, "means");
        double* ds = scaling ? c->field_scales.get<double>(b->n_vars, "scales") : nullptr;
        double* dout = c->field_ring.get<double>(rows.size() * nt_p, "probe series");
        ck(cudaMemcpyAsync(dsel, rows.data(), rows.size() * sizeof(long long), cudaMemcpyHostToDevice, c->stream),
           "rows H2D");
        ck(cudaMemcpyAsync(dqt, qtilde, nt_p * r * sizeof(double), cudaMemcpyHostToDevice, c->stream), "qtilde H2D");
        ck(cudaMemcpyAsync(dm, means, b->rows * sizeof(double), cudaMemcpyHostToDevice, c->stream), "means H2D");
        if (ds) {
            ck(cudaMemcpyAsync(ds, scales, b->n_vars * sizeof(double), cudaMemcpyHostToDevice, c->stream),
               "scales H2D");
        }
        ck(project::launch_basis_rows(b->q, b->ld, static_cast<int>(b->nt), dtr, static_cast<int>(r), dsel, nsel,
                                      dbasis, c->stream),
           "basis_rows");
        ck(project::launch_probe_series(dbasis, static_cast<int>(r), dqt, static_cast<int>(nt_p), dsel, dm, ds,
                                        static_cast<long long>(b->nx_i), nsel, dout, c->stream),
           "probe series");
        std::vector<double> h(rows.size() * nt_p);
        ck(cudaMemcpyAsync(h.data(), dout, h.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream), "D2H");
        c->sync("reconstruct_probes");
        for (size_t k = 0; k < which.size(); ++k) {
            std::memcpy(series + which[k] * nt_p, &h[k * nt_p], nt_p * sizeof(double));
        }
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

}  // extern "C"
