// dopinf_b200_pipeline.hpp — the reference's pipeline::run_rank / run
// (proj/src/pipeline.cpp:229-398, pipeline.hpp:41-74) with the snapshot pass
// kept on the B200 from the file to the field: Steps I–III are one streamed
// call per rank (file ‖ H2D ‖ transform ‖ Gram, dopinf_b200_snapshot_pass_file)
// or, when the ranks share a GPU, the resident stage chain over the caller's
// Comm; the projection reads the device-resident D; the probes and the
// per-rank field file come from the resident block. The eigensolve, rank
// selection and the OpInf/ROM search stay on the reference path (north star)
// unless Options asks for their device versions. The artifacts are the
// reference's, in its formats and file names.
//
// Drop-in: include after the reference's headers and dopinf_b200.hpp, then
// call dopinf_b200::pipeline::run(cfg) where the reference calls
// pipeline::run(cfg). With Options::gram_order = DOPINF_B200_GRAM_ORDER_REFERENCE
// every artifact but the timings is the reference's byte for byte (the field
// file within 1e-15: its Φ_r·Q̃ᵀ runs on the tensor pipe); tests/cpp/parity_main.cpp
// checks that on BASELINE config 1.
#pragma once

#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <mutex>
#include <optional>
#include <string>
#include <vector>

#include "dopinf/artifacts.hpp"
#include "dopinf/data.hpp"
#include "dopinf/errors.hpp"
#include "dopinf/kernels.hpp"
#include "dopinf/opinf.hpp"
#include "dopinf/pipeline.hpp"
#include "dopinf/pod.hpp"
#include "dopinf/postprocess.hpp"
#include "dopinf/rom_search.hpp"
#include "dopinf/transform.hpp"
#include "dopinf_b200.hpp"

namespace dopinf_b200 {
namespace pipeline {

struct Options {
    int device = 0;                                  // the GPU every rank of this process binds
    int gram_order = DOPINF_B200_GRAM_ORDER_TENSOR;  // _REFERENCE: D bit-identical to the reference
    bool device_eig = false;                         // pod::eig_sym_desc / reduced_map on the device
    bool device_search = false;                      // rom_search::grid_search on the device
};

namespace detail {
namespace ref = ::dopinf;

// pipeline.cpp:94-107 check_probes (same ConfigError text).
inline void check_probes(const ref::postprocess::ProbeSet& probes, const ref::data::SnapshotHeader& h) {
    for (const auto& p : probes) {
        if (p.var >= h.n_vars) {
            throw ref::ConfigError("probe variable " + std::to_string(p.var) + " out of range (file has " +
                                   std::to_string(h.n_vars) + " variables)");
        }
        if (p.index >= h.nx) {
            throw ref::ConfigError("probe index " + std::to_string(p.index) + " out of range (nx = " +
                                   std::to_string(h.nx) + ")");
        }
    }
}

// pipeline.cpp:109-126 resolve_nt_p / check_fixed_rank.
inline std::size_t resolve_nt_p(const ref::pipeline::PipelineConfig& cfg, const ref::data::SnapshotHeader& h) {
    const std::size_t nt_p = cfg.nt_p == 0 ? h.nt : cfg.nt_p;
    if (nt_p < h.nt) {
        throw ref::ConfigError("nt_p = " + std::to_string(nt_p) + " is shorter than the training horizon nt = " +
                               std::to_string(h.nt));
    }
    return nt_p;
}

inline void check_fixed_rank(const ref::pipeline::PipelineConfig& cfg, const ref::data::SnapshotHeader& h) {
    if (cfg.fixed_rank > 0 && static_cast<std::uint64_t>(cfg.fixed_rank) > h.nt) {
        throw ref::ConfigError("rank = " + std::to_string(cfg.fixed_rank) + " exceeds the snapshot count nt = " +
                               std::to_string(h.nt));
    }
}

// pipeline.cpp:128-139: probe artifact names and owners.
inline std::string probe_file_name(const ref::postprocess::Probe& p) {
    return "probe_v" + std::to_string(p.var) + "_g" + std::to_string(p.index) + ".bin";
}

inline int probe_owner(const ref::data::PartitionPlan& plan, const ref::postprocess::Probe& p) {
    for (std::size_t r = 0; r < plan.size(); ++r) {
        if (p.index >= plan[r].begin && p.index < plan[r].end) return static_cast<int>(r);
    }
    return -1;
}

// pipeline.cpp:77-91: %.17g reals, comma-joined lists.
inline std::string real17(double v) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

inline std::string reals17(const std::vector<double>& v) {
    std::string out;
    for (std::size_t i = 0; i < v.size(); ++i) out += (i ? "," : "") + real17(v[i]);
    return out;
}

// pipeline.cpp:145-172: resolved.cfg in the reference's key order and format.
inline void write_resolved(const std::string& path, const ref::pipeline::PipelineConfig& cfg, int workers) {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw ref::DataFormatError("cannot create resolved config: " + path);
    out << "data = " << cfg.data_path << '\n' << "workers = " << workers << '\n';
    out << "backend = " << ref::kernels::backend_name(ref::kernels::active()) << '\n';
    if (cfg.fixed_rank > 0) {
        out << "rank = " << cfg.fixed_rank << '\n';
    } else {
        out << "energy = " << real17(cfg.energy) << '\n';
    }
    out << "scaling = " << (cfg.scaling ? "on" : "off") << '\n';
    out << "b1 = " << reals17(cfg.b1) << '\n' << "b2 = " << reals17(cfg.b2) << '\n';
    out << "max_growth = " << real17(cfg.max_growth) << '\n' << "nt_p = " << cfg.nt_p << '\n';
    if (!cfg.probes.empty()) {
        out << "probes = ";
        for (std::size_t i = 0; i < cfg.probes.size(); ++i) {
            out << (i ? "," : "") << cfg.probes[i].var << ':' << cfg.probes[i].index;
        }
        out << '\n';
    }
    out << "field = " << (cfg.write_field ? "on" : "off") << '\n' << "out = " << cfg.out_dir << '\n';
}

// pipeline.cpp:174-190: timings.csv.
inline void write_timings(const std::string& path, const ref::pipeline::RunResult& res, int size) {
    std::ofstream out(path, std::ios::trunc);
    if (!out) throw ref::DataFormatError("cannot create timing file: " + path);
    out << "rank,stage,seconds\n";
    for (int rank = 0; rank < size; ++rank) {
        for (std::size_t s = 0; s < ref::pipeline::kStageCount; ++s) {
            out << rank << ',' << ref::pipeline::kStageNames[s] << ','
                << real17(res.stage_seconds[static_cast<std::size_t>(rank) * ref::pipeline::kStageCount + s]) << '\n';
        }
    }
    out << res.owner_rank << ",rom_winner," << real17(res.rom_seconds) << '\n';
}

inline double stage(const Context& c, dopinf_b200_stage s) { return c.stage_ms(s) * 1e-3; }
}  // namespace detail

// pipeline::run_rank (pipeline.cpp:229-398) for the rank `comm` describes, on
// the Context bound to this thread.
inline ::dopinf::pipeline::RunResult run_rank(const ::dopinf::pipeline::PipelineConfig& cfg,
                                              ::dopinf::comm::Comm& comm, const Options& opt = {}) {
    namespace ref = ::dopinf;
    namespace fs = std::filesystem;
    using clock = std::chrono::steady_clock;
    Context& ctx = ::dopinf_b200::detail::ctx();
    const int rank = comm.rank(), size = comm.size();
    const fs::path out_dir(cfg.out_dir);
    fs::create_directories(out_dir);

    ref::pipeline::RunResult result;
    result.stage_seconds.assign(static_cast<std::size_t>(size) * ref::pipeline::kStageCount, 0.0);
    double* my = result.stage_seconds.data() + static_cast<std::size_t>(rank) * ref::pipeline::kStageCount;
    auto since = [](clock::time_point t0) { return std::chrono::duration<double>(clock::now() - t0).count(); };

    // Step I: header and plan (the reference's own checks and messages).
    auto t0 = clock::now();
    const ref::data::SnapshotHeader header = data::read_header<ref::data::SnapshotHeader>(cfg.data_path);
    detail::check_probes(cfg.probes, header);
    detail::check_fixed_rank(cfg, header);
    const ref::data::PartitionPlan plan = data::partition_rows<ref::data::RowRange>(header.nx, size);
    const std::size_t nt_p = detail::resolve_nt_p(cfg, header);
    const ref::data::RowRange rr = plan[static_cast<std::size_t>(rank)];
    const std::size_t nx_i = rr.count(), nt = header.nt, rows = header.n_vars * nx_i;
    result.n_vars = header.n_vars;
    result.nx = header.nx;
    result.nt = nt;
    result.nt_p = nt_p;

    // Steps I–III on the device. One streamed call when the Context's ranks are
    // the Comm's (or there is one rank); the resident stage chain over the
    // caller's Comm when the ranks share a GPU through size-1 Contexts.
    ref::transform::TransformParams params;
    params.scaling_enabled = cfg.scaling;
    ref::Matrix gram(nt, nt);
    std::optional<DeviceBlock> block;
    if (ctx.size() == size) {
        params.local_means.resize(rows);
        std::vector<double> scales(header.n_vars);
        dopinf_b200_block* b = nullptr;
        Context::check_exact(dopinf_b200_snapshot_pass_file(ctx.handle(), cfg.data_path.c_str(), rr.begin, rr.end,
                                                            cfg.scaling ? 1 : 0, &b, params.local_means.data(),
                                                            scales.data(), gram.data()),
                             ctx.handle());
        block.emplace(ctx, b);
        if (cfg.scaling) params.scales = scales;
        // the streamed call overlaps the read with the device stages: report the
        // device stage times and the rest of the wall time as the load
        const double total = since(t0);
        my[2] = detail::stage(ctx, DOPINF_B200_STAGE_STREAM_GRAM) + detail::stage(ctx, DOPINF_B200_STAGE_ALLREDUCE);
        my[1] = std::max(0.0, detail::stage(ctx, DOPINF_B200_STAGE_STREAM) - my[2]);
        my[0] = std::max(0.0, total - my[1] - my[2]);
    } else {
        block.emplace(data::read_block_device(cfg.data_path, plan, rank, header));
        my[0] = since(t0);
        t0 = clock::now();
        params.local_means = transform::center_in_place(*block);
        if (cfg.scaling) {
            params.scales = transform::compute_global_scales(*block, header, comm);
            transform::scale_in_place(*block, params.scales);
        }
        my[1] = since(t0);
        t0 = clock::now();
        gram = pod::global_gram(pod::local_gram<ref::Matrix>(*block), comm);
        my[2] = since(t0);
    }

    // Step III (replicated): eigensolve, rank, T_r on the reference path (or the
    // device's, from the resident D), Q̂ = T_rᵀD on the device.
    t0 = clock::now();
    ref::pod::EigenSpectrum spectrum;
    ref::Matrix tr, qhat;
    if (opt.device_eig) {
        spectrum = pod::eig_sym_desc<ref::pod::EigenSpectrum>(gram);
    } else {
        spectrum = ref::pod::eig_sym_desc(gram);
    }
    if (cfg.fixed_rank > 0) {
        result.r = static_cast<std::size_t>(cfg.fixed_rank);
    } else {
        const ref::pod::RankSelection sel = ref::pod::select_rank(spectrum.eigenvalues, cfg.energy);
        result.r = sel.r;
        result.rank_capped = sel.capped;
    }
    result.retained = ref::pod::retained_energy(spectrum.eigenvalues, result.r);
    tr = opt.device_eig ? pod::reduced_map_device<ref::Matrix>(nt, result.r) : ref::pod::reduced_map(spectrum, result.r);
    qhat = pod::project(tr, gram);
    my[3] = since(t0);

    // Step IV: the regularisation search.
    t0 = clock::now();
    const ref::rom_search::SearchConfig search{cfg.b1, cfg.b2, cfg.max_growth, nt_p};
    const ref::rom_search::SearchOutcome outcome =
        opt.device_search ? rom_search::grid_search<ref::rom_search::SearchOutcome>(qhat, search, comm)
                          : ref::rom_search::grid_search(qhat, search, comm);
    my[4] = since(t0);
    result.pair_opt = outcome.pair_opt;
    result.train_err = outcome.train_err;
    result.owner_rank = outcome.owner_rank;
    result.rom_seconds = outcome.rom_seconds;

    // Step V: per-rank artifacts from the resident block.
    t0 = clock::now();
    {
        std::vector<ref::artifacts::NamedMatrix> blobs;
        blobs.push_back({"means", ref::Matrix(1, params.local_means.size(), params.local_means)});
        if (cfg.scaling) blobs.push_back({"scales", ref::Matrix(1, params.scales.size(), params.scales)});
        blobs.push_back({"range", ref::Matrix(1, 2, {static_cast<double>(rr.begin), static_cast<double>(rr.end)})});
        ref::artifacts::write_blobs((out_dir / ("transform_rank" + std::to_string(rank) + ".bin")).string(), blobs);
        const auto series = postprocess::reconstruct_probes<ref::postprocess::ProbeSeries>(*block, tr, outcome.trajectory,
                                                                                          cfg.probes, params);
        for (const auto& s : series) {
            ref::artifacts::write_raw_vector((out_dir / detail::probe_file_name(s.probe)).string(), s.values);
        }
        if (cfg.write_field) {
            std::string names;
            for (const auto& n : header.var_names) names += n + std::string(1, '\0');
            const std::string path = (out_dir / ("field_rank" + std::to_string(rank) + ".snp1")).string();
            Context::check_exact(dopinf_b200_write_field(block->handle(), tr.data(), result.r,
                                                         outcome.trajectory.data(), nt_p, params.local_means.data(),
                                                         cfg.scaling ? params.scales.data() : nullptr,
                                                         cfg.scaling ? 1 : 0, names.data(), path.c_str()),
                                 ctx.handle());
        }
    }
    my[5] = since(t0);
    block.reset();

    // the whole-group timing table (pipeline.cpp:354-355)
    comm.allreduce(result.stage_seconds, ref::comm::ReduceOp::Sum);

    if (rank == 0) {  // pipeline.cpp:357-396
        ref::artifacts::write_result((out_dir / "result.txt").string(), result.pair_opt, result.r, result.train_err);
        const std::vector<double> gamma =
            ref::opinf::build_regularizer(result.r, ref::opinf::quad_len(result.r), result.pair_opt);
        const ref::opinf::ReducedOperators ops = ref::opinf::solve_opinf(ref::opinf::assemble_data(qhat), gamma);
        ref::artifacts::write_blobs((out_dir / "operators.bin").string(),
                                    {{"A", ops.a}, {"F", ops.f}, {"c", ref::Matrix(1, ops.c.size(), ops.c)}});
        ref::artifacts::write_blobs((out_dir / "reduced_map.bin").string(), {{"Tr", tr}});
        ref::artifacts::write_blobs((out_dir / "trajectory.bin").string(), {{"Qtilde", outcome.trajectory}});
        std::ofstream probe_manifest((out_dir / "probes_manifest.txt").string(), std::ios::trunc);
        for (const auto& p : cfg.probes) {
            probe_manifest << "var=" << p.var << " index=" << p.index << " owner=" << detail::probe_owner(plan, p)
                           << " file=" << detail::probe_file_name(p) << " steps=" << nt_p << '\n';
        }
        if (cfg.write_field) {
            std::ofstream field_manifest((out_dir / "field_manifest.txt").string(), std::ios::trunc);
            for (int r = 0; r < size; ++r) {
                const ref::data::RowRange range = plan[static_cast<std::size_t>(r)];
                field_manifest << "rank=" << r << " file=field_rank" << r << ".snp1 rows=" << range.begin << ':'
                               << range.end << " vars=" << header.n_vars << " steps=" << nt_p << '\n';
            }
        }
        ref::pipeline::PipelineConfig resolved = cfg;
        resolved.nt_p = nt_p;
        detail::write_resolved((out_dir / "resolved.cfg").string(), resolved, size);
        detail::write_timings((out_dir / "timings.csv").string(), result, size);
    }
    return result;
}

// pipeline::run (pipeline.cpp:400-414): cfg.workers in-process ranks sharing
// the process's GPU, each with a size-1 Context (the reference's Comm carries
// the MAX and the Gram SUM in ascending rank order).
inline ::dopinf::pipeline::RunResult run(const ::dopinf::pipeline::PipelineConfig& cfg, const Options& opt = {}) {
    if (!::dopinf::kernels::set_backend(cfg.kernels_backend)) {
        throw ::dopinf::ConfigError("kernel backend '" + cfg.kernels_backend + "' is not available on this machine");
    }
    ::dopinf::pipeline::RunResult shared;
    std::mutex mu;
    ::dopinf::comm::run_on_workers(cfg.workers, [&](::dopinf::comm::Comm& comm) {
        Context ctx(opt.device);
        ctx.set_gram_order(opt.gram_order);
        Bind bind(ctx);
        ::dopinf::pipeline::RunResult mine = run_rank(cfg, comm, opt);
        if (comm.rank() == 0) {
            std::lock_guard<std::mutex> lock(mu);
            shared = std::move(mine);
        }
    });
    return shared;
}

}  // namespace pipeline
}  // namespace dopinf_b200
