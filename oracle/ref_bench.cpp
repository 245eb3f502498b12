// ref_bench.cpp — extern "C" entry points over the UNMODIFIED reference
// (compiled from /root/reference/proj/src into oracle/_ref/libdopinf_ref.a).
// TEST INFRASTRUCTURE ONLY: used by tests/ (golden vectors, pins),
// __graft_entry__.smoke() and bench.py's reference / cpu_baseline legs.
// Each function calls the reference's own public API; nothing here
// re-implements reference arithmetic.
#include <chrono>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <vector>

#include "dopinf/comm.hpp"
#include "dopinf/data.hpp"
#include "dopinf/errors.hpp"
#include "dopinf/kernels.hpp"
#include "dopinf/linalg.hpp"
#include "dopinf/opinf.hpp"
#include "dopinf/pod.hpp"
#include "dopinf/postprocess.hpp"
#include "dopinf/rom_search.hpp"
#include "dopinf/synth.hpp"
#include "dopinf/transform.hpp"

using namespace dopinf;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const DegenerateVariableError*>(&e)) return 4;
    if (dynamic_cast<const CollectiveError*>(&e)) return 3;
    if (dynamic_cast<const PartitionError*>(&e)) return 2;
    if (dynamic_cast<const InvalidArgumentError*>(&e)) return 1;
    if (dynamic_cast<const NotPsdError*>(&e)) return 7;
    if (dynamic_cast<const RankDeficiencyError*>(&e)) return 8;
    if (dynamic_cast<const DataFormatError*>(&e)) return 10;
    if (dynamic_cast<const NoAdmissiblePairError*>(&e)) return 11;
    if (dynamic_cast<const SolveError*>(&e)) return 9;
    return 99;
}

Matrix to_matrix(const double* p, std::size_t rows, std::size_t cols) {
    return Matrix(rows, cols, std::vector<double>(p, p + rows * cols));
}

void from_matrix(const Matrix& m, double* out) {
    std::memcpy(out, m.data(), m.size() * sizeof(double));
}

data::SnapshotHeader header_for(std::size_t n_vars, std::size_t nx, std::size_t nt) {
    data::SnapshotHeader h;
    h.n_vars = n_vars;
    h.nx = nx;
    h.nt = nt;
    for (std::size_t j = 0; j < n_vars; ++j) h.var_names.push_back("var" + std::to_string(j));
    return h;
}

// Carve rank `rank`'s LocalBlock out of a full stacked (n_vars*nx) x nt
// matrix, with the on-disk layout (data.hpp:35-42).
data::LocalBlock slice(const double* full, std::size_t n_vars, std::size_t nx, std::size_t nt,
                       const data::PartitionPlan& plan, int rank) {
    const data::RowRange range = plan[static_cast<std::size_t>(rank)];
    const std::size_t nx_i = range.count();
    data::LocalBlock block;
    block.rank = rank;
    block.row_range = range;
    block.values = Matrix(n_vars * nx_i, nt);
    for (std::size_t j = 0; j < n_vars; ++j) {
        std::memcpy(block.values.row(j * nx_i), full + (j * nx + range.begin) * nt,
                    nx_i * nt * sizeof(double));
    }
    return block;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_set_backend(const char* name) { return kernels::set_backend(name) ? 0 : 1; }

const char* ref_backend() { return kernels::backend_name(kernels::active()); }

// synth::Rng stream (synth.cpp:15-34): `count` normals from Rng(seed).
void ref_rng_normals(unsigned long long seed, double* out, std::size_t count) {
    synth::Rng rng(seed);
    for (std::size_t i = 0; i < count; ++i) out[i] = rng.normal();
}

// Steps II-III of pipeline::run_rank (pipeline.cpp:270-280) on `workers`
// in-process ranks over the full stacked matrix `q` (transformed in place,
// rank slices written back). Stage seconds: [transform, gram_reduce], each
// between barrier() fences, max over ranks.
int ref_snapshot_pass(double* q, std::size_t n_vars, std::size_t nx, std::size_t nt,
                      int workers, int scaling, double* d_out, double* means_out,
                      double* scales_out, double* stage_seconds) {
    try {
        const data::SnapshotHeader header = header_for(n_vars, nx, nt);
        const data::PartitionPlan plan = data::partition_rows(nx, workers);
        std::mutex mu;
        double t_transform = 0.0, t_gram = 0.0;
        comm::run_on_workers(workers, [&](comm::Comm& comm) {
            using clock = std::chrono::steady_clock;
            data::LocalBlock block = slice(q, n_vars, nx, nt, plan, comm.rank());
            comm.barrier();
            const auto t0 = clock::now();
            std::vector<double> means = transform::center_in_place(block);
            std::vector<double> scales;
            if (scaling) {
                scales = transform::compute_global_scales(block, header, comm);
                transform::scale_in_place(block, scales);
            }
            comm.barrier();
            const auto t1 = clock::now();
            Matrix d = pod::global_gram(pod::local_gram(block), comm);
            comm.barrier();
            const auto t2 = clock::now();
            std::lock_guard lock(mu);
            t_transform = std::max(t_transform, std::chrono::duration<double>(t1 - t0).count());
            t_gram = std::max(t_gram, std::chrono::duration<double>(t2 - t1).count());
            const data::RowRange range = block.row_range;
            const std::size_t nx_i = range.count();
            for (std::size_t j = 0; j < n_vars; ++j) {
                std::memcpy(q + (j * nx + range.begin) * nt, block.values.row(j * nx_i),
                            nx_i * nt * sizeof(double));
                if (means_out) {
                    std::memcpy(means_out + j * nx + range.begin, means.data() + j * nx_i,
                                nx_i * sizeof(double));
                }
            }
            if (comm.rank() == 0) {
                if (d_out) from_matrix(d, d_out);
                if (scales_out && scaling) std::memcpy(scales_out, scales.data(), n_vars * 8);
            }
        });
        if (stage_seconds) {
            stage_seconds[0] = t_transform;
            stage_seconds[1] = t_gram;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// pod::global_gram(pod::local_gram(block)) on `workers` in-process ranks over
// a single-variable q (rows x cols), as tests/acceptance.cpp:240-257 runs it.
int ref_global_gram(const double* q, std::size_t rows, std::size_t cols, int workers, double* out) {
    try {
        const data::PartitionPlan plan = data::partition_rows(rows, workers);
        std::mutex mu;
        comm::run_on_workers(workers, [&](comm::Comm& comm) {
            data::LocalBlock block = slice(q, 1, rows, cols, plan, comm.rank());
            Matrix d = pod::global_gram(pod::local_gram(block), comm);
            if (comm.rank() == 0) {
                std::lock_guard lock(mu);
                from_matrix(d, out);
            }
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Per-rank local Gram only (pod.cpp:11-13), for pinning the oracle.
int ref_gram(const double* q, std::size_t rows, std::size_t cols, double* out) {
    try {
        from_matrix(linalg::gram(to_matrix(q, rows, cols)), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// transform::center_in_place on a single block (transform.cpp:10-20).
int ref_center(double* q, std::size_t rows, std::size_t cols, double* means) {
    try {
        data::LocalBlock block;
        block.row_range = {0, rows};
        block.values = to_matrix(q, rows, cols);
        std::vector<double> m = transform::center_in_place(block);
        from_matrix(block.values, q);
        std::memcpy(means, m.data(), rows * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// compute_global_scales + scale_in_place on one rank (transform.cpp:22-49).
int ref_scale(double* q, std::size_t n_vars, std::size_t nx_i, std::size_t cols,
              double* scales_out) {
    try {
        data::LocalBlock block;
        block.row_range = {0, nx_i};
        block.values = to_matrix(q, n_vars * nx_i, cols);
        const data::SnapshotHeader header = header_for(n_vars, nx_i, cols);
        int rc = 0;
        comm::run_on_workers(1, [&](comm::Comm& comm) {
            std::vector<double> s = transform::compute_global_scales(block, header, comm);
            transform::scale_in_place(block, s);
            std::memcpy(scales_out, s.data(), n_vars * sizeof(double));
        });
        from_matrix(block.values, q);
        return rc;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// pod::project (pod.cpp:103-105): Qhat = Tr' D.
int ref_project(const double* tr, const double* d, std::size_t nt, std::size_t r, double* out) {
    try {
        from_matrix(pod::project(to_matrix(tr, nt, r), to_matrix(d, nt, nt)), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// linalg::matmul (postprocess.cpp:66 reconstruct_field's Phi_r = Q Tr).
int ref_matmul(const double* a, std::size_t m, std::size_t k, const double* b, std::size_t nb,
               double* out) {
    try {
        from_matrix(linalg::matmul(to_matrix(a, m, k), to_matrix(b, k, nb)), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// postprocess::basis_rows (postprocess.cpp:12-34).
int ref_basis_rows(const double* q, std::size_t rows, std::size_t cols, const double* tr,
                   std::size_t r, const std::size_t* sel, std::size_t nsel, double* out) {
    try {
        data::LocalBlock block;
        block.row_range = {0, rows};
        block.values = to_matrix(q, rows, cols);
        std::vector<std::size_t> idx(sel, sel + nsel);
        from_matrix(postprocess::basis_rows(block, to_matrix(tr, cols, r), idx), out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// The consumer right after the hot path, on the reference path
// (pod.cpp:20-65 eig_sym_desc, :84-101 reduced_map): returns lambda (nt)
// and Tr (nt x r).
int ref_eig_reduced_map(const double* d, std::size_t nt, std::size_t r, double* lambda,
                        double* tr) {
    try {
        const pod::EigenSpectrum spec = pod::eig_sym_desc(to_matrix(d, nt, nt));
        std::memcpy(lambda, spec.eigenvalues.data(), nt * sizeof(double));
        if (r > 0) from_matrix(pod::reduced_map(spec, r), tr);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Steps IV of run_rank on one rank (rom_search.cpp:185-262): Qhat (r x nt)
// -> winning trajectory Qtilde (nt_p x r) and training error.
int ref_grid_search(const double* qhat, std::size_t r, std::size_t nt, const double* b1,
                    std::size_t n1, const double* b2, std::size_t n2, double max_growth,
                    std::size_t nt_p, double* qtilde, double* pair_err) {
    try {
        rom_search::SearchConfig cfg{std::vector<double>(b1, b1 + n1),
                                     std::vector<double>(b2, b2 + n2), max_growth, nt_p};
        const Matrix qh = to_matrix(qhat, r, nt);
        comm::run_on_workers(1, [&](comm::Comm& comm) {
            const rom_search::SearchOutcome out = rom_search::grid_search(qh, cfg, comm);
            from_matrix(out.trajectory, qtilde);
            pair_err[0] = out.pair_opt.beta1;
            pair_err[1] = out.pair_opt.beta2;
            pair_err[2] = out.train_err;
        });
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// data::write_snapshots (data.cpp:105-131): `names` holds n_vars NUL-terminated
// names back to back; `full` is the stacked (n_vars*nx) x nt matrix.
int ref_write_snapshots(const char* path, std::size_t n_vars, std::size_t nx, std::size_t nt,
                        const char* names, const double* full) {
    try {
        data::SnapshotHeader h;
        h.n_vars = n_vars;
        h.nx = nx;
        h.nt = nt;
        const char* p = names;
        for (std::size_t j = 0; j < n_vars; ++j) {
            h.var_names.emplace_back(p);
            p += h.var_names.back().size() + 1;
        }
        std::vector<Matrix> vars;
        for (std::size_t j = 0; j < n_vars; ++j) vars.push_back(to_matrix(full + j * nx * nt, nx, nt));
        data::write_snapshots(path, h, vars);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// data::read_header (data.cpp:133-162): dims out, names back to back.
int ref_read_header(const char* path, std::size_t* dims, char* names, std::size_t names_cap) {
    try {
        const data::SnapshotHeader h = data::read_header(path);
        dims[0] = h.n_vars;
        dims[1] = h.nx;
        dims[2] = h.nt;
        std::size_t at = 0;
        for (const auto& n : h.var_names) {
            if (at + n.size() + 1 > names_cap) return 1;
            std::memcpy(names + at, n.c_str(), n.size() + 1);
            at += n.size() + 1;
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// data::read_block (data.cpp:164-202) for rank `rank` of partition_rows(nx, p).
int ref_read_block(const char* path, int p, int rank, double* out) {
    try {
        const data::SnapshotHeader h = data::read_header(path);
        const data::PartitionPlan plan = data::partition_rows(h.nx, p);
        const data::LocalBlock b = data::read_block(path, plan, rank, h);
        from_matrix(b.values, out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// postprocess::reconstruct_field (postprocess.cpp:63-70) on one rank's
// transformed block q ((n_vars*nx_i) x nt) with T_r (nt x r), Q̃ (nt_p x r).
int ref_reconstruct_field(const double* q, std::size_t n_vars, std::size_t nx_i, std::size_t nt, const double* tr,
                          std::size_t r, const double* qtilde, std::size_t nt_p, const double* means,
                          const double* scales, int scaling, double* out) {
    try {
        data::LocalBlock block;
        block.row_range = {0, nx_i};
        block.values = to_matrix(q, n_vars * nx_i, nt);
        transform::TransformParams params;
        params.local_means.assign(means, means + n_vars * nx_i);
        if (scaling) params.scales.assign(scales, scales + n_vars);
        params.scaling_enabled = scaling != 0;
        from_matrix(postprocess::reconstruct_field(block, to_matrix(tr, nt, r), to_matrix(qtilde, nt_p, r), params),
                    out);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// rom_search::integrate (rom_search.cpp:60-85) with caller operators:
// a r x r, f r x s, c r, q0 r -> traj n_steps x r; returns finite in *finite.
int ref_integrate(const double* a, const double* f, const double* c, std::size_t r, const double* q0,
                  std::size_t n_steps, double* traj, int* finite) {
    try {
        opinf::ReducedOperators ops;
        ops.a = to_matrix(a, r, r);
        ops.f = to_matrix(f, r, opinf::quad_len(r));
        ops.c.assign(c, c + r);
        const rom_search::IntegrateResult res = rom_search::integrate(ops, std::vector<double>(q0, q0 + r), n_steps);
        from_matrix(res.trajectory, traj);
        *finite = res.finite ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// opinf::solve_opinf (opinf.cpp:69-92) for one pair on assemble_data(qhat):
// a r x r, f r x s, c r.
int ref_solve_opinf(const double* qhat, std::size_t r, std::size_t nt, double beta1, double beta2, double* a,
                    double* f, double* c) {
    try {
        const opinf::OpInfData data = opinf::assemble_data(to_matrix(qhat, r, nt));
        const auto gamma = opinf::build_regularizer(r, opinf::quad_len(r), {beta1, beta2});
        const opinf::ReducedOperators ops = opinf::solve_opinf(data, gamma);
        from_matrix(ops.a, a);
        from_matrix(ops.f, f);
        std::memcpy(c, ops.c.data(), r * sizeof(double));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// postprocess::reconstruct_probes (postprocess.cpp:36-61) on one rank's block
// (rows [begin, begin + nx_i) of every variable): owned probes' series into
// out (n_probes x nt_p, owned rows only) and owned[i].
int ref_reconstruct_probes(const double* q, std::size_t n_vars, std::size_t nx_i, std::size_t begin, std::size_t nt,
                           const double* tr, std::size_t r, const double* qtilde, std::size_t nt_p,
                           const double* means, const double* scales, int scaling, const std::size_t* var,
                           const std::size_t* index, std::size_t n_probes, double* out, int* owned) {
    try {
        data::LocalBlock block;
        block.row_range = {begin, begin + nx_i};
        block.values = to_matrix(q, n_vars * nx_i, nt);
        transform::TransformParams params;
        params.local_means.assign(means, means + n_vars * nx_i);
        if (scaling) params.scales.assign(scales, scales + n_vars);
        params.scaling_enabled = scaling != 0;
        postprocess::ProbeSet probes;
        for (std::size_t i = 0; i < n_probes; ++i) probes.push_back({var[i], index[i]});
        const auto series = postprocess::reconstruct_probes(block, to_matrix(tr, nt, r), to_matrix(qtilde, nt_p, r),
                                                            probes, params);
        for (std::size_t i = 0; i < n_probes; ++i) owned[i] = 0;
        for (const auto& sr : series) {
            for (std::size_t i = 0; i < n_probes; ++i) {
                if (probes[i] == sr.probe && !owned[i]) {
                    owned[i] = 1;
                    std::memcpy(out + i * nt_p, sr.values.data(), nt_p * sizeof(double));
                    break;
                }
            }
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"

#include "dopinf/pipeline.hpp"

extern "C" {

// pipeline::run (pipeline.cpp:400-414), Steps I–V from the SNP1 file `path`
// into out_dir: scaling on, r = fixed_rank (0: energy 0.9995), an n1 × n2
// (β1, β2) grid, max_growth, nt_p, the probes (var, index). stage_seconds
// receives rank 0's six stage times (load, transform, gram_reduce,
// eig_project, search, postprocess); result = {r, beta1, beta2, train_err}.
int ref_pipeline_run(const char* path, const char* out_dir, int workers, long fixed_rank, int scaling,
                     const double* b1, std::size_t n1, const double* b2, std::size_t n2, double max_growth,
                     std::size_t nt_p, const std::size_t* probe_var, const std::size_t* probe_index,
                     std::size_t n_probes, double* stage_seconds, double* result) {
    try {
        pipeline::PipelineConfig cfg;
        cfg.data_path = path;
        cfg.out_dir = out_dir;
        cfg.workers = workers;
        cfg.fixed_rank = fixed_rank;
        cfg.scaling = scaling != 0;
        cfg.b1.assign(b1, b1 + n1);
        cfg.b2.assign(b2, b2 + n2);
        cfg.max_growth = max_growth;
        cfg.nt_p = nt_p;
        for (std::size_t i = 0; i < n_probes; ++i) cfg.probes.push_back({probe_var[i], probe_index[i]});
        const pipeline::RunResult res = pipeline::run(cfg);
        for (std::size_t s = 0; s < pipeline::kStageCount; ++s) stage_seconds[s] = res.stage_seconds[s];
        result[0] = static_cast<double>(res.r);
        result[1] = res.pair_opt.beta1;
        result[2] = res.pair_opt.beta2;
        result[3] = res.train_err;
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

}  // extern "C"
