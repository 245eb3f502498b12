// dopinf_b200.hpp — header-only C++ host layer over the C ABI (dopinf_b200.h)
// with the reference's stage signatures, so the reference pipeline can call it
// in place of its own Steps II–III (paths relative to /root/reference/proj):
//
//   dopinf_b200::transform::center_in_place(block)              transform.hpp:27
//   dopinf_b200::transform::compute_global_scales(block, hdr, comm)  transform.hpp:32-34
//   dopinf_b200::transform::scale_in_place(block, scales)       transform.hpp:37
//   dopinf_b200::pod::local_gram(block)                          pod.hpp:28
//   dopinf_b200::pod::global_gram(local, comm)                   pod.hpp:31
//   dopinf_b200::pod::project(tr, d)                             pod.hpp:49
//   dopinf_b200::postprocess::basis_rows(block, tr, rows)        postprocess.hpp:25-26
//   dopinf_b200::postprocess::basis(block, tr)  (Φ_r of reconstruct_field, postprocess.cpp:66)
//   dopinf_b200::rom_search::grid_search<OutcomeT>(qhat, config, comm)      rom_search.hpp:87-91
//   dopinf_b200::postprocess::reconstruct_probes<SeriesT>(block, tr, qtilde, probes, params)  postprocess.hpp:37-40
//   dopinf_b200::postprocess::reconstruct_field(block, tr, qtilde, params)  postprocess.hpp:43-45
//   dopinf_b200::data::partition_rows(nx, p)                     data.hpp:47
//   dopinf_b200::data::read_header<HeaderT>(path)                data.hpp:52
//   dopinf_b200::data::read_block<LocalBlockT>(path, plan, rank, header)  data.hpp:54
//   dopinf_b200::data::read_block_device(path, plan, rank, header)  (the same rows, left on the device)
//
// The functions are templates over the caller's block / matrix / header types
// (duck-typed on the members the reference's data::LocalBlock, Matrix and
// SnapshotHeader have), so they accept the reference's own types without this
// header including them. Value semantics are kept: a transform mutates the
// caller's host block. Each rank thread binds its Context first
// (dopinf_b200::Bind), mirroring one Comm per rank under run_on_workers.
//
// Residency: each host-block function uploads (and, for the transforms,
// downloads) the block. Every stage also has an overload on DeviceBlock
// (data::to_device / data::read_block_device): the same chain written against
// a DeviceBlock keeps the block on the GPU from the first stage to the last —
//   auto dev = dopinf_b200::data::read_block_device(path, plan, rank, header);
//   params.local_means = dopinf_b200::transform::center_in_place(dev);
//   params.scales = dopinf_b200::transform::compute_global_scales(dev, header, comm);
//   dopinf_b200::transform::scale_in_place(dev, params.scales);
//   Matrix gram = dopinf_b200::pod::global_gram(dopinf_b200::pod::local_gram<Matrix>(dev), comm);
// include/dopinf_b200_pipeline.hpp chains them into pipeline::run_rank.
//
// Errors: with DOPINF_B200_REFERENCE_ERRORS defined (after including the
// reference's "dopinf/errors.hpp"), failures throw the reference classes
// (dopinf::InvalidArgumentError, PartitionError, CollectiveError,
// DegenerateVariableError, dopinf::Error); otherwise the same-named classes in
// namespace dopinf_b200.
#pragma once

#include <cstddef>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>
#if __cplusplus >= 202002L
#include <span>
#endif

#include "dopinf_b200.h"

namespace dopinf_b200 {

#if defined(DOPINF_B200_REFERENCE_ERRORS)
using Error = ::dopinf::Error;
using InvalidArgumentError = ::dopinf::InvalidArgumentError;
using PartitionError = ::dopinf::PartitionError;
using CollectiveError = ::dopinf::CollectiveError;
using DegenerateVariableError = ::dopinf::DegenerateVariableError;
using NotPsdError = ::dopinf::NotPsdError;
using RankDeficiencyError = ::dopinf::RankDeficiencyError;
using SolveError = ::dopinf::SolveError;
using DataFormatError = ::dopinf::DataFormatError;
using NoAdmissiblePairError = ::dopinf::NoAdmissiblePairError;
#else
struct Error : std::runtime_error {
    explicit Error(const std::string& m) : std::runtime_error(m) {}
};
struct InvalidArgumentError : Error {
    using Error::Error;
};
struct PartitionError : Error {
    using Error::Error;
};
struct CollectiveError : Error {
    using Error::Error;
};
struct DegenerateVariableError : Error {
    using Error::Error;
};
struct NotPsdError : Error {
    using Error::Error;
};
struct RankDeficiencyError : Error {
    using Error::Error;
};
struct SolveError : Error {
    using Error::Error;
};
struct DataFormatError : Error {
    using Error::Error;
};
struct NoAdmissiblePairError : Error {
    using Error::Error;
};
#endif

[[noreturn]] inline void raise(int status, const std::string& msg) {
    switch (status) {
        case DOPINF_B200_ERR_INVALID_ARGUMENT: throw InvalidArgumentError(msg);
        case DOPINF_B200_ERR_PARTITION: throw PartitionError(msg);
        case DOPINF_B200_ERR_COLLECTIVE: throw CollectiveError(msg);
        case DOPINF_B200_ERR_DEGENERATE_VARIABLE: throw DegenerateVariableError(msg);
        case DOPINF_B200_ERR_NOT_PSD: throw NotPsdError(msg);
        case DOPINF_B200_ERR_RANK_DEFICIENCY: throw RankDeficiencyError(msg);
        case DOPINF_B200_ERR_SOLVE: throw SolveError(msg);
        case DOPINF_B200_ERR_DATA_FORMAT: throw DataFormatError(msg);
        case DOPINF_B200_ERR_NO_ADMISSIBLE_PAIR: throw NoAdmissiblePairError(msg);
        default: throw Error(msg);
    }
}

// ---- per-rank context ---------------------------------------------------------
class Context {
public:
    Context(int device, int rank = 0, int size = 1, const unsigned char* nccl_id = nullptr) {
        const int rc = dopinf_b200_ctx_create(device, rank, size, nccl_id, &ctx_);
        if (rc != DOPINF_B200_OK) raise(rc, std::string("dopinf_b200_ctx_create: ") + dopinf_b200_status_string(rc));
    }
    ~Context() { dopinf_b200_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    static std::vector<unsigned char> unique_id() {
        std::vector<unsigned char> id(DOPINF_B200_UNIQUE_ID_BYTES);
        check(dopinf_b200_get_unique_id(id.data()), nullptr, "get_unique_id");
        return id;
    }

    int rank() const { return dopinf_b200_ctx_rank(ctx_); }
    int size() const { return dopinf_b200_ctx_size(ctx_); }
    dopinf_b200_ctx* handle() const { return ctx_; }

    // comm::Comm::allreduce (comm.hpp:20-28): 0 = Sum, 1 = Max, 2 = Min.
    void allreduce(double* data, std::size_t count, int op) {
        check(dopinf_b200_allreduce(ctx_, data, count, op), ctx_, "allreduce");
    }
    void barrier() { check(dopinf_b200_barrier(ctx_), ctx_, "barrier"); }
    // DOPINF_B200_GRAM_ORDER_TENSOR (default) or _REFERENCE (bit-identical D).
    void set_gram_order(int order) { check(dopinf_b200_set_gram_order(ctx_, order), ctx_, "set_gram_order"); }
    double stage_ms(dopinf_b200_stage s) const {
        double ms = 0.0;
        dopinf_b200_stage_ms(ctx_, s, &ms);
        return ms;
    }

    static void check(int rc, const dopinf_b200_ctx* c, const char* what) {
        if (rc != DOPINF_B200_OK) raise(rc, std::string(what) + ": " + dopinf_b200_last_error(c));
    }
    // The library's message unchanged (the reference's own text for data::).
    static void check_exact(int rc, const dopinf_b200_ctx* c) {
        if (rc != DOPINF_B200_OK) raise(rc, dopinf_b200_last_error(c));
    }

private:
    dopinf_b200_ctx* ctx_ = nullptr;
};

namespace detail {
inline Context*& bound() {
    thread_local Context* ctx = nullptr;
    return ctx;
}
inline Context& ctx() {
    if (!bound()) throw InvalidArgumentError("dopinf_b200: no Context bound on this thread (use dopinf_b200::Bind)");
    return *bound();
}
}  // namespace detail

// RAII binding of a rank's Context to the calling thread.
class Bind {
public:
    explicit Bind(Context& c) : prev_(detail::bound()) { detail::bound() = &c; }
    ~Bind() { detail::bound() = prev_; }

private:
    Context* prev_;
};

namespace detail {
#if __cplusplus >= 202002L
// comm::ReduceOp of the caller's Comm (comm.hpp:9: Sum, Max, Min), deduced from
// its allreduce(std::span<double>, ReduceOp) (comm.hpp:24).
template <class C, class Op>
Op reduce_op_of(void (C::*)(std::span<double>, Op));
template <class CommT>
using ReduceOpT = decltype(reduce_op_of(&CommT::allreduce));
constexpr int kSum = 0, kMax = 1;

// Which collectives a stage uses. The bound Context's own (NCCL) when it spans
// the caller's ranks; the caller's Comm when every rank binds a size-1
// Context — the reference's in-process ranks (comm_inprocess.cpp:159-178) or
// MPI ranks sharing fewer GPUs than ranks: each rank runs its local half on
// the device and the reduction is the reference's own.
template <class CommT>
bool host_collectives(CommT& comm, const char* what) {
    Context& c = ctx();
    if (comm.size() == c.size() && comm.rank() == c.rank()) return false;
    if (c.size() == 1) return true;
    throw CollectiveError(std::string(what) + ": comm does not match the bound device context");
}
#else
template <class CommT>
bool host_collectives(CommT& comm, const char* what) {
    if (comm.size() == ctx().size() && comm.rank() == ctx().rank()) return false;
    throw CollectiveError(std::string(what) + ": comm does not match the bound device context");
}
#endif
}  // namespace detail

// Device-resident LocalBlock (data.hpp:38-42): (n_vars·nx_i) × nt on the GPU.
// Every stage below has an overload on DeviceBlock, so the reference's stage
// chain (pipeline.cpp:270-298) written against a DeviceBlock runs with the
// block resident: one upload (data::to_device or data::read_block_device),
// then only means, scales and D cross PCIe.
class DeviceBlock {
public:
    DeviceBlock(Context& c, std::size_t n_vars, std::size_t nx_i, std::size_t row_begin, std::size_t nt)
        : ctx_(c) {
        Context::check(dopinf_b200_block_create(c.handle(), n_vars, nx_i, row_begin, nt, &b_), c.handle(),
                       "block_create");
    }
    ~DeviceBlock() { dopinf_b200_block_destroy(b_); }
    DeviceBlock(const DeviceBlock&) = delete;
    DeviceBlock& operator=(const DeviceBlock&) = delete;
    DeviceBlock(DeviceBlock&& o) noexcept : ctx_(o.ctx_), b_(o.b_) { o.b_ = nullptr; }
    // Take ownership of a block the library created (dopinf_b200_block_read).
    DeviceBlock(Context& c, dopinf_b200_block* owned) : ctx_(c), b_(owned) {}

    void upload(const double* host, std::size_t ld) {
        Context::check(dopinf_b200_block_upload(b_, host, ld), ctx_.handle(), "upload");
    }
    void download(double* host, std::size_t ld) const {
        Context::check(dopinf_b200_block_download(b_, host, ld), ctx_.handle(), "download");
    }
    dopinf_b200_block* handle() const { return b_; }
    Context& context() const { return ctx_; }
    std::size_t n_vars() const { return shape(0); }
    std::size_t nx_i() const { return shape(1); }
    std::size_t row_begin() const { return shape(2); }
    std::size_t nt() const { return shape(3); }
    std::size_t rows() const { return n_vars() * nx_i(); }

private:
    std::size_t shape(int k) const {
        std::size_t dims[4] = {};
        Context::check(dopinf_b200_block_shape(b_, dims), nullptr, "block_shape");
        return dims[k];
    }
    Context& ctx_;
    dopinf_b200_block* b_ = nullptr;
};

namespace detail {
// n_vars of a block: rows / nx_i (the reference derives it from the header).
template <class LocalBlockT>
std::size_t n_vars_of(const LocalBlockT& block) {
    const std::size_t nx_i = block.row_range.count();
    return nx_i == 0 ? 1 : block.values.rows() / nx_i;
}

template <class LocalBlockT>
DeviceBlock uploaded(const LocalBlockT& block, std::size_t n_vars) {
    DeviceBlock d(ctx(), n_vars, block.row_range.count(), block.row_range.begin, block.values.cols());
    d.upload(block.values.data(), block.values.cols());
    return d;
}
}  // namespace detail

namespace data {
// data.cpp:86-103. Returns a vector of (begin, end) as PlanT's element type.
template <class RowRangeT>
std::vector<RowRangeT> partition_rows(std::size_t nx, int p) {
    if (p < 1) throw PartitionError("partition_rows: rank count must be >= 1, got " + std::to_string(p));
    if (static_cast<std::size_t>(p) > nx) {
        throw PartitionError("partition_rows: rank count " + std::to_string(p) + " exceeds row count " +
                             std::to_string(nx));
    }
    std::vector<std::size_t> b(static_cast<std::size_t>(p)), e(static_cast<std::size_t>(p));
    Context::check(dopinf_b200_partition_rows(nx, p, b.data(), e.data()), nullptr, "partition_rows");
    std::vector<RowRangeT> plan(static_cast<std::size_t>(p));
    for (std::size_t r = 0; r < plan.size(); ++r) {
        plan[r].begin = b[r];
        plan[r].end = e[r];
    }
    return plan;
}

// data::read_header (data.cpp:133-162): same checks, same DataFormatError text.
template <class HeaderT>
HeaderT read_header(const std::string& path) {
    std::uint64_t dims[4] = {};
    std::size_t need = 0;
    Context::check_exact(dopinf_b200_snp1_header(path.c_str(), dims, nullptr, 0, &need), nullptr);
    std::vector<char> names(need + 1);
    Context::check_exact(dopinf_b200_snp1_header(path.c_str(), dims, names.data(), names.size(), nullptr), nullptr);
    HeaderT h;
    h.n_vars = dims[0];
    h.nx = dims[1];
    h.nt = dims[2];
    h.var_names.clear();
    for (std::size_t at = 0; at < need; at += h.var_names.back().size() + 1) h.var_names.emplace_back(&names[at]);
    return h;
}

namespace detail {
// data.cpp:166-177: the plan covers [0, nx) contiguously and rank lies in it.
template <class PlanT, class HeaderT>
void check_plan(const PlanT& plan, int rank, const HeaderT& header) {
    if (plan.empty() || plan.front().begin != 0 || plan.back().end != header.nx) {
        throw PartitionError("read_block: plan does not cover the file's rows");
    }
    for (std::size_t r = 1; r < plan.size(); ++r) {
        if (plan[r].begin != plan[r - 1].end) throw PartitionError("read_block: plan intervals are not contiguous");
    }
    if (rank < 0 || static_cast<std::size_t>(rank) >= plan.size()) {
        throw PartitionError("read_block: rank " + std::to_string(rank) + " outside plan of size " +
                             std::to_string(plan.size()));
    }
}
}  // namespace detail

// The rank's rows of every variable, read through the pinned ring straight
// into a device block (no host Matrix).
template <class PlanT, class HeaderT>
DeviceBlock read_block_device(const std::string& path, const PlanT& plan, int rank, const HeaderT& header) {
    detail::check_plan(plan, rank, header);
    Context& c = ::dopinf_b200::detail::ctx();
    dopinf_b200_block* b = nullptr;
    const auto& range = plan[static_cast<std::size_t>(rank)];
    Context::check_exact(dopinf_b200_block_read(c.handle(), path.c_str(), range.begin, range.end, &b), c.handle());
    return DeviceBlock(c, b);
}

// data::read_block (data.cpp:164-202) with the reference's return type.
template <class LocalBlockT, class PlanT, class HeaderT>
LocalBlockT read_block(const std::string& path, const PlanT& plan, int rank, const HeaderT& header) {
    DeviceBlock d = read_block_device(path, plan, rank, header);
    LocalBlockT block;
    block.rank = rank;
    block.row_range = plan[static_cast<std::size_t>(rank)];
    block.values = decltype(block.values)(header.n_vars * block.row_range.count(), header.nt);
    d.download(block.values.data(), header.nt);
    return block;
}

// A host LocalBlock's values on the device (one upload), for the resident
// overloads below; to_host copies them back into a host block.
template <class LocalBlockT>
DeviceBlock to_device(const LocalBlockT& block, std::size_t n_vars) {
    return ::dopinf_b200::detail::uploaded(block, n_vars);
}
template <class LocalBlockT>
void to_host(const DeviceBlock& d, LocalBlockT& block) {
    d.download(block.values.data(), block.values.cols());
}
}  // namespace data

namespace transform {
// transform.cpp:10-20 on the resident block: returns the per-row means; the
// subtraction is fused into the next pass over the block.
inline std::vector<double> center_in_place(DeviceBlock& d) {
    std::vector<double> means(d.rows());
    Context::check(dopinf_b200_center(d.handle(), means.data()), d.context().handle(), "center_in_place");
    return means;
}

// transform.cpp:22-41 (MAX over the bound Context's NCCL ranks, or over the
// caller's Comm when every rank binds a size-1 Context).
template <class HeaderT, class CommT>
std::vector<double> compute_global_scales(const DeviceBlock& d, const HeaderT& header, CommT& comm) {
    const bool host = ::dopinf_b200::detail::host_collectives(comm, "compute_global_scales");
    const std::size_t n_vars = static_cast<std::size_t>(header.n_vars);
    std::vector<double> scales(n_vars);
    std::size_t bad = 0;
    int rc = DOPINF_B200_OK;
    if (host) {
#if __cplusplus >= 202002L
        // transform.cpp:28-39: local max-abs, MAX over the caller's Comm, zero check
        Context::check(dopinf_b200_local_maxabs(d.handle(), scales.data()), d.context().handle(),
                       "compute_global_scales");
        comm.allreduce(std::span<double>(scales),
                       static_cast<::dopinf_b200::detail::ReduceOpT<CommT>>(::dopinf_b200::detail::kMax));
        for (std::size_t j = 0; j < n_vars && rc == DOPINF_B200_OK; ++j) {
            if (scales[j] == 0.0) {
                rc = DOPINF_B200_ERR_DEGENERATE_VARIABLE;
                bad = j;
            }
        }
#endif
    } else {
        rc = dopinf_b200_global_scales(d.handle(), scales.data(), &bad);
    }
    if (rc == DOPINF_B200_ERR_DEGENERATE_VARIABLE) {
        throw DegenerateVariableError("variable '" + header.var_names[bad] +
                                      "' is constant in time; max-abs scaling is undefined");
    }
    Context::check(rc, d.context().handle(), "compute_global_scales");
    return scales;
}

// transform.cpp:43-49
inline void scale_in_place(DeviceBlock& d, const std::vector<double>& scales) {
    Context::check(dopinf_b200_scale(d.handle(), scales.data()), d.context().handle(), "scale_in_place");
}

// Host-block versions: the reference's value semantics (the caller's host
// block is mutated), through one upload and one download each.
template <class LocalBlockT>
std::vector<double> center_in_place(LocalBlockT& block) {
    DeviceBlock d = ::dopinf_b200::detail::uploaded(block, ::dopinf_b200::detail::n_vars_of(block));
    std::vector<double> means = center_in_place(d);
    d.download(block.values.data(), block.values.cols());
    return means;
}

template <class LocalBlockT, class HeaderT, class CommT>
std::vector<double> compute_global_scales(const LocalBlockT& block, const HeaderT& header, CommT& comm) {
    const DeviceBlock d = ::dopinf_b200::detail::uploaded(block, static_cast<std::size_t>(header.n_vars));
    return compute_global_scales(d, header, comm);
}

template <class LocalBlockT>
void scale_in_place(LocalBlockT& block, const std::vector<double>& scales) {
    DeviceBlock d = ::dopinf_b200::detail::uploaded(block, scales.size());
    scale_in_place(d, scales);
    d.download(block.values.data(), block.values.cols());
}
}  // namespace transform

namespace pod {
// pod.cpp:11-13 on the resident block: nt x nt as MatrixT (e.g. dopinf::Matrix).
template <class MatrixT>
MatrixT local_gram(const DeviceBlock& d) {
    const std::size_t nt = d.nt();
    MatrixT out(nt, nt);
    Context::check(dopinf_b200_local_gram(d.handle(), out.data()), d.context().handle(), "local_gram");
    return out;
}

// pod.cpp:11-13: returns MatrixT (the block's values type) nt x nt.
template <class LocalBlockT>
auto local_gram(const LocalBlockT& block) -> std::decay_t<decltype(block.values)> {
    using MatrixT = std::decay_t<decltype(block.values)>;
    const DeviceBlock d = ::dopinf_b200::detail::uploaded(block, ::dopinf_b200::detail::n_vars_of(block));
    return local_gram<MatrixT>(d);
}

// pod.cpp:15-18: reduces the device copy of the last local Gram of this rank.
template <class MatrixT, class CommT>
MatrixT global_gram(MatrixT local, CommT& comm) {
    if (::dopinf_b200::detail::host_collectives(comm, "global_gram")) {
#if __cplusplus >= 202002L
        // pod.cpp:15-18 verbatim: the caller's Comm sums the local Grams
        comm.allreduce(std::span<double>(local.data(), local.rows() * local.cols()),
                       static_cast<::dopinf_b200::detail::ReduceOpT<CommT>>(::dopinf_b200::detail::kSum));
#endif
        return local;
    }
    if (local.rows() != local.cols()) throw InvalidArgumentError("global_gram: local Gram is not square");
    Context::check(dopinf_b200_global_gram(::dopinf_b200::detail::ctx().handle(), local.data(), local.rows()),
                   ::dopinf_b200::detail::ctx().handle(), "global_gram");
    return local;
}

// pod.cpp:20-65 on the device (cuSOLVER dsyevd + the reference's descending
// order, clamp and sign convention). SpectrumT is the caller's
// pod::EigenSpectrum-like type {std::vector<double> eigenvalues; MatrixT eigenvectors;}.
template <class SpectrumT, class MatrixT>
SpectrumT eig_sym_desc(const MatrixT& d) {
    if (d.rows() != d.cols()) throw InvalidArgumentError("symmetric_eig: matrix is not square");
    Context& c = ::dopinf_b200::detail::ctx();
    Context::check(dopinf_b200_set_gram(c.handle(), d.data(), d.rows()), c.handle(), "eig_sym_desc");
    SpectrumT out;
    out.eigenvalues.resize(d.rows());
    out.eigenvectors = MatrixT(d.rows(), d.cols());
    const int rc = dopinf_b200_eig_sym_desc(c.handle(), out.eigenvalues.data(), out.eigenvectors.data());
    if (rc == DOPINF_B200_ERR_NOT_PSD) throw NotPsdError(dopinf_b200_last_error(c.handle()));
    Context::check(rc, c.handle(), "eig_sym_desc");
    return out;
}

// pod.cpp:84-101 on the device from the last eig_sym_desc of this thread's context.
template <class MatrixT>
MatrixT reduced_map_device(std::size_t nt, std::size_t r) {
    Context& c = ::dopinf_b200::detail::ctx();
    MatrixT tr(nt, r);
    const int rc = dopinf_b200_reduced_map(c.handle(), r, tr.data());
    if (rc == DOPINF_B200_ERR_RANK_DEFICIENCY) throw RankDeficiencyError(dopinf_b200_last_error(c.handle()));
    Context::check(rc, c.handle(), "reduced_map");
    return tr;
}

// pod.cpp:103-105: Q̂ = T_rᵀ D, the reference's FMA order (bit-identical).
template <class MatrixT>
MatrixT project(const MatrixT& tr, const MatrixT& d) {
    if (tr.rows() != d.rows() || d.rows() != d.cols()) throw InvalidArgumentError("matmul_tn: row counts differ");
    MatrixT out(tr.cols(), d.cols());
    Context::check(dopinf_b200_project_host(::dopinf_b200::detail::ctx().handle(), tr.data(), d.data(), d.rows(),
                                            tr.cols(), out.data()),
                   ::dopinf_b200::detail::ctx().handle(), "project");
    return out;
}
}  // namespace pod

namespace rom_search {
// rom_search::grid_search (rom_search.cpp:185-262) on the device: the bound
// Context's ranks share the candidates as distribute_pairs does (the comm
// argument is the reference's and unused: the Context carries the ranks).
template <class OutcomeT, class MatrixT, class ConfigT, class CommT>
OutcomeT grid_search(const MatrixT& qhat, const ConfigT& config, CommT& comm) {
    // With size-1 Contexts under a wider Comm every rank evaluates all pairs
    // (same winner: the first minimum, as the reference's lowest-rank claim over
    // contiguous pair ranges) and reports the owner distribute_pairs gives it.
    const bool host = ::dopinf_b200::detail::host_collectives(comm, "grid_search");
    Context& c = ::dopinf_b200::detail::ctx();
    std::vector<double> traj(config.nt_p * qhat.rows());
    double pair[2] = {0.0, 0.0}, err = 0.0, secs = 0.0;
    int owner = -1;
    Context::check_exact(dopinf_b200_grid_search(c.handle(), qhat.data(), qhat.rows(), qhat.cols(), config.b1.data(),
                                                 config.b1.size(), config.b2.data(), config.b2.size(),
                                                 config.max_growth, config.nt_p, pair, &err, &owner, &secs,
                                                 traj.data()),
                         c.handle());
    if (host) {  // rom_search.cpp:207 / 236-240: the rank whose pair range holds the winner
        const std::size_t n2 = config.b2.size(), n_reg = config.b1.size() * n2;
        std::size_t idx = 0;
        while (idx < n_reg && !(config.b1[idx / n2] == pair[0] && config.b2[idx % n2] == pair[1])) ++idx;
        for (int r = 0; r < comm.size(); ++r) {
            std::size_t b = 0, e = 0;
            Context::check(dopinf_b200_distribute_pairs(n_reg, r, comm.size(), &b, &e), nullptr, "grid_search");
            if (idx >= b && idx < e) {
                owner = r;
                break;
            }
        }
    }
    OutcomeT out;
    out.pair_opt = {pair[0], pair[1]};
    out.owner_rank = owner;
    out.train_err = err;
    out.rom_seconds = secs;
    out.trajectory = MatrixT(config.nt_p, qhat.rows(), std::move(traj));
    return out;
}
}  // namespace rom_search

namespace postprocess {
// postprocess.cpp:12-34 on the resident block (bit-identical order).
template <class MatrixT>
MatrixT basis_rows(const DeviceBlock& d, const MatrixT& tr, const std::vector<std::size_t>& local_rows) {
    if (d.nt() != tr.rows()) throw InvalidArgumentError("basis_rows: block and map disagree on nt");
    MatrixT out(local_rows.size(), tr.cols());
    Context::check(dopinf_b200_basis_rows(d.handle(), tr.data(), tr.cols(), local_rows.data(), local_rows.size(),
                                          out.data()),
                   d.context().handle(), "basis_rows");
    return out;
}

template <class LocalBlockT, class MatrixT>
MatrixT basis_rows(const LocalBlockT& block, const MatrixT& tr, const std::vector<std::size_t>& local_rows) {
    if (block.values.cols() != tr.rows()) throw InvalidArgumentError("basis_rows: block and map disagree on nt");
    const DeviceBlock d = ::dopinf_b200::detail::uploaded(block, ::dopinf_b200::detail::n_vars_of(block));
    return basis_rows(d, tr, local_rows);
}

// Φ_r = Q · T_r (postprocess.cpp:66), DMMA tall GEMM.
template <class MatrixT>
MatrixT basis(const DeviceBlock& d, const MatrixT& tr) {
    if (d.nt() != tr.rows()) throw InvalidArgumentError("matmul: inner dimensions differ");
    MatrixT out(d.rows(), tr.cols());
    Context::check(dopinf_b200_basis(d.handle(), tr.data(), tr.cols(), out.data()), d.context().handle(), "basis");
    return out;
}

template <class LocalBlockT, class MatrixT>
MatrixT basis(const LocalBlockT& block, const MatrixT& tr) {
    if (block.values.cols() != tr.rows()) throw InvalidArgumentError("matmul: inner dimensions differ");
    const DeviceBlock d = ::dopinf_b200::detail::uploaded(block, ::dopinf_b200::detail::n_vars_of(block));
    return basis(d, tr);
}

// postprocess::reconstruct_probes (postprocess.cpp:36-61), bit-identical: one
// SeriesT {probe, values} per probe whose index lies in the block's row range.
template <class SeriesT, class MatrixT, class ProbeSetT, class ParamsT>
std::vector<SeriesT> reconstruct_probes(const DeviceBlock& d, const MatrixT& tr, const MatrixT& qtilde,
                                        const ProbeSetT& probes, const ParamsT& params) {
    std::vector<std::size_t> var, index;
    for (const auto& p : probes) {
        var.push_back(p.var);
        index.push_back(p.index);
    }
    std::vector<double> out(probes.size() * qtilde.rows());
    std::vector<int> owned(probes.size());
    Context::check_exact(dopinf_b200_reconstruct_probes(d.handle(), tr.data(), tr.cols(), qtilde.data(), qtilde.rows(),
                                                        var.data(), index.data(), probes.size(),
                                                        params.local_means.data(),
                                                        params.scaling_enabled ? params.scales.data() : nullptr,
                                                        params.scaling_enabled ? 1 : 0, out.data(), owned.data()),
                         d.context().handle());
    std::vector<SeriesT> series;
    for (std::size_t i = 0; i < probes.size(); ++i) {
        if (!owned[i]) continue;
        SeriesT s;
        s.probe = probes[i];
        s.values.assign(out.begin() + i * qtilde.rows(), out.begin() + (i + 1) * qtilde.rows());
        series.push_back(std::move(s));
    }
    return series;
}

template <class SeriesT, class LocalBlockT, class MatrixT, class ProbeSetT, class ParamsT>
std::vector<SeriesT> reconstruct_probes(const LocalBlockT& block, const MatrixT& tr, const MatrixT& qtilde,
                                        const ProbeSetT& probes, const ParamsT& params) {
    const DeviceBlock d = ::dopinf_b200::detail::uploaded(block, ::dopinf_b200::detail::n_vars_of(block));
    return reconstruct_probes<SeriesT>(d, tr, qtilde, probes, params);
}

// postprocess::reconstruct_field (postprocess.cpp:63-70): (Q·T_r)·Q̃ᵀ mapped back
// with the TransformParams, (n_vars·nx_i) × nt_p; DMMA with the inverse
// transform fused.
template <class MatrixT, class ParamsT>
MatrixT reconstruct_field(const DeviceBlock& d, const MatrixT& tr, const MatrixT& qtilde, const ParamsT& params) {
    if (d.nt() != tr.rows()) throw InvalidArgumentError("matmul: inner dimensions differ");
    if (qtilde.cols() != tr.cols()) throw InvalidArgumentError("matmul_nt: column counts differ");
    if (d.rows() != params.local_means.size()) {
        throw InvalidArgumentError("inverse_transform_block: row count does not match the transform");
    }
    if (params.scaling_enabled && params.scales.size() != d.n_vars()) {
        throw InvalidArgumentError("reconstruct_field: scales do not match the block's variables");
    }
    MatrixT out(d.rows(), qtilde.rows());
    Context::check(dopinf_b200_reconstruct_field(d.handle(), tr.data(), tr.cols(), qtilde.data(), qtilde.rows(),
                                                 params.local_means.data(),
                                                 params.scaling_enabled ? params.scales.data() : nullptr,
                                                 params.scaling_enabled ? 1 : 0, out.data()),
                   d.context().handle(), "reconstruct_field");
    return out;
}

template <class LocalBlockT, class MatrixT, class ParamsT>
MatrixT reconstruct_field(const LocalBlockT& block, const MatrixT& tr, const MatrixT& qtilde, const ParamsT& params) {
    if (block.values.cols() != tr.rows()) throw InvalidArgumentError("matmul: inner dimensions differ");
    const DeviceBlock d = ::dopinf_b200::detail::uploaded(block, ::dopinf_b200::detail::n_vars_of(block));
    return reconstruct_field(d, tr, qtilde, params);
}
}  // namespace postprocess

}  // namespace dopinf_b200
