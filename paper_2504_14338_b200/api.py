"""Python mirror of the reference's stage API, over the C ABI.

Same names, argument meaning and error behaviour as the reference functions
(paths relative to /root/reference/proj):

  data::partition_rows / read_header / read_block / write_snapshots
                                  data.hpp:47-55,      data.cpp:86-202
  transform::center_in_place      transform.hpp:27,    transform.cpp:10-20
  transform::compute_global_scales transform.hpp:32-34, transform.cpp:22-41
  transform::scale_in_place       transform.hpp:37,    transform.cpp:43-49
  pod::local_gram / global_gram   pod.hpp:28-31,       pod.cpp:11-18
  pod::eig_sym_desc / reduced_map pod.hpp:34-47,       pod.cpp:20-101 (device)
  pod::project                    pod.hpp:49,          pod.cpp:103-105
  rom_search::grid_search / integrate / distribute_pairs
                                  rom_search.hpp:45-91, rom_search.cpp:60-262
  postprocess::basis_rows         postprocess.hpp:25,  postprocess.cpp:12-34
  postprocess::reconstruct_probes / reconstruct_field
                                  postprocess.hpp:37-45, postprocess.cpp:36-70
  (fused) snapshot_pass / snapshot_pass_host / snapshot_pass_file / write_field

Blocks live on the GPU (`LocalBlock` is device resident; `.values` downloads).
The reference's comm::Comm argument is the per-rank `DeviceContext`, whose
collectives run over NCCL. Used by the tests and bench.py; the C++ mirror for
C++ callers is include/dopinf_b200.hpp.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _lib


# ---- exceptions (include/dopinf/errors.hpp:9-73) ----------------------------
class Error(RuntimeError):
    pass


class DataFormatError(Error):
    pass


class PartitionError(Error):
    pass


class CollectiveError(Error):
    pass


class DegenerateVariableError(Error):
    pass


class NotPsdError(Error):
    pass


class RankDeficiencyError(Error):
    pass


class SolveError(Error):
    pass


class NoAdmissiblePairError(Error):
    pass


class InvalidArgumentError(Error):
    pass


class DeviceError(Error):
    """CUDA / NCCL failure (no reference analogue)."""


_STATUS = {
    _lib.ERR_INVALID_ARGUMENT: InvalidArgumentError,
    _lib.ERR_PARTITION: PartitionError,
    _lib.ERR_COLLECTIVE: CollectiveError,
    _lib.ERR_DEGENERATE_VARIABLE: DegenerateVariableError,
    _lib.ERR_DEVICE: DeviceError,
    _lib.ERR_OUT_OF_MEMORY: DeviceError,
    _lib.ERR_NOT_PSD: NotPsdError,
    _lib.ERR_RANK_DEFICIENCY: RankDeficiencyError,
    _lib.ERR_SOLVE: SolveError,
    _lib.ERR_DATA_FORMAT: DataFormatError,
    _lib.ERR_NO_ADMISSIBLE_PAIR: NoAdmissiblePairError,
}


def _check(rc: int, ctx=None, what: str = ""):
    if rc == _lib.OK:
        return
    lib = _lib.load()
    # ctx None: context-free call, its message is thread-local in the library
    msg = lib.dopinf_b200_last_error(ctx._h if ctx is not None else None).decode()
    raise _STATUS.get(rc, Error)(f"{what}: {msg}" if what else msg)


def _out(a: np.ndarray, shape) -> np.ndarray:
    if a.dtype != np.float64 or not a.flags.c_contiguous or a.shape != tuple(shape):
        raise InvalidArgumentError(f"output buffer must be C-contiguous float64 of shape {tuple(shape)}")
    return a


def _f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and out.shape != shape:
        raise InvalidArgumentError(f"expected shape {shape}, got {out.shape}")
    return out


# ---- data.hpp -----------------------------------------------------------------
@dataclass(frozen=True)
class RowRange:
    begin: int = 0
    end: int = 0

    def count(self) -> int:
        return self.end - self.begin


@dataclass
class SnapshotHeader:
    n_vars: int
    nx: int
    nt: int
    var_names: list = field(default_factory=list)

    def __post_init__(self):
        if not self.var_names:
            self.var_names = [f"var{j}" for j in range(self.n_vars)]


def check_uniform(table, rank: int, what: str = "allreduce") -> None:
    """verify_uniform's rule (comm_inprocess.cpp:139-151) on an all-gathered
    table of (sequence, count, tag) rows, through the library: raises
    CollectiveError with the reference's message on a disagreement."""
    t = np.ascontiguousarray(table, dtype=np.int64)
    if t.ndim != 2 or t.shape[1] != 3:
        raise InvalidArgumentError("check_uniform: table must be p x 3")
    msg = C.create_string_buffer(512)
    rc = _lib.load().dopinf_b200_check_uniform(t.ctypes.data_as(C.POINTER(C.c_longlong)), t.shape[0], rank,
                                               what.encode(), msg, 512)
    if rc == _lib.ERR_COLLECTIVE:
        raise CollectiveError(msg.value.decode())
    _check(rc)


def partition_rows(nx: int, p: int) -> list:
    """data.cpp:86-103: floor(nx/p) rows per rank, remainder on the last rank."""
    lib = _lib.load()
    if p < 1:
        raise PartitionError(f"partition_rows: rank count must be >= 1, got {p}")
    if p > nx:
        raise PartitionError(f"partition_rows: rank count {p} exceeds row count {nx}")
    b = np.zeros(p, dtype=np.uintp)
    e = np.zeros(p, dtype=np.uintp)
    rc = lib.dopinf_b200_partition_rows(nx, p, _lib.sptr(b), _lib.sptr(e))
    if rc == _lib.ERR_PARTITION:
        raise PartitionError(f"partition_rows({nx}, {p})")
    _check(rc)
    return [RowRange(int(x), int(y)) for x, y in zip(b, e)]


# ---- per-rank context (comm::Comm) ----------------------------------------------
class DeviceContext:
    """One rank: a B200, its stream, and (size > 1) an NCCL communicator."""

    SUM, MAX, MIN = _lib.SUM, _lib.MAX, _lib.MIN

    def __init__(self, device: int = 0, rank: int = 0, size: int = 1, unique_id: bytes | None = None,
                 gram_reduce: str = "nccl", nccl: bool = False):
        """`nccl=True` gives a size-1 context an NCCL communicator too (its own
        unique id unless one is passed), so every collective code path runs on
        one GPU."""
        lib = _lib.load()
        h = C.c_void_p()
        uid = None
        if size > 1 or nccl:
            if unique_id is None and size == 1:
                unique_id = DeviceContext.unique_id()
            if unique_id is None or len(unique_id) != _lib.UNIQUE_ID_BYTES:
                raise InvalidArgumentError("size > 1 needs the rank-0 unique id bytes")
            uid = C.create_string_buffer(bytes(unique_id), _lib.UNIQUE_ID_BYTES)
        rc = lib.dopinf_b200_ctx_create_ex(device, rank, size, uid, _lib.CTX_NCCL if nccl else 0, C.byref(h))
        if rc != _lib.OK:
            raise _STATUS.get(rc, Error)(f"ctx_create(device={device}, rank={rank}, size={size}) failed: "
                                         f"{lib.dopinf_b200_status_string(rc).decode()}")
        self._h = h
        self._rank, self._size, self.device = rank, size, device
        self._blocks = weakref.WeakSet()  # destroyed before the context
        self.set_gram_reduce(gram_reduce)

    @classmethod
    def external(cls, device: int = 0, nccl_comm: int | None = None, stream: int | None = None,
                 gram_reduce: str = "nccl") -> "DeviceContext":
        """A context on the caller's NCCL communicator / CUDA stream (raw handle
        values; None: one rank / own stream). Rank and size come from the
        communicator; neither handle is destroyed with the context."""
        lib = _lib.load()
        h = C.c_void_p()
        rc = lib.dopinf_b200_ctx_create_external(device, nccl_comm, stream, C.byref(h))
        if rc != _lib.OK:
            raise _STATUS.get(rc, Error)(f"ctx_create_external(device={device}) failed: "
                                         f"{lib.dopinf_b200_status_string(rc).decode()}")
        self = cls.__new__(cls)
        self._h = h
        self._rank, self._size = lib.dopinf_b200_ctx_rank(h), lib.dopinf_b200_ctx_size(h)
        self.device = device
        self._blocks = weakref.WeakSet()
        self.set_gram_reduce(gram_reduce)
        return self

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(_lib.UNIQUE_ID_BYTES)
        _check(_lib.load().dopinf_b200_get_unique_id(buf))
        return buf.raw

    def rank(self) -> int:
        return self._rank

    def size(self) -> int:
        return self._size

    def set_gram_reduce(self, mode: str):
        m = {"ordered": _lib.GRAM_REDUCE_ORDERED, "nccl": _lib.GRAM_REDUCE_NCCL}[mode]
        _check(_lib.load().dopinf_b200_set_gram_reduce(self._h, m), self)

    def set_gram_order(self, order: str):
        """"tensor" (DMMA, default) or "reference": linalg::gram's own FMA order,
        bit-identical D (and the ORDERED cross-rank sum)."""
        m = {"tensor": _lib.GRAM_ORDER_TENSOR, "reference": _lib.GRAM_ORDER_REFERENCE}[order]
        _check(_lib.load().dopinf_b200_set_gram_order(self._h, m), self)

    def allreduce(self, data: np.ndarray, op: int) -> None:
        """Comm::allreduce (comm.hpp:20-28) on a host float64 array, in place."""
        if data.dtype != np.float64 or not data.flags.c_contiguous:
            raise InvalidArgumentError("allreduce: needs a C-contiguous float64 array")
        _check(_lib.load().dopinf_b200_allreduce(self._h, _lib.dptr(data), data.size, op), self, "allreduce")

    def barrier(self) -> None:
        _check(_lib.load().dopinf_b200_barrier(self._h), self, "barrier")

    def set_collective_timeout(self, seconds: float) -> None:
        """Deadline for a queued collective (comm_inprocess.cpp kTimeout = 60 s)."""
        _check(_lib.load().dopinf_b200_set_collective_timeout(self._h, float(seconds)), self)

    def set_collective_checks(self, enabled: bool) -> None:
        """verify_uniform (comm_inprocess.cpp:139-151) before every collective."""
        _check(_lib.load().dopinf_b200_set_collective_checks(self._h, 1 if enabled else 0), self)

    def poisoned(self) -> bool:
        return bool(_lib.load().dopinf_b200_ctx_poisoned(self._h))

    def debug_inject(self, fault: int) -> None:
        _check(_lib.load().dopinf_b200_debug_inject(self._h, fault), self)

    def ordered_sum(self, parts) -> np.ndarray:
        """Device ascending-rank sum of p partials (the ORDERED combine step)."""
        parts = _f64(parts)
        p, count = parts.shape
        out = np.empty(count, dtype=np.float64)
        _check(_lib.load().dopinf_b200_ordered_sum(self._h, _lib.dptr(parts), p, count, _lib.dptr(out)), self,
               "ordered_sum")
        return out

    def stage_ms(self, stage: str) -> float:
        v = C.c_double()
        _check(_lib.load().dopinf_b200_stage_ms(self._h, _lib.STAGES.index(stage), C.byref(v)), self)
        return v.value

    def stream(self) -> int:
        return _lib.load().dopinf_b200_ctx_stream(self._h) or 0

    def close(self):
        if getattr(self, "_h", None):
            for b in list(getattr(self, "_blocks", ())):
                b.close()
            _lib.load().dopinf_b200_ctx_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


# ---- SNP1 snapshot files (data.hpp:11-15) -------------------------------------------
_MAGIC = b"SNP1"


def write_snapshots(path: str, header: SnapshotHeader, variables) -> None:
    """data::write_snapshots (data.cpp:105-131): host-side writer of the SNP1
    container (magic, u64 n_vars/nx/nt, u32-length names, per-variable row-major
    nx × nt float64). Same checks and messages as the reference."""
    _validate_header(header)
    if len(variables) != header.n_vars:
        raise InvalidArgumentError("write_snapshots: variable count mismatch")
    arrs = [np.ascontiguousarray(v, dtype=np.float64) for v in variables]
    if any(a.shape != (header.nx, header.nt) for a in arrs):
        raise InvalidArgumentError("write_snapshots: variable shape mismatch")
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC)
            f.write(np.array([header.n_vars, header.nx, header.nt], dtype="<u8").tobytes())
            for name in header.var_names:
                b = name.encode()
                f.write(np.array([len(b)], dtype="<u4").tobytes())
                f.write(b)
            for a in arrs:
                a.tofile(f)
    except OSError as e:
        raise DataFormatError(f"cannot create snapshot file: {path}") from e


def _validate_header(h: SnapshotHeader) -> None:
    """data.cpp:35-48."""
    if h.n_vars < 1:
        raise DataFormatError("snapshot header: n_vars must be >= 1")
    if h.nx < 1:
        raise DataFormatError("snapshot header: nx must be >= 1")
    if h.nt < 2:
        raise DataFormatError("snapshot header: nt must be >= 2")
    if len(h.var_names) != h.n_vars:
        raise DataFormatError("snapshot header: name count does not match n_vars")
    seen = set()
    for name in h.var_names:
        if not name:
            raise DataFormatError("snapshot header: empty variable name")
        if name in seen:
            raise DataFormatError(f"snapshot header: duplicate variable name '{name}'")
        seen.add(name)


def read_header(path: str) -> SnapshotHeader:
    """data::read_header (data.cpp:133-162) through dopinf_b200_snp1_header."""
    lib = _lib.load()
    dims = (C.c_uint64 * 4)()
    need = C.c_size_t()
    bpath = os.fsencode(path)
    _check(lib.dopinf_b200_snp1_header(bpath, dims, None, 0, C.byref(need)))
    buf = C.create_string_buffer(max(need.value, 1))
    _check(lib.dopinf_b200_snp1_header(bpath, dims, buf, need.value, None))
    names = [n.decode() for n in buf.raw[: need.value].split(b"\0")[:-1]]
    return SnapshotHeader(int(dims[0]), int(dims[1]), int(dims[2]), names)


def _check_plan(plan, rank: int, header: SnapshotHeader) -> RowRange:
    """data.cpp:166-177: the plan covers [0, nx) contiguously and rank is in it."""
    if not plan or plan[0].begin != 0 or plan[-1].end != header.nx:
        raise PartitionError("read_block: plan does not cover the file's rows")
    for a, b in zip(plan, plan[1:]):
        if b.begin != a.end:
            raise PartitionError("read_block: plan intervals are not contiguous")
    if rank < 0 or rank >= len(plan):
        raise PartitionError(f"read_block: rank {rank} outside plan of size {len(plan)}")
    return plan[rank]


def read_block(path: str, plan, rank: int, header: SnapshotHeader, ctx: DeviceContext) -> "LocalBlock":
    """data::read_block (data.cpp:164-202) into a device-resident LocalBlock:
    each variable's slice is one contiguous byte range of the file, read into a
    pinned two-slot ring with the H2D of one chunk overlapping the next read."""
    rr = _check_plan(plan, rank, header)
    h = C.c_void_p()
    _check(_lib.load().dopinf_b200_block_read(ctx._h, os.fsencode(path), rr.begin, rr.end, C.byref(h)), ctx,
           "read_block")
    return LocalBlock._adopt(ctx, h, header.n_vars, rr, header.nt, rank)


def snapshot_pass_file(path: str, plan, rank: int, header: SnapshotHeader, ctx: DeviceContext, scaling: bool,
                       out: dict | None = None):
    """read_block + Steps II-III (pipeline.cpp:254-280) streamed: chunk c+1 is
    read and copied while chunk c is centered and its Gram accumulated.
    Returns (LocalBlock resident and transformed, TransformParams, D)."""
    rr = _check_plan(plan, rank, header)
    rows, nt = header.n_vars * rr.count(), header.nt
    out = out or {}
    means = _out(out["means"], (rows,)) if "means" in out else np.empty(max(rows, 1), dtype=np.float64)
    scales = _out(out["scales"], (header.n_vars,)) if "scales" in out else np.empty(header.n_vars, dtype=np.float64)
    d = _out(out["d"], (nt, nt)) if "d" in out else np.empty((nt, nt), dtype=np.float64)
    h = C.c_void_p()
    rc = _lib.load().dopinf_b200_snapshot_pass_file(ctx._h, os.fsencode(path), rr.begin, rr.end,
                                                    1 if scaling else 0, C.byref(h), _lib.dptr(means),
                                                    _lib.dptr(scales), _lib.dptr(d))
    _check(rc, ctx, "snapshot_pass_file")
    ctx._gram_nt = nt
    block = LocalBlock._adopt(ctx, h, header.n_vars, rr, nt, rank)
    return block, TransformParams(means[:rows], scales if scaling else np.zeros(0), scaling), d


# ---- device-resident data::LocalBlock ----------------------------------------------
class LocalBlock:
    """data::LocalBlock (data.hpp:38-42) held on the device: (n_vars·nx_i) × nt fp64,
    block row j*nx_i + k = variable j at global spatial index row_range.begin + k."""

    def __init__(self, ctx: DeviceContext, n_vars: int, row_range: RowRange, nt: int, values=None,
                 rank: int | None = None):
        lib = _lib.load()
        self.ctx = ctx
        self.rank = ctx.rank() if rank is None else rank
        self.row_range = row_range
        self.n_vars, self.nt = n_vars, nt
        self.nx_i = row_range.count()
        self.rows = n_vars * self.nx_i
        h = C.c_void_p()
        _check(lib.dopinf_b200_block_create(ctx._h, n_vars, self.nx_i, row_range.begin, nt, C.byref(h)), ctx,
               "block_create")
        self._h = h
        ctx._blocks.add(self)
        if values is not None:
            self.upload(values)

    @classmethod
    def _adopt(cls, ctx: DeviceContext, handle: C.c_void_p, n_vars: int, row_range: RowRange, nt: int,
               rank: int | None = None) -> "LocalBlock":
        """Wrap a block the library created (block_read / snapshot_pass_file)."""
        self = cls.__new__(cls)
        self.ctx = ctx
        self.rank = ctx.rank() if rank is None else rank
        self.row_range = row_range
        self.n_vars, self.nt = n_vars, nt
        self.nx_i = row_range.count()
        self.rows = n_vars * self.nx_i
        self._h = handle
        ctx._blocks.add(self)
        return self

    def upload(self, values) -> None:
        v = _f64(values, (self.rows, self.nt))
        _check(_lib.load().dopinf_b200_block_upload(self._h, _lib.dptr(v), self.nt), self.ctx, "upload")

    def upload_ptr(self, host_ptr: int, host_ld: int) -> None:
        """Upload from a raw host pointer (e.g. pinned torch memory)."""
        _check(_lib.load().dopinf_b200_block_upload(self._h, C.cast(host_ptr, _lib._dp), host_ld), self.ctx,
               "upload")

    @property
    def values(self) -> np.ndarray:
        out = np.empty((self.rows, self.nt), dtype=np.float64)
        _check(_lib.load().dopinf_b200_block_download(self._h, _lib.dptr(out), self.nt), self.ctx, "download")
        return out

    def rows_to(self, row0: int, out: np.ndarray) -> np.ndarray:
        """Rows [row0, row0 + len(out)) into `out` ((n, nt) float64, e.g. pinned)."""
        out = _out(out, (out.shape[0], self.nt))
        _check(_lib.load().dopinf_b200_block_download_rows(self._h, row0, out.shape[0], _lib.dptr(out), self.nt),
               self.ctx, "download_rows")
        return out

    def device_ptr(self):
        p = _lib._dp()
        ld = C.c_size_t()
        _check(_lib.load().dopinf_b200_block_device(self._h, C.byref(p), C.byref(ld)), self.ctx)
        return C.cast(p, C.c_void_p).value, ld.value

    def synth_oscillator(self, seed: int, n_modes: int, dt: float = 1e-3, noise: float = 1e-3, amps=None,
                         var0: int = 0):
        """Seeded generator (BASELINE configs 1, 2, 4); var0 > 0 makes the rows of
        variables var0.. of a larger dataset (amps: one entry per block variable)."""
        a = None if amps is None else _f64(amps, (self.n_vars,))
        _check(_lib.load().dopinf_b200_block_synth_oscillator_vars(self._h, var0, seed, n_modes, dt, noise,
                                                                   _lib.dptr(a)), self.ctx, "synth")

    def synth_lowrank(self, seed: int, rank: int = 50, amplitude: float = 10.0):
        _check(_lib.load().dopinf_b200_block_synth_lowrank(self._h, seed, rank, amplitude), self.ctx, "synth")

    def close(self):
        if getattr(self, "_h", None):
            _lib.load().dopinf_b200_block_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


# ---- transform.hpp -------------------------------------------------------------------
@dataclass
class TransformParams:
    local_means: np.ndarray = field(default_factory=lambda: np.zeros(0))
    scales: np.ndarray = field(default_factory=lambda: np.zeros(0))
    scaling_enabled: bool = False

    def row_scale(self, row: int, nx_i: int) -> float:
        return float(self.scales[row // nx_i]) if self.scaling_enabled else 1.0


def center_in_place(block: LocalBlock) -> np.ndarray:
    """transform.cpp:10-20: subtract each row's temporal mean; return the means."""
    means = np.empty(block.rows, dtype=np.float64)
    _check(_lib.load().dopinf_b200_center(block._h, _lib.dptr(means)), block.ctx, "center_in_place")
    return means


def compute_global_scales(block: LocalBlock, header: SnapshotHeader, comm: DeviceContext | None = None):
    """transform.cpp:22-41: per-variable global max-abs (MAX all-reduce over the ranks)."""
    if comm is not None and comm is not block.ctx:
        raise CollectiveError("compute_global_scales: comm must be the block's DeviceContext")
    scales = np.empty(block.n_vars, dtype=np.float64)
    bad = C.c_size_t(0)
    rc = _lib.load().dopinf_b200_global_scales(block._h, _lib.dptr(scales), C.byref(bad))
    if rc == _lib.ERR_DEGENERATE_VARIABLE:
        name = header.var_names[bad.value]
        raise DegenerateVariableError(
            f"variable '{name}' is constant in time; max-abs scaling is undefined")
    _check(rc, block.ctx, "compute_global_scales")
    return scales


def local_maxabs(block: LocalBlock) -> np.ndarray:
    """transform.cpp:28-31: this block's per-variable max |centered q|, no
    collective and no zero check (the caller reduces over its own comm)."""
    out = np.empty(block.n_vars, dtype=np.float64)
    _check(_lib.load().dopinf_b200_local_maxabs(block._h, _lib.dptr(out)), block.ctx, "local_maxabs")
    return out


def scale_in_place(block: LocalBlock, scales) -> None:
    """transform.cpp:43-49: divide each variable's rows by its scale."""
    s = _f64(scales, (block.n_vars,))
    _check(_lib.load().dopinf_b200_scale(block._h, _lib.dptr(s)), block.ctx, "scale_in_place")


# ---- pod.hpp ------------------------------------------------------------------------------
def local_gram(block: LocalBlock) -> np.ndarray:
    """pod.cpp:11-13: D_i = Q_iᵀ Q_i (full symmetric nt × nt)."""
    d = np.empty((block.nt, block.nt), dtype=np.float64)
    _check(_lib.load().dopinf_b200_local_gram(block._h, _lib.dptr(d)), block.ctx, "local_gram")
    block.ctx._gram_nt = block.nt
    return d


def global_gram(local: np.ndarray | None, comm: DeviceContext) -> np.ndarray:
    """pod.cpp:15-18: SUM all-reduce of the local Gram (identical on all ranks).
    The device copy of `local` (from local_gram on this context) is reduced."""
    nt = local.shape[0] if local is not None else None
    d = np.empty((nt, nt), dtype=np.float64) if nt is not None else None
    if d is None:
        raise InvalidArgumentError("global_gram: pass the local Gram returned by local_gram")
    _check(_lib.load().dopinf_b200_global_gram(comm._h, _lib.dptr(d), nt), comm, "global_gram")
    return d


def project(tr, d, ctx: DeviceContext) -> np.ndarray:
    """pod.cpp:103-105: Q̂ = T_rᵀ D (r × nt), reference FMA order on the device."""
    tr = _f64(tr)
    nt, r = tr.shape
    d = _f64(d, (nt, nt))
    out = np.empty((r, nt), dtype=np.float64)
    _check(_lib.load().dopinf_b200_project_host(ctx._h, _lib.dptr(tr), _lib.dptr(d), nt, r, _lib.dptr(out)),
           ctx, "project")
    return out


@dataclass
class EigenSpectrum:
    """pod::EigenSpectrum (pod.hpp:18-21)."""
    eigenvalues: np.ndarray
    eigenvectors: np.ndarray


def eig_sym_desc(ctx: DeviceContext, vectors: bool = True) -> EigenSpectrum:
    """pod::eig_sym_desc (pod.cpp:20-65) of the context's device Gram, on the
    device (cuSOLVER): descending, clamped, sign-normalised."""
    n = _device_gram_size(ctx)
    lam = np.empty(n, dtype=np.float64)
    vec = np.empty((n, n), dtype=np.float64) if vectors else None
    _check(_lib.load().dopinf_b200_eig_sym_desc(ctx._h, _lib.dptr(lam), _lib.dptr(vec)), ctx, "eig_sym_desc")
    return EigenSpectrum(lam, vec)


def set_gram(ctx: DeviceContext, d) -> None:
    """Make a host D (nt × nt, symmetric) the context's device Gram."""
    d = _f64(d)
    if d.ndim != 2 or d.shape[0] != d.shape[1]:
        raise InvalidArgumentError("set_gram: D must be square")
    _check(_lib.load().dopinf_b200_set_gram(ctx._h, _lib.dptr(d), d.shape[0]), ctx, "set_gram")
    ctx._gram_nt = d.shape[0]


def reduced_map(ctx: DeviceContext, r: int, download: bool = True):
    """pod::reduced_map (pod.cpp:84-101) on the device; the T_r stays on the
    context for project_resident(ctx, None) and basis(block, None, r)."""
    n = _device_gram_size(ctx)
    tr = np.empty((n, r), dtype=np.float64) if download else None
    _check(_lib.load().dopinf_b200_reduced_map(ctx._h, r, _lib.dptr(tr)), ctx, "reduced_map")
    return tr


def _device_gram_size(ctx: DeviceContext) -> int:
    n = getattr(ctx, "_gram_nt", None)
    if n is None:
        raise InvalidArgumentError("no Gram on this context")
    return n


def project_resident(ctx: DeviceContext, tr, out: np.ndarray | None = None, r: int | None = None) -> np.ndarray:
    """Q̂ = T_rᵀ D with the context's device-resident (global) Gram. `tr` may be
    None to use the device T_r of reduced_map (then pass r). `out` (r × nt
    float64, e.g. pinned) is filled when given."""
    if tr is None:
        nt = _device_gram_size(ctx)
        out = np.empty((r, nt), dtype=np.float64) if out is None else _out(out, (r, nt))
        _check(_lib.load().dopinf_b200_project(ctx._h, None, nt, r, _lib.dptr(out)), ctx, "project")
        return out
    tr = _f64(tr)
    nt, r = tr.shape
    out = np.empty((r, nt), dtype=np.float64) if out is None else _out(out, (r, nt))
    _check(_lib.load().dopinf_b200_project(ctx._h, _lib.dptr(tr), nt, r, _lib.dptr(out)), ctx, "project")
    return out


# ---- postprocess.hpp -------------------------------------------------------------------------
def basis_rows(block: LocalBlock, tr, local_rows) -> np.ndarray:
    """postprocess.cpp:12-34: rows of Φ_r = Q·T_r for the selected local rows."""
    tr = _f64(tr)
    if tr.shape[0] != block.nt:
        raise InvalidArgumentError("basis_rows: block and map disagree on nt")
    rows = np.ascontiguousarray(local_rows, dtype=np.uintp)
    r = tr.shape[1]
    out = np.empty((rows.size, r), dtype=np.float64)
    _check(_lib.load().dopinf_b200_basis_rows(block._h, _lib.dptr(tr), r, _lib.sptr(rows), rows.size,
                                              _lib.dptr(out)), block.ctx, "basis_rows")
    return out


def basis(block: LocalBlock, tr, download: bool = True, r: int | None = None):
    """Φ_r = Q·T_r over the whole block (postprocess.cpp:66), rows × r. `tr`
    None uses the context's device T_r from reduced_map (pass r)."""
    if tr is not None:
        tr = _f64(tr)
        if tr.shape[0] != block.nt:
            raise InvalidArgumentError("basis: block and map disagree on nt")
        r = tr.shape[1]
    out = np.empty((block.rows, r), dtype=np.float64) if download else None
    _check(_lib.load().dopinf_b200_basis(block._h, _lib.dptr(tr), r, _lib.dptr(out)), block.ctx, "basis")
    return out


# ---- rom_search.hpp (Step IV) ------------------------------------------------------
def logspace(lo: float, hi: float, n: int) -> list:
    """rom_search::logspace (rom_search.cpp:13-29)."""
    import math

    if n < 1:
        raise InvalidArgumentError("logspace: need at least one value")
    if not (lo > 0.0) or not (hi > 0.0):
        raise InvalidArgumentError("logspace: bounds must be positive")
    if n == 1:
        return [lo]
    a, b = math.log10(lo), math.log10(hi)
    return [10.0 ** (a + k * (b - a) / (n - 1)) for k in range(n)]


def default_b1() -> list:
    return logspace(1e-10, 1e0, 8)


def default_b2() -> list:
    return logspace(1e-4, 1e4, 8)


def distribute_pairs(n_reg: int, rank: int, size: int) -> RowRange:
    """rom_search::distribute_pairs (rom_search.cpp:136-149) through the ABI."""
    b, e = C.c_size_t(), C.c_size_t()
    _check(_lib.load().dopinf_b200_distribute_pairs(n_reg, rank, size, C.byref(b), C.byref(e)))
    return RowRange(b.value, e.value)


@dataclass
class SearchConfig:
    """rom_search::SearchConfig (rom_search.hpp:19-24)."""
    b1: list
    b2: list
    max_growth: float = 1.2
    nt_p: int = 0


@dataclass
class SearchOutcome:
    """rom_search::SearchOutcome (rom_search.hpp:35-41)."""
    pair_opt: tuple
    owner_rank: int
    train_err: float
    trajectory: np.ndarray
    rom_seconds: float


def grid_search(qhat, config: SearchConfig, comm: DeviceContext, r: int | None = None,
                nt: int | None = None) -> SearchOutcome:
    """rom_search::grid_search (rom_search.cpp:185-262) on the device. `qhat` is
    the r × nt reduced trajectory (host), or None for the context's device Q̂ of
    the last projection (pass r and nt)."""
    if qhat is not None:
        q = _f64(qhat)
        r, nt = q.shape
    else:
        q = None
    b1, b2 = _f64(list(config.b1)), _f64(list(config.b2))
    nt_p = int(config.nt_p)
    traj = np.empty((max(nt_p, 0), r), dtype=np.float64)
    pair = np.empty(2, dtype=np.float64)
    err = C.c_double()
    owner = C.c_int()
    secs = C.c_double()
    rc = _lib.load().dopinf_b200_grid_search(comm._h, _lib.dptr(q), r, nt, _lib.dptr(b1), b1.size, _lib.dptr(b2),
                                             b2.size, float(config.max_growth), nt_p, _lib.dptr(pair),
                                             C.byref(err), C.byref(owner), C.byref(secs), _lib.dptr(traj))
    _check(rc, comm)
    return SearchOutcome((float(pair[0]), float(pair[1])), int(owner.value), float(err.value), traj,
                         float(secs.value))


def rom_integrate(ctx: DeviceContext, a, f, c, q0, n_steps: int):
    """rom_search::integrate (rom_search.cpp:62-87) on the device -> (trajectory, finite)."""
    a, f, c, q0 = _f64(a), _f64(f), _f64(c), _f64(q0)
    r = a.shape[0]
    traj = np.empty((max(n_steps, 0), r), dtype=np.float64)
    fin = C.c_int()
    rc = _lib.load().dopinf_b200_rom_integrate(ctx._h, _lib.dptr(a), _lib.dptr(f), _lib.dptr(c), r, _lib.dptr(q0),
                                               n_steps, _lib.dptr(traj), C.byref(fin))
    _check(rc, ctx)
    return traj, bool(fin.value)


def _field_args(block: LocalBlock, tr, qtilde, params: TransformParams, r: int | None, what: str):
    if tr is not None:
        tr = _f64(tr)
        if tr.shape[0] != block.nt:
            raise InvalidArgumentError(f"{what}: block and map disagree on nt")
        r = tr.shape[1]
    qt = _f64(qtilde)
    if qt.ndim != 2 or qt.shape[1] != r:
        raise InvalidArgumentError(f"{what}: trajectory must be nt_p x r")
    means = _f64(params.local_means, (block.rows,))
    scales = _f64(params.scales, (block.n_vars,)) if params.scaling_enabled else None
    return tr, r, qt, means, scales


def reconstruct_field(block: LocalBlock, tr, qtilde, params: TransformParams, download: bool = True,
                      r: int | None = None, out: np.ndarray | None = None):
    """postprocess::reconstruct_field (postprocess.cpp:63-70): this rank's field
    (n_vars·nx_i) × nt_p in original coordinates, X = s·(Q·T_r)·Q̃ᵀ + mean, on
    the device (DMMA, inverse transform fused). `tr` None uses the context's
    device T_r (pass r). download=False keeps the field on the device
    (`field_device`)."""
    tr, r, qt, means, scales = _field_args(block, tr, qtilde, params, r, "reconstruct_field")
    nt_p = qt.shape[0]
    if download:
        out = _out(out, (block.rows, nt_p)) if out is not None else np.empty((block.rows, nt_p), dtype=np.float64)
    else:
        out = None
    rc = _lib.load().dopinf_b200_reconstruct_field(block._h, _lib.dptr(tr), r, _lib.dptr(qt), nt_p,
                                                   _lib.dptr(means), _lib.dptr(scales),
                                                   1 if params.scaling_enabled else 0, _lib.dptr(out))
    _check(rc, block.ctx, "reconstruct_field")
    return out


@dataclass
class Probe:
    """postprocess::Probe (postprocess.hpp:13-18): variable and global spatial index."""
    var: int = 0
    index: int = 0


@dataclass
class ProbeSeries:
    probe: Probe
    values: np.ndarray  # nt_p entries, original coordinates


def reconstruct_probes(block: LocalBlock, tr, qtilde, probes, params: TransformParams,
                       r: int | None = None) -> list:
    """postprocess::reconstruct_probes (postprocess.cpp:36-61) on the device,
    bit-identical to the reference: one ProbeSeries per probe this rank owns."""
    tr, r, qt, means, scales = _field_args(block, tr, qtilde, params, r, "reconstruct_probes")
    nt_p = qt.shape[0]
    var = np.ascontiguousarray([p.var for p in probes], dtype=np.uintp)
    index = np.ascontiguousarray([p.index for p in probes], dtype=np.uintp)
    out = np.empty((len(probes), nt_p), dtype=np.float64)
    owned = (C.c_int * max(len(probes), 1))()
    rc = _lib.load().dopinf_b200_reconstruct_probes(block._h, _lib.dptr(tr), r, _lib.dptr(qt), nt_p, _lib.sptr(var),
                                                    _lib.sptr(index), len(probes), _lib.dptr(means),
                                                    _lib.dptr(scales), 1 if params.scaling_enabled else 0,
                                                    _lib.dptr(out), owned)
    _check(rc, block.ctx)
    return [ProbeSeries(p, out[i].copy()) for i, p in enumerate(probes) if owned[i]]


def field_device(block: LocalBlock):
    """(device pointer, pitch in elements) of the last reconstructed field."""
    p = _lib._dp()
    ld = C.c_size_t()
    _check(_lib.load().dopinf_b200_field_device(block._h, C.byref(p), C.byref(ld)), block.ctx, "field_device")
    return C.cast(p, C.c_void_p).value, ld.value


def write_field(block: LocalBlock, tr, qtilde, params: TransformParams, var_names, path: str,
                r: int | None = None) -> None:
    """Step V field output (pipeline.cpp:330-350): reconstruct_field streamed
    straight into the SNP1 file `path` (n_vars, nx = nx_i, nt = nt_p)."""
    tr, r, qt, means, scales = _field_args(block, tr, qtilde, params, r, "write_field")
    if len(var_names) != block.n_vars:
        raise DataFormatError("snapshot header: name count does not match n_vars")
    names = b"".join(n.encode() + b"\0" for n in var_names)
    rc = _lib.load().dopinf_b200_write_field(block._h, _lib.dptr(tr), r, _lib.dptr(qt), qt.shape[0],
                                             _lib.dptr(means), _lib.dptr(scales),
                                             1 if params.scaling_enabled else 0, names, os.fsencode(path))
    _check(rc, block.ctx, "write_field")


def snapshot_pass(block: LocalBlock, scaling: bool, out: dict | None = None):
    """Steps II–III of pipeline::run_rank (pipeline.cpp:270-280) in one call:
    returns (TransformParams, D). `out` may carry preallocated (e.g. pinned)
    "means", "scales" and "d" arrays to fill."""
    out = out or {}
    means = _out(out["means"], (block.rows,)) if "means" in out else np.empty(block.rows, dtype=np.float64)
    scales = _out(out["scales"], (block.n_vars,)) if "scales" in out else np.empty(block.n_vars, dtype=np.float64)
    d = _out(out["d"], (block.nt, block.nt)) if "d" in out else np.empty((block.nt, block.nt), dtype=np.float64)
    _check(_lib.load().dopinf_b200_snapshot_pass(block._h, 1 if scaling else 0, _lib.dptr(means),
                                                 _lib.dptr(scales), _lib.dptr(d)), block.ctx, "snapshot_pass")
    block.ctx._gram_nt = block.nt
    params = TransformParams(means, scales if scaling else np.zeros(0), scaling)
    return params, d


def snapshot_pass_host(block: LocalBlock, host_values, scaling: bool, out: dict | None = None,
                       host_ld: int | None = None):
    """snapshot_pass with the block's values streamed in from HOST memory
    (`host_values`: a (rows × nt) float64 array, or a raw pointer int with
    `host_ld`), chunk H2D overlapping the transform and Gram of landed chunks.
    Leaves the block resident and transformed; returns (TransformParams, D)."""
    out = out or {}
    if isinstance(host_values, int):
        ptr, ld = C.cast(host_values, _lib._dp), int(host_ld or block.nt)
    else:
        hv = _f64(host_values, (block.rows, block.nt))
        ptr, ld = _lib.dptr(hv), block.nt
    means = _out(out["means"], (block.rows,)) if "means" in out else np.empty(block.rows, dtype=np.float64)
    scales = _out(out["scales"], (block.n_vars,)) if "scales" in out else np.empty(block.n_vars, dtype=np.float64)
    d = _out(out["d"], (block.nt, block.nt)) if "d" in out else np.empty((block.nt, block.nt), dtype=np.float64)
    rc = _lib.load().dopinf_b200_snapshot_pass_host(block._h, ptr, ld, 1 if scaling else 0, _lib.dptr(means),
                                                    _lib.dptr(scales), _lib.dptr(d))
    _check(rc, block.ctx, "snapshot_pass_host")
    block.ctx._gram_nt = block.nt
    return TransformParams(means, scales if scaling else np.zeros(0), scaling), d


def kernel_launches() -> int:
    return int(_lib.load().dopinf_b200_kernel_launches())


def stream_pass_synth(ctx: DeviceContext, n_vars: int, row_range: RowRange, nt: int, seed: int, n_modes: int,
                      dt: float = 1e-3, noise: float = 1e-4, amps=None, scaling: bool = True):
    """Steps II-III over device-generated rows that are never resident (config 4:
    403 GB per GPU): returns (TransformParams, D) — means, scales and the Gram."""
    nx_i = row_range.count()
    means = np.empty(max(n_vars * nx_i, 1), dtype=np.float64)
    scales = np.empty(n_vars, dtype=np.float64)
    d = np.empty((nt, nt), dtype=np.float64)
    a = None if amps is None else _f64(amps, (n_vars,))
    rc = _lib.load().dopinf_b200_stream_pass_synth(ctx._h, n_vars, nx_i, row_range.begin, nt, seed, n_modes, dt,
                                                   noise, _lib.dptr(a), 1 if scaling else 0, _lib.dptr(means),
                                                   _lib.dptr(scales), _lib.dptr(d))
    _check(rc, ctx, "stream_pass_synth")
    ctx._gram_nt = nt
    return TransformParams(means[: n_vars * nx_i], scales if scaling else np.zeros(0), scaling), d
