"""ctypes wrappers of the CPU checkers. TEST INFRASTRUCTURE ONLY.

* `Oracle` — the C restatement (oracle/dopinf_oracle.c → _build/libdopinf_oracle.so),
  compiled on demand with gcc if the prebuilt .so is missing (the GPU box has gcc).
* `Reference` — the unmodified reference compiled from /root/reference
  (oracle/_ref/libdopinf_refbench.so, prebuilt here; absent elsewhere → None).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "_build" / "libdopinf_oracle.so"
REF_SO = HERE / "_ref" / "libdopinf_refbench.so"

_dp = C.POINTER(C.c_double)
_sp = C.POINTER(C.c_size_t)


def _d(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class Oracle:
    """CPU restatement of the reference arithmetic (see dopinf_oracle.c)."""

    _lib = None

    def __init__(self):
        if Oracle._lib is None:
            if not ORACLE_SO.exists():
                ORACLE_SO.parent.mkdir(exist_ok=True)
                subprocess.run(["gcc", "-O2", "-std=c11", "-mavx2", "-mfma", "-ffp-contract=off", "-fPIC", "-shared", "-o",
                                str(ORACLE_SO), str(HERE / "dopinf_oracle.c"), "-lm"], check=True)
            lib = C.CDLL(str(ORACLE_SO))
            lib.oracle_rng_new.restype = C.c_void_p
            lib.oracle_rng_new.argtypes = [C.c_uint64]
            lib.oracle_rng_free.argtypes = [C.c_void_p]
            lib.oracle_rng_raw.restype = C.c_uint64
            lib.oracle_rng_raw.argtypes = [C.c_void_p]
            lib.oracle_rng_uniform.restype = C.c_double
            lib.oracle_rng_uniform.argtypes = [C.c_void_p]
            lib.oracle_rng_normal.restype = C.c_double
            lib.oracle_rng_normal.argtypes = [C.c_void_p]
            lib.oracle_rng_fill_normal.argtypes = [C.c_void_p, _dp, C.c_size_t]
            lib.oracle_k_sum.restype = C.c_double
            lib.oracle_k_sum.argtypes = [_dp, C.c_size_t]
            lib.oracle_k_dot.restype = C.c_double
            lib.oracle_k_dot.argtypes = [_dp, _dp, C.c_size_t]
            lib.oracle_k_max_abs.restype = C.c_double
            lib.oracle_k_max_abs.argtypes = [_dp, C.c_size_t]
            lib.oracle_center_in_place.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
            lib.oracle_local_maxabs.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]
            lib.oracle_reduce_scales.restype = C.c_long
            lib.oracle_reduce_scales.argtypes = [_dp, C.c_int, C.c_size_t, _dp]
            lib.oracle_scale_in_place.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]
            lib.oracle_inverse_transform_block.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp,
                                                           C.c_int]
            lib.oracle_gram.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
            lib.oracle_allreduce_sum.argtypes = [_dp, C.c_int, C.c_size_t, _dp]
            lib.oracle_gram_entries.argtypes = [_dp, C.c_size_t, C.c_size_t, _sp, _sp, C.c_size_t, _dp]
            lib.oracle_row_stats.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, _dp]
            lib.oracle_gram_tile.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                             C.c_size_t, _dp]
            lib.oracle_matmul_tn.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _dp]
            lib.oracle_matmul.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _dp]
            lib.oracle_matmul_nt.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _dp]
            lib.oracle_basis_rows.restype = C.c_long
            lib.oracle_basis_rows.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _sp, C.c_size_t, _dp]
            lib.oracle_partition_rows.restype = C.c_int
            lib.oracle_partition_rows.argtypes = [C.c_size_t, C.c_int, _sp, _sp]
            Oracle._lib = lib
        self.lib = Oracle._lib

    # -- rng (synth.cpp:15-34)
    def normals(self, seed: int, count: int) -> np.ndarray:
        r = self.lib.oracle_rng_new(seed)
        out = np.empty(count, dtype=np.float64)
        self.lib.oracle_rng_fill_normal(r, _d(out), count)
        self.lib.oracle_rng_free(r)
        return out

    def rng(self, seed: int):
        return _Rng(self.lib, seed)

    # -- kernels
    def k_dot(self, a, b):
        """kernels_avx2.cpp:32-46 dot_avx2."""
        a, b = _f(a), _f(b)
        return float(self.lib.oracle_k_dot(_d(a), _d(b), a.size))

    def k_sum(self, x):
        x = _f(x)
        return self.lib.oracle_k_sum(_d(x), x.size)

    # -- transform
    def center(self, q):
        q = _f(q).copy()
        rows, cols = q.shape
        means = np.empty(rows)
        self.lib.oracle_center_in_place(_d(q), rows, cols, _d(means))
        return q, means

    def local_maxabs(self, q, n_vars, nx_i):
        q = _f(q)
        out = np.empty(n_vars)
        self.lib.oracle_local_maxabs(_d(q), n_vars, nx_i, q.shape[1], _d(out))
        return out

    def reduce_scales(self, per_rank):
        per_rank = _f(per_rank)
        p, n_vars = per_rank.shape
        out = np.empty(n_vars)
        bad = self.lib.oracle_reduce_scales(_d(per_rank), p, n_vars, _d(out))
        return out, int(bad)

    def scale(self, q, n_vars, nx_i, scales):
        q = _f(q).copy()
        s = _f(scales)
        self.lib.oracle_scale_in_place(_d(q), n_vars, nx_i, q.shape[1], _d(s))
        return q

    def inverse_transform(self, values, nx_i, means, scales, scaling):
        v = _f(values).copy()
        self.lib.oracle_inverse_transform_block(_d(v), v.shape[0], v.shape[1], nx_i, _d(_f(means)),
                                                _d(_f(scales)) if scaling else None, 1 if scaling else 0)
        return v

    # -- pod
    def gram(self, q):
        q = _f(q)
        rows, cols = q.shape
        d = np.empty((cols, cols))
        self.lib.oracle_gram(_d(q), rows, cols, _d(d))
        return d

    def gram_entries(self, q, ii, jj, acc, threads: int = 8):
        """linalg.cpp:50-58 entries (ii[p], jj[p]) continued over the rows of q
        (reference row order per entry; pairs split over threads, each pair's
        chain sequential). acc (float64, len = pairs) is updated in place."""
        from concurrent.futures import ThreadPoolExecutor

        q = np.ascontiguousarray(q, dtype=np.float64)
        ii = np.ascontiguousarray(ii, dtype=np.uintp)
        jj = np.ascontiguousarray(jj, dtype=np.uintp)
        assert acc.dtype == np.float64 and acc.flags.c_contiguous and acc.size == ii.size == jj.size
        rows, ld = q.shape
        bounds = np.linspace(0, ii.size, threads + 1).astype(int)

        def run(t):
            a, b = bounds[t], bounds[t + 1]
            if b > a:
                sub = acc[a:b]
                self.lib.oracle_gram_entries(_d(q), ld, rows, ii[a:b].ctypes.data_as(_sp),
                                             jj[a:b].ctypes.data_as(_sp), b - a, sub.ctypes.data_as(_dp))

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, range(threads)))
        return acc

    def gram_full(self, q, threads: int = 16, tile: int = 128):
        """linalg.cpp:50-58 over the whole of q — the reference's D bit for bit —
        computed as independent 128×128 entry tiles on `threads` threads (the
        oracle's gram() for data too large for one thread)."""
        from concurrent.futures import ThreadPoolExecutor

        assert q.dtype == np.float64 and q.flags.c_contiguous
        rows, k = q.shape
        nb = (k + tile - 1) // tile
        d = np.empty((k, k))
        jobs = [(bi, bj) for bi in range(nb) for bj in range(bi, nb)]

        def run(job):
            bi, bj = job
            i0, j0 = bi * tile, bj * tile
            ni, nj = min(tile, k - i0), min(tile, k - j0)
            out = np.empty((ni, nj))
            self.lib.oracle_gram_tile(_d(q), k, rows, i0, ni, j0, nj, _d(out))
            d[i0:i0 + ni, j0:j0 + nj] = out
            if bi != bj:
                d[j0:j0 + nj, i0:i0 + ni] = out.T

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, jobs))
        return d

    def row_stats(self, q, threads: int = 16):
        """Per row: center_in_place's mean and the max |centered value|
        (transform.cpp:14-15, 29-31) without writing q; rows split over threads."""
        from concurrent.futures import ThreadPoolExecutor

        assert q.dtype == np.float64 and q.flags.c_contiguous
        rows, cols = q.shape
        means, maxabs = np.empty(rows), np.empty(rows)
        bounds = np.linspace(0, rows, threads + 1).astype(int)

        def run(t):
            a, b = bounds[t], bounds[t + 1]
            if b > a:
                self.lib.oracle_row_stats(_d(q[a:b]), cols, b - a, cols, _d(means[a:b]), _d(maxabs[a:b]))

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, range(threads)))
        return means, maxabs

    def center_rows(self, q, threads: int = 16):
        """center() over row slices in parallel (each row is independent):
        returns (centered copy, means) bit-identical to center(q)."""
        from concurrent.futures import ThreadPoolExecutor

        q = np.array(q, dtype=np.float64, order="C", copy=True)
        rows, cols = q.shape
        means = np.empty(rows)
        bounds = np.linspace(0, rows, threads + 1).astype(int)

        def run(t):
            a, b = bounds[t], bounds[t + 1]
            if b > a:
                self.lib.oracle_center_in_place(_d(q[a:b]), b - a, cols, _d(means[a:b]))

        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(run, range(threads)))
        return q, means

    def allreduce_sum(self, parts):
        parts = _f(parts)
        p = parts.shape[0]
        out = np.empty(parts.shape[1:])
        self.lib.oracle_allreduce_sum(_d(parts), p, out.size, _d(out))
        return out

    def matmul_tn(self, a, b):
        a, b = _f(a), _f(b)
        out = np.empty((a.shape[1], b.shape[1]))
        self.lib.oracle_matmul_tn(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[1], _d(out))
        return out

    def project(self, tr, d):
        return self.matmul_tn(tr, d)

    def matmul(self, a, b):
        a, b = _f(a), _f(b)
        out = np.empty((a.shape[0], b.shape[1]))
        self.lib.oracle_matmul(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[1], _d(out))
        return out

    def matmul_nt(self, a, b):
        a, b = _f(a), _f(b)
        out = np.empty((a.shape[0], b.shape[0]))
        self.lib.oracle_matmul_nt(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[0], _d(out))
        return out

    def reconstruct_field(self, q, tr, qtilde, means, scales, nx_i, scaling):
        """postprocess.cpp:63-70: inverse_transform_block(matmul_nt(matmul(q, tr), qtilde))."""
        return self.inverse_transform(self.matmul_nt(self.matmul(q, tr), qtilde), nx_i, means, scales, scaling)

    def basis_rows(self, q, tr, rows):
        q, tr = _f(q), _f(tr)
        sel = np.ascontiguousarray(rows, dtype=np.uintp)
        out = np.empty((sel.size, tr.shape[1]))
        bad = self.lib.oracle_basis_rows(_d(q), q.shape[0], q.shape[1], _d(tr), tr.shape[1],
                                         sel.ctypes.data_as(_sp), sel.size, _d(out))
        if bad >= 0:
            raise IndexError(f"basis_rows: row {int(sel[bad])} outside the local block")
        return out

    def partition_rows(self, nx, p):
        b = np.zeros(max(p, 1), dtype=np.uintp)
        e = np.zeros(max(p, 1), dtype=np.uintp)
        rc = self.lib.oracle_partition_rows(nx, p, b.ctypes.data_as(_sp), e.ctypes.data_as(_sp))
        if rc != 0:
            raise ValueError(f"partition_rows({nx}, {p}) rejected (code {rc})")
        return [(int(x), int(y)) for x, y in zip(b, e)]


class _Rng:
    def __init__(self, lib, seed):
        self.lib = lib
        self.h = lib.oracle_rng_new(seed)

    def normal(self):
        return self.lib.oracle_rng_normal(self.h)

    def uniform(self):
        return self.lib.oracle_rng_uniform(self.h)

    def matrix(self, rows, cols):
        out = np.empty(rows * cols)
        self.lib.oracle_rng_fill_normal(self.h, _d(out), out.size)
        return out.reshape(rows, cols)

    def __del__(self):
        try:
            self.lib.oracle_rng_free(self.h)
        except Exception:  # noqa: BLE001
            pass


class RefError(RuntimeError):
    """A reference exception: `code` as ref_bench.cpp's fail(), `msg` = what()."""

    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code, self.msg = code, msg


class Reference:
    """The unmodified reference (oracle/_ref), or unavailable."""

    _lib = None

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def __init__(self):
        if Reference._lib is None:
            if not REF_SO.exists():
                raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
            lib = C.CDLL(str(REF_SO))
            lib.ref_last_error.restype = C.c_char_p
            lib.ref_backend.restype = C.c_char_p
            lib.ref_set_backend.argtypes = [C.c_char_p]
            lib.ref_rng_normals.argtypes = [C.c_ulonglong, _dp, C.c_size_t]
            lib.ref_snapshot_pass.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.c_int, _dp,
                                              _dp, _dp, _dp]
            lib.ref_gram.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
            lib.ref_global_gram.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_int, _dp]
            lib.ref_center.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
            lib.ref_scale.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp]
            lib.ref_project.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t, _dp]
            lib.ref_matmul.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _dp]
            lib.ref_basis_rows.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _sp, C.c_size_t, _dp]
            lib.ref_eig_reduced_map.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, _dp]
            lib.ref_grid_search.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _dp, C.c_size_t,
                                            C.c_double, C.c_size_t, _dp, _dp]
            lib.ref_pipeline_run.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_long, C.c_int, _dp, C.c_size_t, _dp,
                                             C.c_size_t, C.c_double, C.c_size_t, _sp, _sp, C.c_size_t, _dp, _dp]
            lib.ref_write_snapshots.argtypes = [C.c_char_p, C.c_size_t, C.c_size_t, C.c_size_t, C.c_char_p, _dp]
            lib.ref_read_header.argtypes = [C.c_char_p, _sp, C.c_char_p, C.c_size_t]
            lib.ref_read_block.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp]
            lib.ref_reconstruct_probes.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, _dp,
                                                   C.c_size_t, _dp, C.c_size_t, _dp, _dp, C.c_int, _sp, _sp,
                                                   C.c_size_t, _dp, C.POINTER(C.c_int)]
            lib.ref_integrate.argtypes = [_dp, _dp, _dp, C.c_size_t, _dp, C.c_size_t, _dp, C.POINTER(C.c_int)]
            lib.ref_solve_opinf.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_double, C.c_double, _dp, _dp, _dp]
            lib.ref_reconstruct_field.argtypes = [_dp, C.c_size_t, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _dp,
                                                  C.c_size_t, _dp, _dp, C.c_int, _dp]
            Reference._lib = lib
        self.lib = Reference._lib

    def _ok(self, rc):
        if rc != 0:
            raise RefError(rc, self.lib.ref_last_error().decode())

    def backend(self) -> str:
        return self.lib.ref_backend().decode()

    def normals(self, seed, count):
        out = np.empty(count)
        self.lib.ref_rng_normals(seed, _d(out), count)
        return out

    def snapshot_pass(self, q_full, n_vars, nx, workers, scaling):
        """Steps II-III on `workers` in-process ranks; returns (q_transformed, means, scales, D, seconds)."""
        q = _f(q_full).copy()
        nt = q.shape[1]
        d = np.empty((nt, nt))
        means = np.empty(n_vars * nx)
        scales = np.zeros(n_vars)
        secs = np.zeros(2)
        self._ok(self.lib.ref_snapshot_pass(_d(q), n_vars, nx, nt, workers, 1 if scaling else 0, _d(d),
                                            _d(means), _d(scales), _d(secs)))
        return q, means, scales, d, secs

    def gram(self, q):
        q = _f(q)
        d = np.empty((q.shape[1], q.shape[1]))
        self._ok(self.lib.ref_gram(_d(q), q.shape[0], q.shape[1], _d(d)))
        return d

    def global_gram(self, q, workers):
        q = _f(q)
        d = np.empty((q.shape[1], q.shape[1]))
        self._ok(self.lib.ref_global_gram(_d(q), q.shape[0], q.shape[1], workers, _d(d)))
        return d

    def center(self, q):
        q = _f(q).copy()
        means = np.empty(q.shape[0])
        self._ok(self.lib.ref_center(_d(q), q.shape[0], q.shape[1], _d(means)))
        return q, means

    def scale(self, q, n_vars, nx_i):
        q = _f(q).copy()
        s = np.empty(n_vars)
        self._ok(self.lib.ref_scale(_d(q), n_vars, nx_i, q.shape[1], _d(s)))
        return q, s

    def project(self, tr, d):
        tr, d = _f(tr), _f(d)
        out = np.empty((tr.shape[1], d.shape[0]))
        self._ok(self.lib.ref_project(_d(tr), _d(d), d.shape[0], tr.shape[1], _d(out)))
        return out

    def matmul(self, a, b):
        a, b = _f(a), _f(b)
        out = np.empty((a.shape[0], b.shape[1]))
        self._ok(self.lib.ref_matmul(_d(a), a.shape[0], a.shape[1], _d(b), b.shape[1], _d(out)))
        return out

    def basis_rows(self, q, tr, rows):
        q, tr = _f(q), _f(tr)
        sel = np.ascontiguousarray(rows, dtype=np.uintp)
        out = np.empty((sel.size, tr.shape[1]))
        self._ok(self.lib.ref_basis_rows(_d(q), q.shape[0], q.shape[1], _d(tr), tr.shape[1],
                                         sel.ctypes.data_as(_sp), sel.size, _d(out)))
        return out

    def eig_reduced_map(self, d, r):
        d = _f(d)
        nt = d.shape[0]
        lam = np.empty(nt)
        tr = np.empty((nt, max(r, 1)))
        self._ok(self.lib.ref_eig_reduced_map(_d(d), nt, r, _d(lam), _d(tr)))
        return lam, tr[:, :r]

    def grid_search(self, qhat, b1, b2, max_growth, nt_p):
        qhat = _f(qhat)
        r, nt = qhat.shape
        b1, b2 = _f(b1), _f(b2)
        traj = np.empty((nt_p, r))
        pe = np.empty(3)
        self._ok(self.lib.ref_grid_search(_d(qhat), r, nt, _d(b1), b1.size, _d(b2), b2.size, max_growth, nt_p,
                                          _d(traj), _d(pe)))
        return traj, (pe[0], pe[1]), pe[2]

    def reconstruct_probes(self, q, n_vars, begin, tr, qtilde, means, scales, scaling, var, index):
        """postprocess::reconstruct_probes -> (series n_probes x nt_p, owned flags)."""
        q, tr, qt = _f(q), _f(tr), _f(qtilde)
        rows, nt = q.shape
        nt_p, r = qt.shape
        var = np.ascontiguousarray(var, dtype=np.uintp)
        index = np.ascontiguousarray(index, dtype=np.uintp)
        out = np.full((var.size, nt_p), np.nan)
        owned = (C.c_int * max(var.size, 1))()
        sc = _f(scales) if scaling else np.zeros(max(n_vars, 1))
        self._ok(self.lib.ref_reconstruct_probes(_d(q), n_vars, rows // n_vars, begin, nt, _d(tr), r, _d(qt), nt_p,
                                                 _d(_f(means)), _d(sc), 1 if scaling else 0,
                                                 var.ctypes.data_as(_sp), index.ctypes.data_as(_sp), var.size,
                                                 _d(out), owned))
        return out, np.array(list(owned)[: var.size], dtype=bool)

    def integrate(self, a, f, c, q0, n_steps):
        """rom_search::integrate (rom_search.cpp:60-85) -> (trajectory n_steps x r, finite)."""
        a, f, c, q0 = _f(a), _f(f), _f(c), _f(q0)
        r = a.shape[0]
        traj = np.empty((n_steps, r))
        fin = C.c_int()
        self._ok(self.lib.ref_integrate(_d(a), _d(f), _d(c), r, _d(q0), n_steps, _d(traj), C.byref(fin)))
        return traj, bool(fin.value)

    def solve_opinf(self, qhat, beta1, beta2):
        """opinf::solve_opinf on assemble_data(qhat) -> (A, F, c)."""
        qhat = _f(qhat)
        r, nt = qhat.shape
        s = r * (r + 1) // 2
        a, f, c = np.empty((r, r)), np.empty((r, s)), np.empty(r)
        self._ok(self.lib.ref_solve_opinf(_d(qhat), r, nt, beta1, beta2, _d(a), _d(f), _d(c)))
        return a, f, c

    # ---- data.cpp: SNP1 container ---------------------------------------------------
    def pipeline_run(self, path, out_dir, workers, fixed_rank, scaling, b1, b2, max_growth, nt_p, probes):
        """pipeline::run (pipeline.cpp:400-414) -> (stage_seconds[6] of rank 0, (r, beta1, beta2, train_err))."""
        b1, b2 = _f(b1), _f(b2)
        pv = np.ascontiguousarray([p[0] for p in probes], dtype=np.uintp)
        pi = np.ascontiguousarray([p[1] for p in probes], dtype=np.uintp)
        st, res = np.zeros(6), np.zeros(4)
        self._ok(self.lib.ref_pipeline_run(os.fsencode(str(path)), os.fsencode(str(out_dir)), workers, fixed_rank,
                                           1 if scaling else 0, _d(b1), b1.size, _d(b2), b2.size, max_growth, nt_p,
                                           pv.ctypes.data_as(_sp), pi.ctypes.data_as(_sp), pv.size, _d(st), _d(res)))
        return st, (int(res[0]), float(res[1]), float(res[2]), float(res[3]))

    def write_snapshots(self, path, names, variables):
        """data::write_snapshots (data.cpp:105-131)."""
        full = _f(np.concatenate([np.asarray(v, dtype=np.float64) for v in variables], axis=0))
        nx, nt = np.asarray(variables[0]).shape
        blob = b"".join(n.encode() + b"\0" for n in names)
        self._ok(self.lib.ref_write_snapshots(os.fsencode(str(path)), len(names), nx, nt, blob, _d(full)))

    def read_header(self, path):
        """data::read_header (data.cpp:133-162) -> (n_vars, nx, nt, names)."""
        dims = np.zeros(3, dtype=np.uintp)
        buf = C.create_string_buffer(1 << 16)
        self._ok(self.lib.ref_read_header(os.fsencode(str(path)), dims.ctypes.data_as(_sp), buf, len(buf)))
        n_vars = int(dims[0])
        names = [n.decode() for n in buf.raw.split(b"\0")[:n_vars]]
        return n_vars, int(dims[1]), int(dims[2]), names

    def read_block(self, path, p, rank):
        """data::read_block (data.cpp:164-202) of rank `rank` of partition_rows(nx, p)."""
        n_vars, nx, nt, _ = self.read_header(path)
        nx_i = nx // p if rank + 1 < p else nx - (p - 1) * (nx // p)
        out = np.empty((n_vars * nx_i, nt))
        self._ok(self.lib.ref_read_block(os.fsencode(str(path)), p, rank, _d(out)))
        return out

    def reconstruct_field(self, q, n_vars, tr, qtilde, means, scales, scaling):
        """postprocess::reconstruct_field (postprocess.cpp:63-70) on one rank's block."""
        q, tr, qt = _f(q), _f(tr), _f(qtilde)
        rows, nt = q.shape
        out = np.empty((rows, qt.shape[0]))
        sc = _f(scales) if scaling else np.zeros(max(n_vars, 1))
        self._ok(self.lib.ref_reconstruct_field(_d(q), n_vars, rows // n_vars, nt, _d(tr), tr.shape[1], _d(qt),
                                                qt.shape[0], _d(_f(means)), _d(sc), 1 if scaling else 0, _d(out)))
        return out
