"""ctypes binding of the C ABI (include/dopinf_b200.h).

This is exactly the binding a reference-side maintainer would write (see
INTEGRATION.md). It fails loudly when the in-tree sm_100a extension is
missing: there is no CPU fallback for the snapshot pass.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libdopinf_b200.so"

OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_PARTITION = 2
ERR_COLLECTIVE = 3
ERR_DEGENERATE_VARIABLE = 4
ERR_DEVICE = 5
ERR_OUT_OF_MEMORY = 6
ERR_NOT_PSD = 7
ERR_RANK_DEFICIENCY = 8
ERR_SOLVE = 9
ERR_DATA_FORMAT = 10
ERR_NO_ADMISSIBLE_PAIR = 11

SUM, MAX, MIN = 0, 1, 2
CTX_NCCL = 1
INJECT_STALL = 1
INJECT_OOB_STORE = 2
GRAM_REDUCE_ORDERED, GRAM_REDUCE_NCCL = 0, 1
GRAM_ORDER_TENSOR, GRAM_ORDER_REFERENCE = 0, 1

STAGES = ["upload", "stats", "scales", "apply", "gram", "gram_reduce", "allreduce", "unpack",
          "project", "basis", "download", "stream", "stream_gram", "field"]
UNIQUE_ID_BYTES = 128

_dp = C.POINTER(C.c_double)
_sp = C.POINTER(C.c_size_t)
_vp = C.c_void_p
_llp = C.POINTER(C.c_longlong)

# name: (restype, argtypes)
SIGNATURES = {
    "dopinf_b200_abi_version": (C.c_int, []),
    "dopinf_b200_status_string": (C.c_char_p, [C.c_int]),
    "dopinf_b200_kernel_launches": (C.c_uint64, []),
    "dopinf_b200_get_unique_id": (C.c_int, [C.c_char_p]),
    "dopinf_b200_ctx_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)]),
    "dopinf_b200_ctx_create_external": (C.c_int, [C.c_int, _vp, _vp, C.POINTER(_vp)]),
    "dopinf_b200_ctx_create_ex": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_uint, C.POINTER(_vp)]),
    "dopinf_b200_set_collective_timeout": (C.c_int, [_vp, C.c_double]),
    "dopinf_b200_set_collective_checks": (C.c_int, [_vp, C.c_int]),
    "dopinf_b200_ctx_poisoned": (C.c_int, [_vp]),
    "dopinf_b200_check_uniform": (C.c_int, [C.POINTER(C.c_longlong), C.c_int, C.c_int, C.c_char_p, C.c_char_p,
                                            C.c_size_t]),
    "dopinf_b200_debug_inject": (C.c_int, [_vp, C.c_int]),
    "dopinf_b200_debug_guard_violations": (C.c_longlong, []),
    "dopinf_b200_debug_gram_coverage": (C.c_int, [C.c_int, _llp, _llp, _llp, _llp]),
    "dopinf_b200_ordered_sum": (C.c_int, [_vp, _dp, C.c_int, C.c_size_t, _dp]),
    "dopinf_b200_ctx_destroy": (None, [_vp]),
    "dopinf_b200_ctx_rank": (C.c_int, [_vp]),
    "dopinf_b200_ctx_size": (C.c_int, [_vp]),
    "dopinf_b200_last_error": (C.c_char_p, [_vp]),
    "dopinf_b200_set_gram_reduce": (C.c_int, [_vp, C.c_int]),
    "dopinf_b200_set_gram_order": (C.c_int, [_vp, C.c_int]),
    "dopinf_b200_allreduce": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int]),
    "dopinf_b200_barrier": (C.c_int, [_vp]),
    "dopinf_b200_stage_ms": (C.c_int, [_vp, C.c_int, _dp]),
    "dopinf_b200_ctx_stream": (_vp, [_vp]),
    "dopinf_b200_partition_rows": (C.c_int, [C.c_size_t, C.c_int, _sp, _sp]),
    "dopinf_b200_block_create": (C.c_int, [_vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t,
                                            C.POINTER(_vp)]),
    "dopinf_b200_block_destroy": (None, [_vp]),
    "dopinf_b200_block_upload": (C.c_int, [_vp, _dp, C.c_size_t]),
    "dopinf_b200_block_download": (C.c_int, [_vp, _dp, C.c_size_t]),
    "dopinf_b200_block_download_rows": (C.c_int, [_vp, C.c_size_t, C.c_size_t, _dp, C.c_size_t]),
    "dopinf_b200_block_synth_oscillator_vars": (C.c_int, [_vp, C.c_int, C.c_uint64, C.c_int, C.c_double,
                                                           C.c_double, _dp]),
    "dopinf_b200_block_device": (C.c_int, [_vp, C.POINTER(_dp), _sp]),
    "dopinf_b200_block_shape": (C.c_int, [_vp, _sp]),
    "dopinf_b200_block_synth_oscillator": (C.c_int, [_vp, C.c_uint64, C.c_int, C.c_double, C.c_double,
                                                      _dp]),
    "dopinf_b200_block_synth_lowrank": (C.c_int, [_vp, C.c_uint64, C.c_int, C.c_double]),
    "dopinf_b200_center": (C.c_int, [_vp, _dp]),
    "dopinf_b200_global_scales": (C.c_int, [_vp, _dp, _sp]),
    "dopinf_b200_local_maxabs": (C.c_int, [_vp, _dp]),
    "dopinf_b200_scale": (C.c_int, [_vp, _dp]),
    "dopinf_b200_local_gram": (C.c_int, [_vp, _dp]),
    "dopinf_b200_global_gram": (C.c_int, [_vp, _dp, C.c_size_t]),
    "dopinf_b200_project": (C.c_int, [_vp, _dp, C.c_size_t, C.c_size_t, _dp]),
    "dopinf_b200_project_host": (C.c_int, [_vp, _dp, _dp, C.c_size_t, C.c_size_t, _dp]),
    "dopinf_b200_eig_sym_desc": (C.c_int, [_vp, _dp, _dp]),
    "dopinf_b200_set_gram": (C.c_int, [_vp, _dp, C.c_size_t]),
    "dopinf_b200_reduced_map": (C.c_int, [_vp, C.c_size_t, _dp]),
    "dopinf_b200_basis": (C.c_int, [_vp, _dp, C.c_size_t, _dp]),
    "dopinf_b200_basis_device": (C.c_int, [_vp, C.POINTER(_dp), _sp]),
    "dopinf_b200_basis_rows": (C.c_int, [_vp, _dp, C.c_size_t, _sp, C.c_size_t, _dp]),
    "dopinf_b200_snapshot_pass": (C.c_int, [_vp, C.c_int, _dp, _dp, _dp]),
    "dopinf_b200_snapshot_pass_host": (C.c_int, [_vp, _dp, C.c_size_t, C.c_int, _dp, _dp, _dp]),
    "dopinf_b200_stream_pass_synth": (C.c_int, [_vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64,
                                                 C.c_int, C.c_double, C.c_double, _dp, C.c_int, _dp, _dp, _dp]),
    "dopinf_b200_snp1_header": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t,
                                          C.POINTER(C.c_size_t)]),
    "dopinf_b200_distribute_pairs": (C.c_int, [C.c_size_t, C.c_int, C.c_int, _sp, _sp]),
    "dopinf_b200_grid_search": (C.c_int, [_vp, _dp, C.c_size_t, C.c_size_t, _dp, C.c_size_t, _dp, C.c_size_t,
                                          C.c_double, C.c_size_t, _dp, _dp, C.POINTER(C.c_int), _dp, _dp]),
    "dopinf_b200_rom_integrate": (C.c_int, [_vp, _dp, _dp, _dp, C.c_size_t, _dp, C.c_size_t, _dp,
                                            C.POINTER(C.c_int)]),
    "dopinf_b200_reconstruct_field": (C.c_int, [_vp, _dp, C.c_size_t, _dp, C.c_size_t, _dp, _dp, C.c_int, _dp]),
    "dopinf_b200_reconstruct_probes": (C.c_int, [_vp, _dp, C.c_size_t, _dp, C.c_size_t, _sp, _sp, C.c_size_t, _dp,
                                                 _dp, C.c_int, _dp, C.POINTER(C.c_int)]),
    "dopinf_b200_field_device": (C.c_int, [_vp, C.POINTER(_dp), C.POINTER(C.c_size_t)]),
    "dopinf_b200_write_field": (C.c_int, [_vp, _dp, C.c_size_t, _dp, C.c_size_t, _dp, _dp, C.c_int, C.c_char_p,
                                          C.c_char_p]),
    "dopinf_b200_block_read": (C.c_int, [_vp, C.c_char_p, C.c_size_t, C.c_size_t, C.POINTER(_vp)]),
    "dopinf_b200_snapshot_pass_file": (C.c_int, [_vp, C.c_char_p, C.c_size_t, C.c_size_t, C.c_int, C.POINTER(_vp),
                                                 _dp, _dp, _dp]),
}

_lib = None


class ExtensionMissing(RuntimeError):
    pass


def load() -> C.CDLL:
    """Load the in-tree extension; raise (never fall back) when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ExtensionMissing(
            f"{LIB_PATH} is missing: build the sm_100a extension with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(str(LIB_PATH), mode=getattr(os, "RTLD_GLOBAL", 0))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def dptr(arr):
    """double* of a C-contiguous float64 numpy array (or None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(_dp)


def sptr(arr):
    if arr is None:
        return None
    return arr.ctypes.data_as(_sp)
