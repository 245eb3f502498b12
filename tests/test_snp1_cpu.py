"""SNP1 container (reference data.hpp:11-15, data.cpp:35-162) on the CPU: the
C-ABI header parser (dopinf_b200_snp1_header, context-free, no GPU needed) and
the host writer against the UNMODIFIED reference (oracle/_ref) — identical
files, identical headers, and for every malformed file the same
DataFormatError message, byte for byte."""
import struct

import numpy as np
import pytest

from paper_2504_14338_b200 import api


def _vars(n_vars, nx, nt, seed=0):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((nx, nt)) for _ in range(n_vars)]


def _raw(n_vars, nx, nt, names, payload=b""):
    out = b"SNP1" + struct.pack("<QQQ", n_vars, nx, nt)
    for n in names:
        b = n.encode() if isinstance(n, str) else n
        out += struct.pack("<I", len(b)) + b
    return out + payload


def _both_fail(reference, path):
    with pytest.raises(api.DataFormatError) as ours:
        api.read_header(str(path))
    from oracle.cpu import RefError

    with pytest.raises(RefError) as ref:
        reference.read_header(path)
    assert ref.value.code == 10  # DataFormatError (ref_bench.cpp fail())
    assert str(ours.value) == ref.value.msg
    return ref.value.msg


@pytest.mark.parametrize("shape", [(1, 1, 2), (3, 17, 5), (2, 1000, 64)])
def test_writer_bytes_match_reference(tmp_path, reference, shape):
    n_vars, nx, nt = shape
    names = [f"u{j}" if j % 2 else f"pressure_{j}" for j in range(n_vars)]
    vs = _vars(n_vars, nx, nt, seed=nx)
    ours, ref = tmp_path / "ours.snp", tmp_path / "ref.snp"
    api.write_snapshots(str(ours), api.SnapshotHeader(n_vars, nx, nt, names), vs)
    reference.write_snapshots(ref, names, vs)
    assert ours.read_bytes() == ref.read_bytes()


def test_header_matches_reference(tmp_path, reference):
    names = ["ρ", "velocity_x", "E" * 300]
    path = tmp_path / "h.snp"
    reference.write_snapshots(path, names, _vars(3, 11, 4))
    h = api.read_header(str(path))
    assert (h.n_vars, h.nx, h.nt, h.var_names) == reference.read_header(path)
    dims = (np.zeros(4, dtype=np.uint64))
    from paper_2504_14338_b200 import _lib
    import ctypes as C

    d = (C.c_uint64 * 4)()
    assert _lib.load().dopinf_b200_snp1_header(str(path).encode(), d, None, 0, None) == 0
    dims[:] = list(d)
    # data_offset = 4 + 3*8 + sum(4 + len(name)) (data.cpp:51-58)
    assert dims[3] == 28 + sum(4 + len(n.encode()) for n in names)
    assert path.stat().st_size == dims[3] + 3 * 11 * 4 * 8


def test_names_buffer_too_small(tmp_path, reference):
    from paper_2504_14338_b200 import _lib
    import ctypes as C

    path = tmp_path / "n.snp"
    reference.write_snapshots(path, ["alpha", "beta"], _vars(2, 3, 2))
    d = (C.c_uint64 * 4)()
    need = C.c_size_t()
    lib = _lib.load()
    assert lib.dopinf_b200_snp1_header(str(path).encode(), d, None, 0, C.byref(need)) == 0
    assert need.value == len("alpha") + 1 + len("beta") + 1
    buf = C.create_string_buffer(4)
    assert lib.dopinf_b200_snp1_header(str(path).encode(), d, buf, 4, None) == _lib.ERR_INVALID_ARGUMENT
    assert b"too small" in lib.dopinf_b200_last_error(None)


MALFORMED = {
    "bad_magic": lambda: b"SNP2" + bytes(40),
    "short_magic": lambda: b"SN",
    "trunc_n_vars": lambda: b"SNP1" + b"\x01\x00",
    "trunc_nx": lambda: b"SNP1" + struct.pack("<Q", 1) + b"\x05",
    "trunc_nt": lambda: b"SNP1" + struct.pack("<QQ", 1, 5),
    "implausible_n_vars": lambda: b"SNP1" + struct.pack("<QQQ", (1 << 20) + 1, 5, 5),
    "trunc_name_len": lambda: _raw(2, 3, 2, ["a"]) + b"\x01",
    "trunc_name_bytes": lambda: _raw(1, 3, 2, []) + struct.pack("<I", 10) + b"abc",
    "huge_name_len": lambda: _raw(1, 3, 2, []) + struct.pack("<I", 1 << 24),
    "n_vars_zero": lambda: _raw(0, 3, 2, []),
    "nx_zero": lambda: _raw(1, 0, 2, ["a"]),
    "nt_one": lambda: _raw(1, 3, 1, ["a"], bytes(24)),
    "empty_name": lambda: _raw(2, 3, 2, ["a", ""], bytes(96)),
    "duplicate_name": lambda: _raw(3, 3, 2, ["a", "b", "a"], bytes(144)),
    "trunc_payload_first": lambda: _raw(2, 3, 2, ["a", "b"], bytes(8)),
    "trunc_payload_second": lambda: _raw(2, 3, 2, ["a", "b"], bytes(48 + 40)),
    "trunc_payload_last_byte": lambda: _raw(3, 3, 2, ["a", "b", "c"], bytes(144 - 1)),
    "no_payload": lambda: _raw(3, 4, 2, ["x", "y", "z"]),
}


@pytest.mark.parametrize("case", sorted(MALFORMED))
def test_malformed_header_messages_match_reference(tmp_path, reference, case):
    path = tmp_path / f"{case}.snp"
    path.write_bytes(MALFORMED[case]())
    msg = _both_fail(reference, path)
    assert msg  # the reference's own text, e.g. "snapshot file truncated in variable 'b': ..."


def test_missing_file(tmp_path, reference):
    msg = _both_fail(reference, tmp_path / "does_not_exist.snp")
    assert msg.startswith("cannot open snapshot file")


def test_trailing_bytes_are_accepted(tmp_path, reference):
    # check_payload only rejects short files (data.cpp:75)
    path = tmp_path / "t.snp"
    path.write_bytes(_raw(1, 2, 2, ["a"], bytes(32 + 7)))
    assert api.read_header(str(path)).nx == 2
    assert reference.read_header(path)[1] == 2


@pytest.mark.parametrize("bad", ["count", "shape", "dup"])
def test_writer_validation_matches_reference(tmp_path, bad):
    vs = _vars(2, 3, 4)
    if bad == "count":
        h, v, err = api.SnapshotHeader(3, 3, 4), vs, api.InvalidArgumentError
    elif bad == "shape":
        h, v, err = api.SnapshotHeader(2, 3, 5), vs, api.InvalidArgumentError
    else:
        h, v, err = api.SnapshotHeader(2, 3, 4, ["a", "a"]), vs, api.DataFormatError
    with pytest.raises(err):
        api.write_snapshots(str(tmp_path / "w.snp"), h, v)
