"""The C++ drop-in (include/dopinf_b200.hpp) compiled against the reference's
own headers and library (tests/cpp/parity_main.cpp, built by build() in the
container that has /root/reference): the reference's scenarios with Steps
II-III, Q̂ and Φ_r swapped for the B200 ones, checked against the reference."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "parity"


def test_cpp_dropin_parity():
    if not BIN.exists():
        pytest.skip("tests/cpp/_build/parity not built (needs /root/reference at build time)")
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout


C_BIN = Path(__file__).resolve().parent / "c" / "_build" / "abi_smoke"


def test_c_abi_from_plain_c():
    # tests/c/abi_smoke.c: the ABI from C11 (no C++ anywhere on the caller's side)
    if not C_BIN.exists():
        from paper_2504_14338_b200 import build

        build.build_c_smoke()
    res = subprocess.run([str(C_BIN)], capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "all checks passed" in res.stdout
