"""The Gram kernel's tile plan, checked on the host (no GPU): for every K the
split-n reduction must write each entry of the packed upper triangle exactly
once — through the compile-time mma masks of diagonal / edge tiles, the warp-
tile halves, and the (odd rows, even columns) diagonal mma tiles that are
skipped and written from their transposes (gram.cu scatter_index, the same
function the reduction kernel runs). Also bounds the executed DMMA work: the
useful work is K(K+1) flop per row (the upper triangle)."""
import ctypes as C

import pytest

from paper_2504_14338_b200 import _lib


def coverage(K):
    lib = _lib.load()
    e, c, d, m = (C.c_longlong() for _ in range(4))
    rc = lib.dopinf_b200_debug_gram_coverage(K, C.byref(e), C.byref(c), C.byref(d), C.byref(m))
    assert rc == 0
    return e.value, c.value, d.value, m.value


@pytest.mark.parametrize("K", list(range(1, 300)) + [383, 384, 385, 511, 512, 513, 600, 1023, 1024, 1025,
                                                     1199, 1200, 1201, 1500, 2047, 2048, 2049, 4096])
def test_every_upper_entry_written_once(K):
    entries, covered, duplicates, _ = coverage(K)
    assert entries == K * (K + 1) // 2
    assert covered == entries
    assert duplicates == 0


@pytest.mark.parametrize("K,bound", [(600, 1.04), (1200, 1.007), (1500, 1.011), (4096, 1.002)])
def test_executed_dmma_work_close_to_useful(K, bound):
    # one 8x8x4 DMMA = 512 flop per 4 rows: 128 flop per row per executed mma tile
    *_, mma_tiles = coverage(K)
    ratio = mma_tiles * 128 / (K * (K + 1))
    assert 1.0 <= ratio <= bound


def test_rejects_bad_arguments():
    lib = _lib.load()
    x = C.c_longlong()
    assert lib.dopinf_b200_debug_gram_coverage(0, C.byref(x), C.byref(x), C.byref(x), C.byref(x)) == 1
