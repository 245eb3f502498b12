"""CPU-only checks of the host side: the C ABI library loads and exports every
symbol include/dopinf_b200.h declares, its host-only entry points behave like
the reference, it fails loudly (never falls back) without a GPU, and the
multi-rank host logic works over torch.distributed/gloo with world_size 2."""
import ctypes as C
import os
import re
import socket
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "dopinf_b200.h"


def lib():
    from paper_2504_14338_b200 import _lib

    return _lib.load()


def declared_symbols():
    text = HEADER.read_text()
    decl = r"(?m)^(?:int|void|uint64_t|long long|const char)\s*\*?\s*(dopinf_b200_\w+)\s*\("
    return sorted(set(re.findall(decl, text)))


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 30
    l = lib()
    missing = [n for n in names if not hasattr(l, n)]
    assert not missing, missing
    from paper_2504_14338_b200 import _lib

    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a_only():
    # The fatbin carries sm_100a SASS and nothing else (no PTX/CPU fallback).
    import subprocess

    so = ROOT / "paper_2504_14338_b200" / "libdopinf_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs
    sass = subprocess.run(["cuobjdump", "-sass", str(so)], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass and "UTMALDG" in sass


def test_abi_version_and_status_strings():
    l = lib()
    assert l.dopinf_b200_abi_version() == 2
    assert l.dopinf_b200_status_string(4) == b"DegenerateVariableError"
    assert l.dopinf_b200_status_string(2) == b"PartitionError"


def test_partition_rows_matches_oracle(oracle):
    from paper_2504_14338_b200 import api

    for nx in (1, 2, 7, 64, 101, 146339):
        for p in range(1, min(nx, 9) + 1):
            assert [(r.begin, r.end) for r in api.partition_rows(nx, p)] == oracle.partition_rows(nx, p)
    with pytest.raises(api.PartitionError):
        api.partition_rows(3, 4)
    with pytest.raises(api.PartitionError):
        api.partition_rows(10, 0)


def test_context_fails_loudly_without_gpu():
    """No CUDA device here: creating a context must raise, not fall back."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2504_14338_b200 import api

    with pytest.raises(api.Error):
        api.DeviceContext(0)


def test_missing_extension_raises(tmp_path, monkeypatch):
    from paper_2504_14338_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", tmp_path / "nope.so")
    with pytest.raises(_lib.ExtensionMissing):
        _lib.load()


def test_product_does_not_import_oracle():
    """The product path never imports, links or loads the checker (build.py only
    compiles it, as the build step must)."""
    bad = re.compile(r"(import\s+oracle|from\s+oracle|libdopinf_oracle|libdopinf_ref|oracle/_ref|oracle\.cpu)")
    for path in (ROOT / "paper_2504_14338_b200").rglob("*"):
        if path.suffix in (".py", ".cu", ".cuh", ".h", ".cpp") and path.name != "build.py":
            assert not bad.search(path.read_text()), path
    assert "oracle" not in (ROOT / "include" / "dopinf_b200.h").read_text()


# ---- world_size 2 over gloo: the N>1 host path of bench.py ------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q, nv, nx, nt, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.cpu import Oracle
    from paper_2504_14338_b200 import api
    from paper_2504_14338_b200.distributed import max_over_ranks, share_unique_id

    o = Oracle()
    # bench.py's control plane: rank 0 makes a real NCCL unique id through the
    # C ABI and every rank receives the same 128 bytes
    uid = share_unique_id(rank)
    ids = [None] * world
    dist.all_gather_object(ids, uid)
    assert len(uid) == 128 and all(i == uid for i in ids)
    # the library's verify_uniform rule (dopinf_b200_check_uniform) on the
    # descriptors the ranks all-gather: same verdict on every rank
    verdicts = []
    for count_of in (lambda r: 6, lambda r: 3 if r == 1 else 2):
        desc = torch.tensor([7, count_of(rank), 0], dtype=torch.int64)
        rows = [torch.zeros(3, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(rows, desc)
        try:
            api.check_uniform(torch.stack(rows).numpy(), rank, "allreduce")
            verdicts.append("ok")
        except api.CollectiveError as e:
            verdicts.append(str(e))
    # the reference data flow over the ranks (restated with the oracle): MAX of
    # the scales, ascending-rank SUM of the Grams (comm_inprocess.cpp order)
    plan = api.partition_rows(nx, world)
    b, e = plan[rank].begin, plan[rank].end
    block = np.concatenate([q[j * nx + b: j * nx + e] for j in range(nv)])
    c, _ = o.center(block)
    local_max = torch.from_numpy(o.local_maxabs(c, nv, e - b))
    dist.all_reduce(local_max, op=dist.ReduceOp.MAX)
    c = o.scale(c, nv, e - b, local_max.numpy())
    parts = [torch.zeros(nt * nt, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(o.gram(c).ravel()))
    d = torch.from_numpy(o.allreduce_sum(np.stack([p.numpy() for p in parts])))
    assert max_over_ranks(float(rank)) == world - 1
    np.save(f"{out}.{rank}.npy", np.array(verdicts, dtype=object), allow_pickle=True)
    if rank == 0:
        np.save(out, d.numpy())
    dist.destroy_process_group()


def test_two_rank_gloo_control_plane(tmp_path):
    """world_size 2 over gloo: the real unique-id exchange, the library's
    collective agreement rule on both ranks, and the reference's data flow
    (oracle restatement) against the one-process oracle pass."""
    import torch.multiprocessing as mp

    from oracle.cpu import Oracle
    from _helpers import oracle_pass

    o = Oracle()
    nv, nx, nt = 2, 37, 9
    q = o.rng(99).matrix(nv * nx, nt)
    out = tmp_path / "d.npy"
    mp.start_processes(_rank_main, args=(2, _free_port(), q, nv, nx, nt, str(out)), nprocs=2, join=True,
                       start_method="spawn")
    d = np.load(out).reshape(nt, nt)
    _, _, _, d_ref = oracle_pass(o, q, nv, nx, 2)
    assert np.array_equal(d, d_ref)  # ascending-rank sum = the reference's in-process order
    v0 = list(np.load(f"{out}.0.npy", allow_pickle=True))
    v1 = list(np.load(f"{out}.1.npy", allow_pickle=True))
    assert v0[0] == v1[0] == "ok"
    # test_comm.cpp:95-112: a count mismatch raises on every rank, naming the counts
    assert v0[1] == "allreduce: rank 0 passed count 2, rank 1 passed count 3"
    assert v1[1] == "allreduce: rank 1 passed count 3, rank 0 passed count 2"


def test_check_uniform_rules():
    from paper_2504_14338_b200 import api

    ok = np.array([[4, 10, 1], [4, 10, 1], [4, 10, 1]])
    for r in range(3):
        api.check_uniform(ok, r)
    with pytest.raises(api.CollectiveError, match=r"^allreduce: rank 2 passed count 10, rank 0 passed count 10 "
                                                  r"\(operations differ\)$"):
        api.check_uniform(np.array([[4, 10, 0], [4, 10, 0], [4, 10, 1]]), 2)  # test_comm.cpp:114-123
    with pytest.raises(api.CollectiveError, match="out of step"):
        api.check_uniform(np.array([[4, 10, 1], [5, 10, 1]]), 0, "broadcast")


def test_distribute_pairs_known_answers():
    # test_rom_search.cpp:178-191, through the ABI (host only, no GPU)
    from paper_2504_14338_b200 import api

    for rank in range(8):
        rr = api.distribute_pairs(64, rank, 8)
        assert rr.begin == 8 * rank and rr.count() == 8
    assert api.distribute_pairs(10, 0, 3) == api.RowRange(0, 3)
    assert api.distribute_pairs(10, 1, 3) == api.RowRange(3, 6)
    assert api.distribute_pairs(10, 2, 3) == api.RowRange(6, 10)
    assert [api.distribute_pairs(2, r, 4).count() for r in range(4)] == [1, 1, 0, 0]
    with pytest.raises(api.InvalidArgumentError, match="no candidates"):
        api.distribute_pairs(0, 0, 1)
    with pytest.raises(api.InvalidArgumentError, match="bad rank/size"):
        api.distribute_pairs(4, 4, 4)
