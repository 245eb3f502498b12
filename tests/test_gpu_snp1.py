"""SNP1 file → device (reference data.cpp:164-202, pipeline.cpp:254-280) on the
B200, through the C ABI: dopinf_b200_block_read returns exactly the bytes the
reference's read_block returns for every rank of every plan, and
dopinf_b200_snapshot_pass_file (read streamed through the pinned ring,
overlapped with centering and the Gram) leaves the same transformed block,
means and scales as the resident pass, bit for bit, with D within the Gram
tolerance of the oracle."""
import numpy as np
import pytest

from _helpers import oracle_pass

pytestmark = pytest.mark.gpu

GRAM_TOL = 1e-12  # north star: Gram rel. Frobenius ≤ 1e-12


def api():
    from paper_2504_14338_b200 import api as a

    return a


def _file(tmp_path, n_vars, nx, nt, seed, name="s.snp"):
    a = api()
    rng = np.random.default_rng(seed)
    vs = [rng.standard_normal((nx, nt)) * 10.0 ** j + 2.0 * j for j in range(n_vars)]
    path = tmp_path / name
    a.write_snapshots(str(path), a.SnapshotHeader(n_vars, nx, nt, [f"v{j}" for j in range(n_vars)]), vs)
    return str(path), np.concatenate(vs)


# nx = 70,001 puts three 32,768-row chunks in each variable: the pinned ring is
# reused several times within one call; nt = 7 exercises the padded pitch.
@pytest.mark.parametrize("n_vars,nx,nt,p", [(1, 5, 2, 1), (3, 70001, 7, 1), (3, 70001, 7, 3), (2, 1000, 64, 4)])
def test_block_read_matches_reference(tmp_path, ctx, reference, n_vars, nx, nt, p):
    a = api()
    path, _ = _file(tmp_path, n_vars, nx, nt, seed=nx + p)
    h = a.read_header(path)
    plan = a.partition_rows(h.nx, p)
    for rank in range(p):
        b = a.read_block(path, plan, rank, h, ctx)
        assert b.row_range == plan[rank]
        assert np.array_equal(b.values, reference.read_block(path, p, rank))
        b.close()


@pytest.mark.parametrize("n_vars,nx,nt,scaling", [(3, 70001, 7, True), (2, 4096, 120, False), (4, 2500, 301, True)])
def test_snapshot_pass_file_matches_resident(tmp_path, ctx, oracle, n_vars, nx, nt, scaling):
    a = api()
    path, q = _file(tmp_path, n_vars, nx, nt, seed=nt)
    h = a.read_header(path)
    plan = a.partition_rows(h.nx, 1)
    blk, params, d = a.snapshot_pass_file(path, plan, 0, h, ctx, scaling)
    ref = a.LocalBlock(ctx, n_vars, plan[0], nt, values=q)
    p_ref, d_ref = a.snapshot_pass(ref, scaling)
    assert np.array_equal(params.local_means, p_ref.local_means)
    if scaling:
        assert np.array_equal(params.scales, p_ref.scales)
    assert np.array_equal(blk.values, ref.values)
    full, _, _, od = oracle_pass(oracle, q, n_vars, nx, 1, scaling)
    assert np.array_equal(blk.values, full)
    assert np.linalg.norm(d - od) / np.linalg.norm(od) <= GRAM_TOL
    assert np.linalg.norm(d_ref - od) / np.linalg.norm(od) <= GRAM_TOL
    assert np.array_equal(d, d.T)


def test_snapshot_pass_file_rank_slice(tmp_path, ctx, oracle):
    # a rank's slice of a 3-rank plan on a one-rank context: its own rows only
    a = api()
    n_vars, nx, nt = 2, 9001, 33
    path, q = _file(tmp_path, n_vars, nx, nt, seed=5)
    h = a.read_header(path)
    plan = a.partition_rows(nx, 3)
    blk, params, d = a.snapshot_pass_file(path, plan, 2, h, ctx, scaling=False)
    r = plan[2]
    sl = np.concatenate([q[j * nx + r.begin: j * nx + r.end] for j in range(n_vars)])
    c, m = oracle.center(sl)
    assert np.array_equal(params.local_means, m)
    assert np.array_equal(blk.values, c)
    assert np.linalg.norm(d - oracle.gram(c)) / np.linalg.norm(oracle.gram(c)) <= GRAM_TOL


def test_file_pass_is_deterministic(tmp_path, ctx):
    a = api()
    path, _ = _file(tmp_path, 2, 40000, 96, seed=9)
    h = a.read_header(path)
    plan = a.partition_rows(h.nx, 1)
    _, _, d1 = a.snapshot_pass_file(path, plan, 0, h, ctx, True)
    _, _, d2 = a.snapshot_pass_file(path, plan, 0, h, ctx, True)
    assert np.array_equal(d1, d2)


def test_file_errors(tmp_path, ctx):
    a = api()
    path, _ = _file(tmp_path, 2, 100, 4, seed=1)
    h = a.read_header(path)
    plan = a.partition_rows(h.nx, 2)
    with pytest.raises(a.PartitionError, match="outside plan"):
        a.read_block(path, plan, 2, h, ctx)
    with pytest.raises(a.PartitionError, match="does not cover"):
        a.read_block(path, plan[:1], 0, h, ctx)
    with pytest.raises(a.PartitionError, match="not contiguous"):
        a.read_block(path, [a.RowRange(0, 40), a.RowRange(50, 100)], 0, h, ctx)
    raw = open(path, "rb").read()
    short = tmp_path / "short.snp"
    short.write_bytes(raw[:-8])
    with pytest.raises(a.DataFormatError, match="truncated in variable 'v1'"):
        a.read_block(str(short), plan, 0, h, ctx)
    with pytest.raises(a.DataFormatError, match="truncated in variable 'v1'"):
        a.snapshot_pass_file(str(short), plan, 0, h, ctx, True)
    const = tmp_path / "const.snp"
    a.write_snapshots(str(const), a.SnapshotHeader(2, 10, 3, ["a", "b"]), [np.ones((10, 3)), np.eye(10, 3)])
    with pytest.raises(a.DegenerateVariableError):
        a.snapshot_pass_file(str(const), a.partition_rows(10, 1), 0, a.read_header(str(const)), ctx, True)
    # the context stays usable after every failure
    b = a.read_block(path, plan, 1, h, ctx)
    assert b.values.shape == (2 * 50, 4)
