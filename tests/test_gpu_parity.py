"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same input bytes. Tolerances are the north-star's (BASELINE.json): Gram
relative Frobenius <= 1e-12, Q̂/Φ_r <= 1e-9; transform, projection and
basis_rows are expected (and asserted) bit-identical to the reference order.
"""
import numpy as np
import pytest

from conftest import rel_frob
from _helpers import oracle_pass

pytestmark = pytest.mark.gpu

GRAM_TOL = 1e-12   # north_star: Gram relative Frobenius error
BASIS_TOL = 1e-9   # north_star: Φ_r / Q̂ after sign normalisation


def api():
    from paper_2504_14338_b200 import api as a

    return a


def make_block(ctx, q, n_vars=1):
    a = api()
    rows, nt = q.shape
    nx = rows // n_vars
    return a.LocalBlock(ctx, n_vars, a.RowRange(0, nx), nt, values=q)


# ---- Step II transform: bit-identical to transform.cpp -----------------------------
@pytest.mark.parametrize("n_vars,nx,nt", [(1, 20, 7), (2, 15, 11), (2, 12, 9), (3, 33, 64), (4, 257, 130),
                                          (2, 1000, 601), (1, 5, 1), (1, 3, 2), (2, 64, 4)])
def test_transform_bitwise(ctx, oracle, n_vars, nx, nt):
    a = api()
    rng = np.random.default_rng(nx * 31 + nt)
    q = rng.standard_normal((n_vars * nx, nt)) * rng.uniform(0.1, 1e3) + rng.uniform(-5, 5)
    block = make_block(ctx, q, n_vars)
    header = a.SnapshotHeader(n_vars, nx, nt)
    means = a.center_in_place(block)
    oq, om = oracle.center(q)
    assert np.array_equal(means, om)
    assert np.array_equal(block.values, oq)  # centering alone, materialised
    if nt == 1:  # one snapshot: every centered row is 0 -> the reference throws
        with pytest.raises(a.DegenerateVariableError, match="var0"):
            a.compute_global_scales(block, header, ctx)
        return
    scales = a.compute_global_scales(block, header, ctx)
    os_, bad = oracle.reduce_scales(oracle.local_maxabs(oq, n_vars, nx)[None, :])
    assert bad == -1 and np.array_equal(scales, os_)
    a.scale_in_place(block, scales)
    assert np.array_equal(block.values, oracle.scale(oq, n_vars, nx, os_))


def test_transform_fused_pass_matches_separate_passes(ctx, oracle):
    # center -> scales -> scale without an intermediate download (the fused apply pass)
    a = api()
    rng = np.random.default_rng(5)
    q = rng.standard_normal((2 * 300, 77)) * 3 + 1
    block = make_block(ctx, q, 2)
    a.center_in_place(block)
    s = a.compute_global_scales(block, a.SnapshotHeader(2, 300, 77))
    a.scale_in_place(block, s)
    oq, _ = oracle.center(q)
    assert np.array_equal(block.values, oracle.scale(oq, 2, 300, oracle.local_maxabs(oq, 2, 300)))


def test_known_answers(ctx):
    # test_transform.cpp:40-50, 87-96
    a = api()
    b = make_block(ctx, np.array([[1.0, 3.0], [2.0, 2.0]]), 1)
    assert list(a.center_in_place(b)) == [2.0, 2.0]
    assert np.array_equal(b.values, [[-1.0, 1.0], [0.0, 0.0]])
    b = make_block(ctx, np.array([[-4.0, 2.0, 1.0]]), 1)
    s = a.compute_global_scales(b, a.SnapshotHeader(1, 1, 3))
    assert list(s) == [4.0]
    a.scale_in_place(b, s)
    assert np.array_equal(b.values, [[-1.0, 0.5, 0.25]])


def test_degenerate_variable_names_it(ctx):
    # test_transform.cpp:115-128
    a = api()
    b = make_block(ctx, np.array([[4.0, 4, 4], [1, 2, 3]]), 2)
    a.center_in_place(b)
    with pytest.raises(a.DegenerateVariableError, match="var0"):
        a.compute_global_scales(b, a.SnapshotHeader(2, 1, 3))


def test_scaled_bound_attained(ctx):
    # test_transform.cpp:98-113
    a = api()
    rng = np.random.default_rng(8)
    b = make_block(ctx, rng.standard_normal((30, 11)), 2)
    a.center_in_place(b)
    a.scale_in_place(b, a.compute_global_scales(b, a.SnapshotHeader(2, 15, 11)))
    v = b.values
    assert np.all(np.abs(v) <= 1.0) and np.max(np.abs(v)) == 1.0


# ---- Step III Gram ---------------------------------------------------------------------
GRAM_SHAPES = [(20, 6), (13, 7), (57, 23), (500, 50), (33, 20), (100, 12), (450, 48), (77, 31), (9, 9),
               (1, 1), (3, 5), (2000, 127), (2000, 128), (2000, 129), (1500, 255), (700, 256), (4000, 300),
               (6000, 600), (12345, 200), (32, 1)]


@pytest.mark.parametrize("m,k", GRAM_SHAPES)
def test_gram_matches_oracle(ctx, oracle, m, k):
    a = api()
    rng = np.random.default_rng(m * 1000 + k)
    q = rng.standard_normal((m, k))
    b = make_block(ctx, q)
    d = a.local_gram(b)
    ref = oracle.gram(q)
    assert rel_frob(d, ref) <= GRAM_TOL
    assert np.array_equal(d, d.T)  # bitwise symmetric (linalg.hpp:17)
    d2 = a.global_gram(d, ctx)
    assert np.array_equal(d, d2)   # one rank: the reduction is the identity
    assert np.array_equal(a.local_gram(b), d)  # deterministic split-n order


def test_gram_rank_deficient(ctx, oracle):
    # acceptance.cpp:207-221 rank-deficient shapes: q = A (m×r) B (r×nt)
    a = api()
    for i, (m, nt, r) in enumerate([(500, 50, 5), (300, 30, 3), (120, 40, 10), (64, 16, 1)]):
        rng = oracle.rng(1012 + i)
        q = oracle.matmul(rng.matrix(m, r), rng.matrix(r, nt))
        d = a.local_gram(make_block(ctx, q))
        assert rel_frob(d, oracle.gram(q)) <= GRAM_TOL


def test_gram_empty_block(ctx):
    a = api()
    b = a.LocalBlock(ctx, 2, a.RowRange(0, 0), 9)
    assert np.array_equal(a.local_gram(b), np.zeros((9, 9)))


def test_gram_multi_var_and_scaled(ctx, oracle):
    a = api()
    rng = np.random.default_rng(17)
    nv, nx, nt = 4, 777, 96
    q = rng.standard_normal((nv * nx, nt)) * np.repeat([1e-2, 1.0, 1e3, 1e5], nx)[:, None]
    b = make_block(ctx, q, nv)
    params, d = a.snapshot_pass(b, scaling=True)
    oq, om = oracle.center(q)
    os_, _ = oracle.reduce_scales(oracle.local_maxabs(oq, nv, nx)[None, :])
    oq = oracle.scale(oq, nv, nx, os_)
    assert np.array_equal(params.local_means, om) and np.array_equal(params.scales, os_)
    assert np.array_equal(b.values, oq)
    assert rel_frob(d, oracle.gram(oq)) <= GRAM_TOL


# ---- projection / basis ---------------------------------------------------------------------
@pytest.mark.parametrize("nt,r", [(6, 3), (50, 10), (128, 40), (600, 10), (257, 80)])
def test_project_bitwise(ctx, oracle, nt, r):
    a = api()
    rng = np.random.default_rng(nt + r)
    q = rng.standard_normal((3 * nt, nt))
    d = oracle.gram(q)
    tr = rng.standard_normal((nt, r))
    assert np.array_equal(a.project(tr, d, ctx), oracle.project(tr, d))


def test_project_resident_uses_device_gram(ctx, oracle):
    a = api()
    rng = np.random.default_rng(3)
    q = rng.standard_normal((400, 40))
    b = make_block(ctx, q)
    d = a.global_gram(a.local_gram(b), ctx)
    tr = rng.standard_normal((40, 7))
    assert np.array_equal(a.project_resident(ctx, tr), oracle.project(tr, d))


@pytest.mark.parametrize("rows,nt,r", [(24, 8, 5), (1000, 64, 10), (5000, 300, 20), (3000, 257, 40),
                                       (2048, 1200, 80), (130, 17, 3), (777, 33, 130)])
def test_basis_matches_oracle(ctx, oracle, rows, nt, r):
    a = api()
    rng = np.random.default_rng(rows + nt + r)
    q = rng.standard_normal((rows, nt))
    tr = rng.standard_normal((nt, r)) / np.sqrt(nt)
    b = make_block(ctx, q)
    phi = a.basis(b, tr)
    ref = oracle.matmul(q, tr)
    assert rel_frob(phi, ref) <= 1e-13
    assert np.max(np.abs(phi - ref)) <= BASIS_TOL * np.max(np.abs(ref))
    sel = rng.integers(0, rows, size=min(rows, 17))
    assert np.array_equal(a.basis_rows(b, tr, sel), oracle.basis_rows(q, tr, sel))


def test_basis_rows_rejects_bad_rows(ctx):
    # test_postprocess.cpp:58-65
    a = api()
    b = make_block(ctx, np.array([[1.0, 0], [0, 1], [1, 1], [2, 2]]))
    with pytest.raises(a.InvalidArgumentError):
        a.basis_rows(b, np.zeros((3, 2)), [0])
    with pytest.raises(a.InvalidArgumentError):
        a.basis_rows(b, np.zeros((2, 2)), [4])


def test_partition_rows_known_answers():
    # test_data.cpp:19-47
    a = api()
    assert [(x.begin, x.end) for x in a.partition_rows(10, 3)] == [(0, 3), (3, 6), (6, 10)]
    big = a.partition_rows(146339, 4)
    assert [x.count() for x in big] == [36584, 36584, 36584, 36587]
    for bad in (0, -1):
        with pytest.raises(a.PartitionError):
            a.partition_rows(10, bad)
    with pytest.raises(a.PartitionError):
        a.partition_rows(3, 4)


# ---- device generator + config-1 sized end to end ---------------------------------------------------
def test_config1_pass_against_oracle(ctx, oracle):
    """BASELINE config 1 shape: 2 vars × 16,384 points, K = 600, scaling on."""
    a = api()
    nv, nx, nt = 2, 16384, 600
    b = a.LocalBlock(ctx, nv, a.RowRange(0, nx), nt)
    b.synth_oscillator(seed=1, n_modes=20, dt=1e-3, noise=1e-3)
    raw = b.values
    params, d = a.snapshot_pass(b, scaling=True)
    oq, om = oracle.center(raw)
    os_, _ = oracle.reduce_scales(oracle.local_maxabs(oq, nv, nx)[None, :])
    oq = oracle.scale(oq, nv, nx, os_)
    assert np.array_equal(params.local_means, om)
    assert np.array_equal(params.scales, os_)
    assert np.array_equal(b.values, oq)
    ref = oracle.gram(oq)
    assert rel_frob(d, ref) <= GRAM_TOL


# ---- streamed pass from host memory (dopinf_b200_snapshot_pass_host) ----------------------------
@pytest.mark.parametrize("nv,nx,nt,scaling", [(2, 40000, 64, True), (3, 33000, 37, True), (1, 70000, 129, False),
                                              (4, 100, 9, True), (2, 65536, 200, True)])
def test_streamed_pass_matches_resident(ctx, oracle, nv, nx, nt, scaling):
    a = api()
    rng = np.random.default_rng(nx + nt)
    q = rng.standard_normal((nv * nx, nt)) * np.repeat(10.0 ** np.arange(nv), nx)[:, None] + 3.0
    b1 = make_block(ctx, q, nv)
    p1, d1 = a.snapshot_pass(b1, scaling=scaling)
    v1 = b1.values
    b2 = a.LocalBlock(ctx, nv, a.RowRange(0, nx), nt)
    p2, d2 = a.snapshot_pass_host(b2, q, scaling=scaling)
    assert np.array_equal(p1.local_means, p2.local_means)
    if scaling:
        assert np.array_equal(p1.scales, p2.scales)
    assert np.array_equal(b2.values, v1)          # bit-identical transformed block
    oq, _ = oracle.center(q)
    if scaling:
        oq = oracle.scale(oq, nv, nx, p1.scales)
    assert rel_frob(d2, oracle.gram(oq)) <= GRAM_TOL
    assert np.array_equal(d2, d2.T)
    _, d3 = a.snapshot_pass_host(b2, q, scaling=scaling)
    assert np.array_equal(d2, d3)                 # deterministic


def test_streamed_pass_degenerate_variable(ctx):
    a = api()
    q = np.vstack([np.full((50, 6), 2.5), np.random.default_rng(0).standard_normal((50, 6))])
    b = a.LocalBlock(ctx, 2, a.RowRange(0, 50), 6)
    with pytest.raises(a.DegenerateVariableError):
        a.snapshot_pass_host(b, q, scaling=True)


# ---- against the reference's own outputs (tests/golden, made by the unmodified reference) ------------
def _golden():
    from pathlib import Path

    return np.load(Path(__file__).parent / "golden" / "reference_vectors.npz")


@pytest.mark.parametrize("i", list(range(20)))
def test_sweep_against_reference_golden(ctx, oracle, i):
    a = api()
    g = _golden()
    m, nt, rk = (int(v) for v in g["sweep_meta"][i])
    rng = oracle.rng(1000 + i)
    q = rng.matrix(m, nt) if rk == 0 else oracle.matmul(rng.matrix(m, rk), rng.matrix(rk, nt))
    b = make_block(ctx, q)
    d = a.local_gram(b)
    assert rel_frob(d, g[f"sweep_{i}_gram_p1"]) <= GRAM_TOL
    tr = g[f"sweep_{i}_tr"]
    assert np.array_equal(a.project(tr, g[f"sweep_{i}_gram_p1"], ctx), g[f"sweep_{i}_qhat"])
    assert np.array_equal(a.basis_rows(b, tr, g[f"sweep_{i}_basis_sel"]), g[f"sweep_{i}_basis_rows"])
    phi = a.basis(b, tr)
    assert rel_frob(phi, oracle.matmul(q, tr)) <= BASIS_TOL


@pytest.mark.parametrize("tag", ["t12", "t8", "t21", "t77"])
def test_transform_against_reference_golden(ctx, oracle, tag):
    a = api()
    g = _golden()
    nv, nx, nt, seed = next((int(x) for x in row) for row in g["transform_meta"]
                            if {12: "t12", 8: "t8", 21: "t21", 77: "t77"}[int(row[3])] == tag)
    q = oracle.rng(seed).matrix(nv * nx, nt)
    b = make_block(ctx, q, nv)
    params, d = a.snapshot_pass(b, scaling=True)
    assert np.array_equal(b.values, g[f"transform_{tag}_p1_q"])
    assert np.array_equal(params.local_means, g[f"transform_{tag}_p1_means"])
    assert np.array_equal(params.scales, g[f"transform_{tag}_p1_scales"])
    assert rel_frob(d, g[f"transform_{tag}_p1_gram"]) <= GRAM_TOL


def test_synth_stream_pass_matches_resident(ctx, oracle):
    """Config-4 path: device-generated, never-resident rows (two 262,144-row ring
    chunks per variable here) give the resident pass's means and scales bit for
    bit and its Gram within tolerance."""
    a = api()
    nv, nx, nt = 2, 300000, 24
    amps = np.array([1e-2, 1e5])
    b = a.LocalBlock(ctx, nv, a.RowRange(5, 5 + nx), nt)
    b.synth_oscillator(seed=7, n_modes=12, dt=1e-3, noise=1e-4, amps=amps)
    p1, d1 = a.snapshot_pass(b, scaling=True)
    p2, d2 = a.stream_pass_synth(ctx, nv, a.RowRange(5, 5 + nx), nt, seed=7, n_modes=12, dt=1e-3, noise=1e-4,
                                 amps=amps, scaling=True)
    assert np.array_equal(p1.local_means, p2.local_means)
    assert np.array_equal(p1.scales, p2.scales)
    assert rel_frob(d2, d1) <= GRAM_TOL
    assert ctx.stage_ms("stream_gram") > 0.0


def test_external_stream_context(ctx):
    # dopinf_b200_ctx_create_external: the caller's stream (here torch's), no communicator
    import torch

    a = api()
    s = torch.cuda.Stream()
    ext = a.DeviceContext.external(0, None, s.cuda_stream)
    assert ext.rank() == 0 and ext.size() == 1 and ext.stream() == s.cuda_stream
    rng = np.random.default_rng(4)
    q = rng.standard_normal((2 * 3000, 40)) + 2.0
    b1 = a.LocalBlock(ext, 2, a.RowRange(0, 3000), 40, values=q)
    b2 = a.LocalBlock(ctx, 2, a.RowRange(0, 3000), 40, values=q)
    p1, d1 = a.snapshot_pass(b1, True)
    p2, d2 = a.snapshot_pass(b2, True)
    assert np.array_equal(p1.local_means, p2.local_means) and np.array_equal(d1, d2)
    ext.close()
    s.synchronize()  # the caller's stream outlives the context


@pytest.mark.parametrize("case", list(range(30)))
def test_random_shapes_against_oracle(ctx, oracle, case):
    # seeded random shapes around the tile / chunk / warp-tile boundaries: the fused
    # pass (transform bit-identical, Gram <= 1e-12) and the projection (bit-identical)
    a = api()
    rng = np.random.default_rng(1000 + case)
    nv = int(rng.integers(1, 5))
    nx = int(rng.choice([1, 2, 7, 63, 64, 65, 127, 129, 500, 4097]))
    nt = int(rng.choice([2, 3, 8, 15, 16, 17, 33, 127, 128, 129, 200, 257]))
    if nt == 1 or nx * nv == 0:
        return
    scaling = bool(rng.integers(2))
    q = rng.standard_normal((nv * nx, nt)) * rng.uniform(1e-3, 1e3) + rng.uniform(-10, 10)
    if scaling and nt >= 2:
        q[:, 0] += 1.0  # no variable constant in time
    b = a.LocalBlock(ctx, nv, a.RowRange(0, nx), nt, values=q)
    params, d = a.snapshot_pass(b, scaling)
    full, means, scales, od = oracle_pass(oracle, q, nv, nx, 1, scaling)
    assert np.array_equal(params.local_means, means)
    if scaling:
        assert np.array_equal(params.scales, scales)
    assert np.array_equal(b.values, full)
    assert rel_frob(d, od) <= GRAM_TOL
    assert np.array_equal(d, d.T)
    r = int(rng.integers(1, nt + 1))
    tr = rng.standard_normal((nt, r))
    assert np.array_equal(a.project(tr, d, ctx), oracle.project(tr, d))


# ---- acceptance.cpp:351-419 (criterion 2): partition invariance on the device ------------
@pytest.mark.parametrize("p", [1, 2, 4, 7])
def test_partition_invariance(ctx, oracle, p):
    """The p ranks of partition_rows run one after another on this GPU through
    the stage API (center_in_place → compute_global_scales → scale_in_place →
    local_gram); the MAX and SUM collectives are done on the host in ascending
    rank order (comm_inprocess.cpp:101-112). Transformed rows are bit-identical
    to the unpartitioned oracle's, the summed Gram within the Gram tolerance."""
    a = api()
    nv, nx, nt = 3, 1001, 72
    rng = np.random.default_rng(23)
    q = rng.standard_normal((nv * nx, nt)) * np.repeat([1e-3, 1.0, 1e4], nx)[:, None] + 5.0
    oq, _ = oracle.center(q)
    os_, _ = oracle.reduce_scales(oracle.local_maxabs(oq, nv, nx)[None, :])
    oq = oracle.scale(oq, nv, nx, os_)
    blocks, local_scales = [], []
    for rr in a.partition_rows(nx, p):
        rows = np.concatenate([q[v * nx + rr.begin:v * nx + rr.end] for v in range(nv)])
        b = a.LocalBlock(ctx, nv, rr, nt, values=rows)
        a.center_in_place(b)
        local_scales.append(a.local_maxabs(b))  # the rank-local half; MAX below (transform.cpp:28-32)
        blocks.append((rr, b))
    scales = np.max(np.stack(local_scales), axis=0)
    assert np.array_equal(scales, os_)
    d = None
    for rr, b in blocks:
        a.scale_in_place(b, scales)
        got = b.values
        for v in range(nv):
            want = oq[v * nx + rr.begin:v * nx + rr.end]
            assert np.array_equal(got[v * rr.count():(v + 1) * rr.count()], want)
        g = a.local_gram(b)
        d = g if d is None else d + g
        b.close()
    assert np.array_equal(d, d.T)
    assert rel_frob(d, oracle.gram(oq)) <= GRAM_TOL


@pytest.mark.parametrize("rows,nt", [(210003, 7), (150001, 128), (120007, 300)])
def test_gram_grouped_reduce(ctx, oracle, rows, nt):
    """Few tiles, many splits: the split-n reduction runs in two fixed-order
    levels (groups of consecutive splits, then the groups); odd split counts
    leave a short last group."""
    a = api()
    q = np.random.default_rng(rows).standard_normal((rows, nt)) + 1.0
    b = make_block(ctx, q)
    _, d = a.snapshot_pass(b, scaling=False)
    oq, _ = oracle.center(q)
    assert rel_frob(d, oracle.gram(oq)) <= GRAM_TOL
    b.upload(q)
    _, d2 = a.snapshot_pass(b, scaling=False)
    assert np.array_equal(d, d2) and np.array_equal(d, d.T)


def test_contexts_in_concurrent_threads(oracle):
    """The reference runs its ranks as threads (comm_inprocess.cpp:159-178):
    independent contexts driven from concurrent host threads (ctypes releases
    the GIL) give the same bits as the same passes run one after another."""
    import threading

    a = api()
    rng = np.random.default_rng(77)
    qs = [rng.standard_normal((2 * 20000, 96)) * (k + 1) + k for k in range(3)]
    seq = []
    with a.DeviceContext(0) as c:
        for q in qs:
            b = make_block(c, q, 2)
            p, d = a.snapshot_pass(b, True)
            seq.append((p.local_means.copy(), p.scales.copy(), d, b.values))
            b.close()
    out = [None] * len(qs)
    errors = []

    def worker(k):
        try:
            with a.DeviceContext(0) as c:
                for _ in range(3):
                    b = make_block(c, qs[k], 2)
                    p, d = a.snapshot_pass(b, True)
                    out[k] = (p.local_means.copy(), p.scales.copy(), d, b.values)
                    b.close()
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(qs))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for got, want in zip(out, seq):
        for x, y in zip(got, want):
            assert np.array_equal(x, y)


def test_local_maxabs_no_zero_check(ctx):
    """A rank whose rows of a variable are constant in time reports 0 for it
    (the zero check belongs after the MAX, transform.cpp:33-39)."""
    a = api()
    q = np.vstack([np.full((10, 5), 3.0), np.arange(50.0).reshape(10, 5)])
    b = make_block(ctx, q, 2)
    a.center_in_place(b)
    m = a.local_maxabs(b)
    assert m[0] == 0.0 and m[1] == 2.0


# ---- reference-order Gram mode: D bit-identical to linalg::gram ---------------------------------
@pytest.mark.parametrize("rows,nt", [(0, 5), (1, 1), (17, 7), (300, 127), (300, 128), (257, 129), (4099, 600),
                                     (33, 1200), (2000, 301)])
def test_reference_order_gram_bitwise(oracle, rows, nt):
    a = api()
    with a.DeviceContext(0) as c:
        c.set_gram_order("reference")
        rng = np.random.default_rng(rows * 13 + nt)
        q = rng.standard_normal((rows, nt)) * rng.uniform(0.1, 100.0, (rows, 1))
        blk = a.LocalBlock(c, 1, a.RowRange(0, rows), nt, values=q)
        d = a.local_gram(blk)
        assert np.array_equal(d, oracle.gram(q) if rows else np.zeros((nt, nt)))
        blk.close()


@pytest.mark.parametrize("n_vars,nx,nt,p", [(2, 3000, 97, 1), (4, 1001, 64, 3), (3, 5000, 130, 2)])
def test_reference_order_pass_matches_reference_dataflow(oracle, n_vars, nx, nt, p):
    # pipeline.cpp:270-280 over p ranks with the stage API in reference order:
    # center, per-rank max-abs -> MAX, scale, local Gram, ascending-rank sum
    # (what the ORDERED reduction does over NCCL): D is the reference's bit for bit
    a = api()
    rng = np.random.default_rng(nx + p)
    q = rng.standard_normal((n_vars * nx, nt)) * rng.uniform(0.5, 20.0, (n_vars * nx, 1)) + 1.0
    _, _, scales_ref, d_ref = oracle_pass(oracle, q, n_vars, nx, p)
    with a.DeviceContext(0) as c:
        c.set_gram_order("reference")
        blocks = []
        for rr in a.partition_rows(nx, p):
            vals = np.concatenate([q[j * nx + rr.begin: j * nx + rr.end] for j in range(n_vars)])
            blk = a.LocalBlock(c, n_vars, rr, nt, values=vals)
            a.center_in_place(blk)
            blocks.append(blk)
        maxima = np.max([a.local_maxabs(b) for b in blocks], axis=0)
        assert np.array_equal(maxima, scales_ref)
        grams = []
        for blk in blocks:
            a.scale_in_place(blk, maxima)
            grams.append(a.local_gram(blk))
            blk.close()
        assert np.array_equal(oracle.allreduce_sum(np.stack(grams)), d_ref)


def test_reference_order_streamed_and_synth(oracle):
    a = api()
    n_vars, nx, nt = 3, 50000, 200
    rng = np.random.default_rng(3)
    q = rng.standard_normal((n_vars * nx, nt)) * np.array([1e-2, 1.0, 1e5]).repeat(nx)[:, None] + 0.5
    _, _, scales_ref, d_ref = oracle_pass(oracle, q, n_vars, nx, 1)
    with a.DeviceContext(0) as c:
        c.set_gram_order("reference")
        blk = a.LocalBlock(c, n_vars, a.RowRange(0, nx), nt)
        params, d = a.snapshot_pass_host(blk, q, scaling=True)  # per-variable Gram after its MAX
        assert np.array_equal(params.scales, scales_ref) and np.array_equal(d, d_ref)
        blk.close()
        with pytest.raises(a.InvalidArgumentError, match="reference-order Gram needs the rows resident"):
            a.stream_pass_synth(c, 2, a.RowRange(0, 1000), 64, seed=1, n_modes=4)
