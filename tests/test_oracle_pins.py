"""Pin the CPU oracle (oracle/dopinf_oracle.c) before trusting it:
  1. bit-for-bit against the golden vectors the UNMODIFIED reference produced
     (tests/golden/reference_vectors.npz, tests/golden/make_golden.py);
  2. against the reference's own known-answer tests (test_transform.cpp,
     test_linalg.cpp, test_pod.cpp, test_data.cpp);
  3. bit-for-bit against the compiled reference itself on random shapes, when
     oracle/_ref is present (build container).
CPU only.
"""
from pathlib import Path

import numpy as np
import pytest

GOLDEN = np.load(Path(__file__).parent / "golden" / "reference_vectors.npz")


from _helpers import oracle_pass  # noqa: E402


@pytest.mark.parametrize("row", list(range(4)))
def test_transform_golden(oracle, row):
    nv, nx, nt, seed = (int(v) for v in GOLDEN["transform_meta"][row])
    tag = {12: "t12", 8: "t8", 21: "t21", 77: "t77"}[seed]
    q = oracle.rng(seed).matrix(nv * nx, nt)
    qc, mc = oracle.center(q)
    assert np.array_equal(qc, GOLDEN[f"transform_{tag}_centered"])
    assert np.array_equal(mc, GOLDEN[f"transform_{tag}_center_means"])
    for p in (1, 2, 3):
        if f"transform_{tag}_p{p}_q" not in GOLDEN:
            continue
        full, means, scales, d = oracle_pass(oracle, q, nv, nx, p)
        assert np.array_equal(full, GOLDEN[f"transform_{tag}_p{p}_q"])
        assert np.array_equal(means, GOLDEN[f"transform_{tag}_p{p}_means"])
        assert np.array_equal(scales, GOLDEN[f"transform_{tag}_p{p}_scales"])
        assert np.array_equal(d, GOLDEN[f"transform_{tag}_p{p}_gram"])


@pytest.mark.parametrize("tag,m,k,seed", [("g41", 20, 6, 41), ("g5", 13, 7, 5), ("g73", 30, 8, 73),
                                          ("g6", 26, 20, 6)])
def test_gram_golden(oracle, tag, m, k, seed):
    q = oracle.rng(seed).matrix(m, k)
    for p in (1, 2, 4):
        plan = oracle.partition_rows(m, p)
        d = oracle.allreduce_sum(np.stack([oracle.gram(q[b:e]) for b, e in plan]))
        assert np.array_equal(d, GOLDEN[f"gram_{tag}_p{p}"])
        if p == 1:
            assert np.array_equal(d, d.T)


def sweep_input(oracle, i):
    m, nt, rk = (int(v) for v in GOLDEN["sweep_meta"][i])
    rng = oracle.rng(1000 + i)
    if rk == 0:
        return rng.matrix(m, nt)
    a = rng.matrix(m, rk)
    return oracle.matmul(a, rng.matrix(rk, nt))


@pytest.mark.parametrize("i", list(range(20)))
def test_sweep_golden(oracle, i):
    q = sweep_input(oracle, i)
    d1 = oracle.gram(q)
    assert np.array_equal(d1, GOLDEN[f"sweep_{i}_gram_p1"])
    plan = oracle.partition_rows(q.shape[0], 7)
    d7 = oracle.allreduce_sum(np.stack([oracle.gram(q[b:e]) for b, e in plan]))
    assert np.array_equal(d7, GOLDEN[f"sweep_{i}_gram_p7"])
    tr = GOLDEN[f"sweep_{i}_tr"]
    assert np.array_equal(oracle.project(tr, d1), GOLDEN[f"sweep_{i}_qhat"])
    sel = GOLDEN[f"sweep_{i}_basis_sel"]
    assert np.array_equal(oracle.basis_rows(q, tr, sel), GOLDEN[f"sweep_{i}_basis_rows"])


def test_pipeline_golden(oracle):
    nv, nx, nt, r = (int(v) for v in GOLDEN["pipeline_meta"])
    full, _, _, d = oracle_pass(oracle, GOLDEN["pipeline_input"], nv, nx, 1)
    assert np.array_equal(full, GOLDEN["pipeline_q"])
    assert np.array_equal(d, GOLDEN["pipeline_gram"])
    assert np.array_equal(oracle.project(GOLDEN["pipeline_tr"], d), GOLDEN["pipeline_qhat"])


# ---- known-answer tests of the reference suites -------------------------------------------
def test_kat_transform(oracle):
    q, m = oracle.center(np.array([[1.0, 3.0], [2.0, 2.0]]))        # test_transform.cpp:40-44
    assert list(m) == [2.0, 2.0] and np.array_equal(q, [[-1.0, 1.0], [0.0, 0.0]])
    q, m = oracle.center(np.array([[-3.0, 1.0, 3.0, -1.0]]))       # :46-49
    assert list(m) == [0.0] and np.array_equal(q, [[-3.0, 1.0, 3.0, -1.0]])
    # :69-85 cross-rank MAX: ranks hold [-3, 1] and [-2, 5] of one variable
    s, bad = oracle.reduce_scales(np.array([[oracle.local_maxabs(np.array([[-3.0, 1.0]]), 1, 1)[0]],
                                            [oracle.local_maxabs(np.array([[-2.0, 5.0]]), 1, 1)[0]]]))
    assert list(s) == [5.0] and bad == -1
    q = np.array([[-4.0, 2.0, 1.0]])                                  # :87-96
    s, _ = oracle.reduce_scales(oracle.local_maxabs(q, 1, 1)[None, :])
    assert list(s) == [4.0] and np.array_equal(oracle.scale(q, 1, 1, s), [[-1.0, 0.5, 0.25]])
    q, _ = oracle.center(np.array([[4.0, 4, 4], [1, 2, 3]]))          # :115-128 degenerate var0
    _, bad = oracle.reduce_scales(oracle.local_maxabs(q, 2, 1)[None, :])
    assert bad == 0


def test_kat_scaled_bound(oracle):
    # test_transform.cpp:98-113 with the reference stream Rng(8)
    q, _ = oracle.center(oracle.rng(8).matrix(30, 11))
    s, _ = oracle.reduce_scales(oracle.local_maxabs(q, 2, 15)[None, :])
    v = oracle.scale(q, 2, 15, s)
    assert np.all(np.abs(v) <= 1.0) and np.max(np.abs(v)) == 1.0


def test_kat_forward_inverse(oracle):
    # test_transform.cpp:130-150
    raw = oracle.rng(21).matrix(24, 9)
    q, m = oracle.center(raw)
    s, _ = oracle.reduce_scales(oracle.local_maxabs(q, 2, 12)[None, :])
    back = oracle.inverse_transform(oracle.scale(q, 2, 12, s), 12, m, s, True)
    assert np.allclose(back, raw, rtol=1e-12, atol=0)


def test_kat_linalg(oracle):
    # test_linalg.cpp:14-38
    a = np.array([[1.0, 2, 3], [4, 5, 6]])
    b = np.array([[7.0, 8], [9, 10], [11, 12]])
    assert np.array_equal(oracle.matmul(a, b), [[58, 64], [139, 154]])
    tn = oracle.matmul_tn(a, np.eye(2))
    assert tn[0, 0] == 1 and tn[0, 1] == 4 and tn[2, 1] == 6
    g = oracle.gram(oracle.rng(5).matrix(13, 7))                     # :40-62
    assert np.array_equal(g, g.T)


def test_kat_partition(oracle):
    # test_data.cpp:19-62
    assert oracle.partition_rows(8, 2) == [(0, 4), (4, 8)]
    assert oracle.partition_rows(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert [e - b for b, e in oracle.partition_rows(146339, 4)] == [36584, 36584, 36584, 36587]
    assert oracle.partition_rows(5, 1) == [(0, 5)]
    for nx, p in ((10, 0), (10, -1), (3, 4)):
        with pytest.raises(ValueError):
            oracle.partition_rows(nx, p)
    for nx in (1, 2, 7, 64, 101):
        for p in range(1, nx + 1):
            plan = oracle.partition_rows(nx, p)
            assert plan[0][0] == 0 and plan[-1][1] == nx
            assert all(plan[i][0] == plan[i - 1][1] for i in range(1, p))
            assert all(e - b == nx // p for b, e in plan[:-1])


# ---- direct pin against the compiled reference (build container only) -----------------------------
def test_rng_matches_reference(oracle, reference):
    for seed in (1, 12, 1000, 4242):
        assert np.array_equal(oracle.normals(seed, 2001), reference.normals(seed, 2001))


@pytest.mark.parametrize("m,k", [(20, 7), (13, 7), (57, 23), (500, 50), (3, 1), (1, 5), (33, 4), (129, 130)])
def test_oracle_bitwise_vs_reference(oracle, reference, m, k):
    rng = np.random.default_rng(m * 7 + k)
    q = rng.standard_normal((m, k)) * 10 + 3
    assert np.array_equal(oracle.gram(q), reference.gram(q))
    assert all(np.array_equal(x, y) for x, y in zip(oracle.center(q), reference.center(q)))
    tr = rng.standard_normal((k, min(5, k)))
    d = oracle.gram(q)
    assert np.array_equal(oracle.project(tr, d), reference.project(tr, d))
    assert np.array_equal(oracle.matmul(q, tr), reference.matmul(q, tr))
    assert np.array_equal(oracle.basis_rows(q, tr, [0, m - 1]), reference.basis_rows(q, tr, [0, m - 1]))


@pytest.mark.parametrize("nv,nx,nt,p", [(2, 15, 11, 1), (2, 15, 11, 2), (3, 40, 33, 3), (4, 50, 17, 4)])
def test_oracle_pass_vs_reference(oracle, reference, nv, nx, nt, p):
    q = np.random.default_rng(nv + nx + nt + p).standard_normal((nv * nx, nt)) * 5 - 2
    rq, rm, rs, rd, _ = reference.snapshot_pass(q, nv, nx, p, True)
    oq, om, os_, od = oracle_pass(oracle, q, nv, nx, p)
    assert np.array_equal(rq, oq) and np.array_equal(rm, om) and np.array_equal(rs, os_)
    assert np.array_equal(rd, od)


@pytest.mark.parametrize("nv,nx,nt,r,nt_p,scaling", [(2, 15, 11, 3, 7, True), (1, 40, 33, 10, 21, False),
                                                   (3, 50, 64, 20, 128, True), (2, 30, 90, 40, 181, True),
                                                   (1, 20, 70, 68, 9, True), (2, 9, 12, 5, 2, False)])
def test_oracle_field_vs_reference(oracle, reference, nv, nx, nt, r, nt_p, scaling):
    # postprocess::reconstruct_field (postprocess.cpp:63-70), bit for bit: matmul's
    # FMA chains, matmul_nt's 8-lane dot (incl. the 4-block and the tail), scale_shift
    rng = oracle.rng(nt + r)
    raw = rng.matrix(nv * nx, nt)
    q, means = oracle.center(raw)
    scales = None
    if scaling:
        scales, _ = oracle.reduce_scales(oracle.local_maxabs(q, nv, nx)[None, :])
        q = oracle.scale(q, nv, nx, scales)
    tr = rng.matrix(nt, r)
    qt = rng.matrix(nt_p, r)
    want = reference.reconstruct_field(q, nv, tr, qt, means, scales, scaling)
    got = oracle.reconstruct_field(q, tr, qt, means, scales, nx, scaling)
    assert np.array_equal(got, want)



@pytest.mark.parametrize("r,nt_p", [(3, 7), (10, 21), (20, 9), (13, 5)])
def test_oracle_probes_vs_reference(oracle, reference, r, nt_p):
    # postprocess::reconstruct_probes restated: basis_rows, kernels::dot, then
    # inverse_transform_row's scale_shift (one FMA per entry), bit for bit
    nv, nx, nt = 2, 30, 17
    rng = oracle.rng(r * 7 + nt_p)
    q, means = oracle.center(rng.matrix(nv * nx, nt))
    scales, _ = oracle.reduce_scales(oracle.local_maxabs(q, nv, nx)[None, :])
    q = oracle.scale(q, nv, nx, scales)
    tr, qt = rng.matrix(nt, r), rng.matrix(nt_p, r)
    var, index = [0, 1, 1, 0], [3, 0, 29, 17]
    want, owned = reference.reconstruct_probes(q, nv, 0, tr, qt, means, scales, True, var, index)
    assert owned.all()
    rows = [v * nx + i for v, i in zip(var, index)]
    basis = oracle.basis_rows(q, tr, np.array(rows, dtype=np.uintp))
    got = np.empty_like(want)
    for k, row in enumerate(rows):
        series = np.array([[oracle.k_dot(basis[k], qt[t]) for t in range(nt_p)]])
        got[k] = oracle.inverse_transform(series, 1, means[row:row + 1], scales[row // nx:row // nx + 1], True)[0]
    assert np.array_equal(got, want)


# ---- the sliced checkers used at config scale (tests/test_gpu_configs.py) ------------------------
@pytest.mark.parametrize("m,k", [(1, 1), (37, 9), (1000, 64), (333, 130)])
def test_sliced_checkers_match_whole_block(oracle, m, k):
    # gram_entries carried over row slices = entries of the whole-block gram
    # (the golden-pinned restatement of linalg.cpp:50-58); row_stats = center's
    # means and the max |centered| that compute_global_scales takes
    q = oracle.rng(m * 7 + k).matrix(m, k) * 3.0 + 1.5
    c, means = oracle.center(q)
    m2, mx = oracle.row_stats(q, threads=3)
    assert np.array_equal(m2, means) and np.array_equal(mx, np.abs(c).max(axis=1))
    c2, means2 = oracle.center_rows(q, threads=5)
    assert np.array_equal(c2, c) and np.array_equal(means2, means)
    d = oracle.gram(c)
    ii, jj = np.triu_indices(k)
    acc = np.zeros(ii.size)
    for a, b in ((0, m // 3), (m // 3, m // 2), (m // 2, m)):
        oracle.gram_entries(c[a:b], ii, jj, acc, threads=4)
    assert np.array_equal(acc, d[ii, jj])
    assert np.array_equal(oracle.gram_full(c, threads=3, tile=16), d)  # tiled, multi-threaded


def test_sliced_gram_entries_vs_reference(oracle, reference):
    q = oracle.rng(5).matrix(4000, 48)
    d = reference.gram(q)
    ii, jj = np.triu_indices(48)
    acc = np.zeros(ii.size)
    for a in range(0, 4000, 1024):
        oracle.gram_entries(q[a:a + 1024], ii, jj, acc)
    assert np.array_equal(acc, d[ii, jj])
    assert np.array_equal(oracle.gram_full(q, threads=4, tile=32), d)
