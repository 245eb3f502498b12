"""§8(f) next-row 1: pod::eig_sym_desc / reduced_map on the device (cuSOLVER
dsyevd + the reference's descending order, clamp and sign convention),
checked against the reference's own eig (oracle/_ref: LAPACK dsyev through
pod::eig_sym_desc) when it is present, else against numpy's LAPACK with the
same conventions. Tolerances: eigenvalues <= 1e-10 relative to λ1 (north
star), eigenvectors / T_r / Q̂ <= 1e-9 on well-separated leading modes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def api():
    from paper_2504_14338_b200 import api as a

    return a


def host_eig_sym_desc(d):
    """pod.cpp:20-65 conventions over numpy's LAPACK (fallback checker)."""
    w, v = np.linalg.eigh(d)
    w, v = w[::-1].copy(), v[:, ::-1].copy()
    lam1 = w[0]
    w[(w < 0) & (w >= -1e-10 * lam1)] = 0.0
    for k in range(v.shape[1]):
        col = np.abs(v[:, k])
        p = int(np.argmax(col))  # first index of the max
        if v[p, k] < 0:
            v[:, k] = -v[:, k]
    return w, v


def reference_eig(reference_or_none, d, r):
    if reference_or_none is not None:
        return reference_or_none.eig_reduced_map(d, r)
    w, v = host_eig_sym_desc(d)
    return w, v[:, :r] / np.sqrt(w[:r])


@pytest.fixture(scope="module")
def ref():
    from oracle.cpu import Reference

    return Reference() if Reference.available() else None


def test_known_answers(ctx):
    # test_pod.cpp:58-67, 85-93, 130-142
    a = api()
    a.set_gram(ctx, np.eye(2))
    assert list(a.eig_sym_desc(ctx).eigenvalues) == [1.0, 1.0]
    a.set_gram(ctx, np.array([[4.0, 0.0], [0.0, 0.0]]))
    s = a.eig_sym_desc(ctx)
    assert list(s.eigenvalues) == [4.0, 0.0]
    assert s.eigenvectors[0, 0] == 1.0 and s.eigenvectors[1, 1] == 1.0
    with pytest.raises(a.RankDeficiencyError):
        a.reduced_map(ctx, 2)
    with pytest.raises(a.InvalidArgumentError):
        a.reduced_map(ctx, 3)
    a.set_gram(ctx, np.array([[3 * 0.36, 3 * -0.48], [3 * -0.48, 3 * 0.64]]))
    s = a.eig_sym_desc(ctx)
    assert abs(s.eigenvalues[0] - 3.0) < 1e-14
    assert abs(s.eigenvectors[1, 0] - 0.8) < 1e-14 and abs(s.eigenvectors[0, 0] + 0.6) < 1e-14
    a.set_gram(ctx, 4.0 * np.eye(2))
    a.eig_sym_desc(ctx)
    tr = a.reduced_map(ctx, 2)
    assert np.array_equal(tr, a.eig_sym_desc(ctx).eigenvectors / 2.0)


def test_clamp_and_not_psd(ctx, oracle):
    # test_pod.cpp:72-83: round-off negatives clamp to 0, real negatives throw
    a = api()
    rng = oracle.rng(902)
    u, _ = np.linalg.qr(rng.matrix(6, 6))
    for lam, ok in (([2.0, 1.0, 0.5, 0.1, 0.01, -2e-11], True), ([2.0, 1.0, 0.5, 0.1, 0.01, -2e-8], False)):
        d = (u * np.array(lam)) @ u.T
        d = (d + d.T) / 2
        a.set_gram(ctx, d)
        if ok:
            assert a.eig_sym_desc(ctx).eigenvalues[-1] == 0.0
        else:
            with pytest.raises(a.NotPsdError):
                a.eig_sym_desc(ctx)
    a.set_gram(ctx, -np.eye(2))
    with pytest.raises(a.NotPsdError):
        a.eig_sym_desc(ctx)


@pytest.mark.parametrize("m,nt,r", [(3000, 200, 20), (4000, 600, 10), (500, 50, 10), (1500, 1200, 40)])
def test_eig_against_reference(ctx, oracle, ref, m, nt, r):
    a = api()
    rng = np.random.default_rng(m + nt)
    # decaying spectrum (well-separated leading modes), like POD data
    q = rng.standard_normal((m, nt)) * (0.97 ** np.arange(nt))[None, :] + rng.standard_normal((m, 1))
    d = oracle.gram(q)
    a.set_gram(ctx, d)
    s = a.eig_sym_desc(ctx)
    lam_ref, tr_ref = reference_eig(ref, d, r)
    assert np.max(np.abs(s.eigenvalues - lam_ref)) <= 1e-10 * lam_ref[0]
    tr = a.reduced_map(ctx, r)
    rel = np.linalg.norm(tr - tr_ref, axis=0) / np.linalg.norm(tr_ref, axis=0)
    assert np.max(rel) <= 1e-9, rel
    # Q̂ with the device T_r = reference project(T_r, D) within tolerance
    qhat = a.project_resident(ctx, None, r=r)
    qref = oracle.project(tr_ref, d)
    assert np.max(np.abs(qhat - qref)) <= 1e-9 * np.sqrt(lam_ref[0])


def test_device_step_three_end_to_end(ctx, oracle, ref):
    """snapshot_pass -> eig_sym_desc -> reduced_map -> project / basis, all on
    the device, vs the reference chain on the same bytes."""
    a = api()
    nv, nx, nt, r = 2, 4096, 300, 12
    b = a.LocalBlock(ctx, nv, a.RowRange(0, nx), nt)
    b.synth_lowrank(seed=9, rank=50, amplitude=10.0)  # well-separated leading modes
    raw = b.values
    _, d = a.snapshot_pass(b, scaling=True)
    s = a.eig_sym_desc(ctx, vectors=False)
    a.reduced_map(ctx, r, download=False)
    qhat = a.project_resident(ctx, None, r=r)
    phi = a.basis(b, None, r=r)
    oq, _ = oracle.center(raw)
    oq = oracle.scale(oq, nv, nx, oracle.reduce_scales(oracle.local_maxabs(oq, nv, nx)[None, :])[0])
    dref = oracle.gram(oq)
    lam_ref, tr_ref = reference_eig(ref, dref, r)
    assert np.max(np.abs(s.eigenvalues - lam_ref)) <= 1e-10 * lam_ref[0]
    qref = oracle.project(tr_ref, dref)
    assert np.max(np.abs(qhat - qref)) <= 1e-9 * np.sqrt(lam_ref[0])
    pref = oracle.matmul(oq, tr_ref)
    assert np.linalg.norm(phi - pref) <= 1e-9 * np.linalg.norm(pref)
