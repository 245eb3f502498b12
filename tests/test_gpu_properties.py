"""The reference's own invariant tests, run on the device path end to end
(snapshot pass → device eigensolve → device T_r → projection / Φ_r / probes /
field), with the reference's tolerances:

  test_pod.cpp:172-214         T_rᵀ D T_r = I (≤ 1e-10), Q̂ Q̂ᵀ = Λ_r (≤ 1e-8·λ1)
  test_postprocess.cpp:17-56   Φ_rᵀ Φ_r = I (≤ 1e-8)
  test_postprocess.cpp:67-115  full-rank probes reproduce the raw data (≤ 1e-9)
  test_postprocess.cpp:117-133 the full-rank field reproduces the raw data (≤ 1e-9)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def api():
    from paper_2504_14338_b200 import api as a

    return a


def _pipeline(ctx, oracle, nv, nx, nt, seed, scaling=True):
    a = api()
    raw = oracle.rng(seed).matrix(nv * nx, nt) * np.repeat(10.0 ** np.arange(nv), nx)[:, None] + 2.0
    b = a.LocalBlock(ctx, nv, a.RowRange(0, nx), nt, values=raw)
    params, d = a.snapshot_pass(b, scaling)
    spec = a.eig_sym_desc(ctx)
    return a, raw, b, params, d, spec


@pytest.mark.parametrize("nv,nx,nt,r", [(1, 400, 30, 5), (2, 300, 40, 12), (3, 500, 60, 20)])
def test_projection_whitening_and_covariance(ctx, oracle, nv, nx, nt, r):
    a, raw, b, params, d, spec = _pipeline(ctx, oracle, nv, nx, nt, seed=nt)
    tr = a.reduced_map(ctx, r)
    qhat = a.project_resident(ctx, None, r=r)
    lam = spec.eigenvalues
    # T_rᵀ D T_r = I_r (test_pod.cpp:172-190)
    assert np.max(np.abs(tr.T @ d @ tr - np.eye(r))) <= 1e-10
    # Q̂ Q̂ᵀ = Λ_r (test_pod.cpp:192-203)
    assert np.max(np.abs(qhat @ qhat.T - np.diag(lam[:r]))) <= 1e-8 * lam[0]


@pytest.mark.parametrize("nv,nx,nt,r", [(1, 400, 30, 5), (2, 300, 40, 12)])
def test_basis_orthonormal(ctx, oracle, nv, nx, nt, r):
    # Φ_rᵀ Φ_r = I (test_postprocess.cpp:17-56: stacked basis rows orthonormal)
    a, raw, b, params, d, spec = _pipeline(ctx, oracle, nv, nx, nt, seed=3 * nt)
    a.reduced_map(ctx, r, download=False)
    phi = a.basis(b, None, r=r)
    assert np.max(np.abs(phi.T @ phi - np.eye(r))) <= 1e-8


@pytest.mark.parametrize("scaling", [True, False])
def test_full_rank_probes_and_field_reproduce_raw(ctx, oracle, scaling):
    # test_postprocess.cpp:67-133: with r = full rank and Q̃ = Q̂ᵀ, probes and the
    # field map back to the raw snapshots
    nv, nx, nt = 2, 200, 16
    a, raw, b, params, d, spec = _pipeline(ctx, oracle, nv, nx, nt, seed=11, scaling=scaling)
    r = int(np.sum(spec.eigenvalues > 1e-12 * spec.eigenvalues[0]))
    assert r == nt - 1  # centering removes one direction
    tr = a.reduced_map(ctx, r)
    qhat = a.project_resident(ctx, None, r=r)
    qtilde = np.ascontiguousarray(qhat.T)  # nt × r, rows are time
    field = a.reconstruct_field(b, tr, qtilde, params)
    assert np.max(np.abs(field - raw)) <= 1e-9 * np.max(np.abs(raw))
    probes = [a.Probe(v, i) for v in range(nv) for i in (0, 57, nx - 1)]
    series = a.reconstruct_probes(b, tr, qtilde, probes, params)
    for s in series:
        want = raw[s.probe.var * nx + s.probe.index]
        assert np.max(np.abs(s.values - want)) <= 1e-9 * np.max(np.abs(raw))
