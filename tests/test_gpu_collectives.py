"""The library's NCCL data plane on one B200: a size-1 context created with
DOPINF_B200_CTX_NCCL runs every collective code path (MAX of the scales, the
Gram SUM in both reduction modes, the grid search's MIN / SUM / broadcast, the
host-span all-reduce) through a real NCCL communicator. Results must be
bitwise those of a context without a communicator, and the failure
semantics of the reference's group (comm_inprocess.cpp:41-87, 139-151,
171-196) must hold: deadline -> abort -> poisoned context raising
CollectiveError, idempotent global_gram (pod.cpp:15-18 is a pure function).
"""
import time

import numpy as np
import pytest

from conftest import rel_frob

pytestmark = pytest.mark.gpu


def api():
    from paper_2504_14338_b200 import api as a

    return a


@pytest.fixture(scope="module")
def nctx():
    a = api()
    c = a.DeviceContext(0, nccl=True)
    yield c
    c.close()


def _q(seed, n_vars, nx, nt):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n_vars * nx, nt)) * rng.uniform(0.5, 50.0, (n_vars * nx, 1))
    return q + rng.uniform(-3, 3, (n_vars * nx, 1))


@pytest.mark.parametrize("mode", ["nccl", "ordered"])
@pytest.mark.parametrize("n_vars,nx,nt", [(2, 1500, 97), (4, 4099, 256), (1, 77, 1200)])
def test_snapshot_pass_through_nccl_is_bitwise_the_local_path(ctx, nctx, oracle, mode, n_vars, nx, nt):
    a = api()
    q = _q(nx + nt, n_vars, nx, nt)
    nctx.set_gram_reduce(mode)
    b0 = a.LocalBlock(ctx, n_vars, a.RowRange(0, nx), nt, values=q)
    b1 = a.LocalBlock(nctx, n_vars, a.RowRange(0, nx), nt, values=q)
    p0, d0 = a.snapshot_pass(b0, scaling=True)
    p1, d1 = a.snapshot_pass(b1, scaling=True)
    assert np.array_equal(p0.local_means, p1.local_means)
    assert np.array_equal(p0.scales, p1.scales)  # MAX over one rank through ncclAllReduce
    assert np.array_equal(d0, d1)  # SUM / all-gather + ordered sum over one rank
    assert np.array_equal(b0.values, b1.values)
    # and the reference's values
    _, om = oracle.center(q)
    assert np.array_equal(p1.local_means, om)
    b0.close()
    b1.close()
    nctx.set_gram_reduce("nccl")


def test_streamed_passes_through_nccl(ctx, nctx):
    a = api()
    n_vars, nx, nt = 3, 40000, 130
    q = _q(3, n_vars, nx, nt)
    b0 = a.LocalBlock(ctx, n_vars, a.RowRange(0, nx), nt)
    b1 = a.LocalBlock(nctx, n_vars, a.RowRange(0, nx), nt)
    p0, d0 = a.snapshot_pass_host(b0, q, scaling=True)
    p1, d1 = a.snapshot_pass_host(b1, q, scaling=True)  # per-variable MAX collectives in the stream
    assert np.array_equal(p0.scales, p1.scales) and np.array_equal(d0, d1)
    assert np.array_equal(b0.values, b1.values)
    s0, g0 = a.stream_pass_synth(ctx, 2, a.RowRange(0, 70000), 96, seed=4, n_modes=12, amps=[1e-2, 1e5])
    s1, g1 = a.stream_pass_synth(nctx, 2, a.RowRange(0, 70000), 96, seed=4, n_modes=12, amps=[1e-2, 1e5])
    assert np.array_equal(s0.scales, s1.scales) and np.array_equal(g0, g1)


def test_host_allreduce_ops(nctx):
    # test_comm.cpp:15-44 at size 1, through NCCL: SUM (all-gather + ordered sum), MAX, MIN
    a = api()
    data = np.array([0.0, -0.0, 0.5, 3.25])
    for op in (a.DeviceContext.SUM, a.DeviceContext.MAX, a.DeviceContext.MIN):
        x = data.copy()
        nctx.allreduce(x, op)
        assert np.array_equal(x, data)
    nctx.barrier()


@pytest.mark.parametrize("p", [2, 3, 8])
def test_ordered_sum_is_ascending_rank_order(ctx, oracle, p):
    # comm_inprocess.cpp:101-112: acc = part0; acc += part_r, r ascending -> bitwise
    rng = np.random.default_rng(p)
    parts = rng.standard_normal((p, 10007)) * 10.0 ** rng.integers(-8, 8, (p, 10007))
    got = ctx.ordered_sum(parts)
    assert np.array_equal(got, oracle.allreduce_sum(parts))
    acc = parts[0].copy()
    for r in range(1, p):
        acc = acc + parts[r]
    assert np.array_equal(got, acc)


def test_global_gram_is_repeatable_and_checked(nctx, oracle):
    a = api()
    n_vars, nx, nt = 2, 3000, 64
    q = _q(11, n_vars, nx, nt)
    blk = a.LocalBlock(nctx, n_vars, a.RowRange(0, nx), nt, values=q)
    a.center_in_place(blk)
    loc = a.local_gram(blk)
    d1 = a.global_gram(loc, nctx)
    d2 = a.global_gram(loc, nctx)  # the same local partial again: same D (not p * D)
    assert np.array_equal(d1, d2)
    assert rel_frob(d1, oracle.gram(blk.values)) <= 1e-12
    with pytest.raises(a.InvalidArgumentError, match="caller passed nt = 63"):
        a.global_gram(np.zeros((63, 63)), nctx)
    a.set_gram(nctx, d1)
    with pytest.raises(a.InvalidArgumentError, match="no local Gram"):
        a.global_gram(loc, nctx)
    blk.close()


def test_grid_search_through_nccl(ctx, nctx, oracle):
    a = api()
    r, nt = 5, 60
    rng = oracle.rng(r)
    t = np.arange(nt) * 0.05
    qhat = np.stack([np.exp(-0.05 * (i + 1) * t) * np.cos((i + 2) * t + i) / (i + 1) for i in range(r)])
    qhat = qhat + 1e-3 * rng.matrix(r, nt)
    cfg = a.SearchConfig(list(np.logspace(-8, 0, 5)), list(np.logspace(-4, 4, 5)), 1.2, 2 * nt)
    o0 = a.grid_search(qhat, cfg, ctx)
    o1 = a.grid_search(qhat, cfg, nctx)  # MIN of errors + status, MIN owner claim, broadcast of the packet
    assert o0.pair_opt == o1.pair_opt and o0.owner_rank == o1.owner_rank == 0
    assert o0.train_err == o1.train_err and np.array_equal(o0.trajectory, o1.trajectory)


def test_collective_checks_pass_when_ranks_agree(oracle):
    a = api()
    with a.DeviceContext(0, nccl=True) as c:
        c.set_collective_checks(True)
        q = _q(5, 2, 500, 40)
        b = a.LocalBlock(c, 2, a.RowRange(0, 500), 40, values=q)
        params, d = a.snapshot_pass(b, scaling=True)
        _, om = oracle.center(q)
        assert np.array_equal(params.local_means, om)
        b.close()


def test_collective_timeout_aborts_and_poisons():
    # comm_inprocess.cpp:50-63: a wait on an absent peer ends after the deadline
    # with CollectiveError and poisons the group for every later collective.
    a = api()
    from paper_2504_14338_b200 import _lib

    c = a.DeviceContext(0, nccl=True)
    c.set_collective_timeout(2.0)
    q = _q(6, 2, 1000, 50)
    b = a.LocalBlock(c, 2, a.RowRange(0, 1000), 50, values=q)
    c.debug_inject(_lib.INJECT_STALL)  # the next collective's peers "never arrive"
    t0 = time.time()
    with pytest.raises(a.CollectiveError, match="collective timed out waiting for peer ranks"):
        a.snapshot_pass(b, scaling=True)
    waited = time.time() - t0
    assert 1.5 <= waited <= 30.0
    assert c.poisoned()
    with pytest.raises(a.CollectiveError, match="timed out"):
        c.allreduce(np.ones(3), a.DeviceContext.MAX)
    with pytest.raises(a.CollectiveError, match="timed out"):
        a.snapshot_pass(b, scaling=True)
    # device work that needs no collective still runs on the drained stream
    assert b.values.shape == (2000, 50)
    b.close()
    c.close()


def test_communicator_init_with_absent_peer_times_out():
    # A rank whose peers never join (they failed before the init) ends with
    # CollectiveError after the deadline instead of hanging in the init
    # (comm_inprocess.cpp:50-63 semantics applied to communicator creation).
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = (
        "import sys, time\n"
        f"sys.path.insert(0, {str(root)!r})\n"
        "from paper_2504_14338_b200 import api as a\n"
        "uid = a.DeviceContext.unique_id()\n"
        "t0 = time.time()\n"
        "try:\n"
        "    a.DeviceContext(0, rank=0, size=2, unique_id=uid)\n"
        "    print('created')\n"
        "except a.CollectiveError as e:\n"
        "    print('CollectiveError', round(time.time() - t0, 2), e)\n"
    )
    env = dict(os.environ, DOPINF_B200_COLLECTIVE_TIMEOUT="3")
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=240)
    print(res.stdout, res.stderr[-2000:])
    line = res.stdout.strip().splitlines()[-1]
    assert line.startswith("CollectiveError"), res.stdout + res.stderr
    assert "timed out waiting for peer ranks" in res.stderr  # finish_create's diagnostic
    assert 2.5 <= float(line.split()[1]) <= 60.0


def test_guarded_allocations_and_bitwise_repetition():
    # compute-sanitizer is closed on the B200 pool: guard bytes around every
    # library allocation (no kernel may write outside its buffer) and bitwise
    # repetition of the fixed-order kernels (no race) instead
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, DOPINF_B200_GUARD_BYTES="4096")
    res = subprocess.run([sys.executable, str(root / "tools" / "sanitize_kernels.py"), "--reps", "4"], env=env,
                         capture_output=True, text=True, timeout=900)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "guard violations: 0" in res.stdout and "sanitize run ok" in res.stdout
