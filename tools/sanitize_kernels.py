"""Small-shape run of every device kernel of the library, as the checker in
place of compute-sanitizer (closed on the B200 pool: runs under it have left
GPUs needing a reset):

  * memcheck-lite: run with DOPINF_B200_GUARD_BYTES=4096 and every device
    buffer the library allocates is bracketed by guard bytes; any kernel write
    outside its buffer is counted (dopinf_b200_debug_guard_violations);
  * racecheck-lite: every kernel of a fixed-order design (the Gram's split-n
    reduction, Φ_r, the field, the reference-order Gram, the transforms) must
    give bit-identical results over --reps repetitions; a shared-memory or
    mbarrier race shows up as a difference.

Covers the TMA + mbarrier pipelines (gram_dmma_kernel incl. split-n and the
reduce, basis_dmma_kernel, field_dmma_kernel), the reference-order Gram, the
transform kernels, projection, probes, the streamed pass and the grid search.
    DOPINF_B200_GUARD_BYTES=4096 python tools/sanitize_kernels.py --reps 20
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2504_14338_b200 import api  # noqa: E402


def repeat_bitwise(name, fn, reps):
    first = fn()
    for k in range(reps):
        again = fn()
        for a, b in zip(first, again):
            if not np.array_equal(a, b):
                raise SystemExit(f"{name}: repetition {k} differs bitwise from the first")
    return f"{name}: {reps} repetitions bit-identical"


def stress(reps):
    lines = []
    with api.DeviceContext(0) as ctx:
        rng = np.random.default_rng(1)
        for nv, nx, nt in ((1, 70001, 129), (3, 20000, 640), (2, 50000, 1200), (1, 5, 7)):
            q = rng.standard_normal((nv * nx, nt)) * 3.0 + 0.5
            blk = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt)

            def pass_():
                blk.upload(q)
                p, d = api.snapshot_pass(blk, scaling=True)
                return p.local_means, p.scales, d, blk.values
            lines.append(repeat_bitwise(f"snapshot pass {nv}x{nx}x{nt} (stats, apply, DMMA Gram split-n + reduce)",
                                        pass_, reps))
            _, d = api.snapshot_pass(blk, scaling=True)
            r = min(40, nt)
            lam, vec = np.linalg.eigh(d)
            keep = max(1, int(np.sum(lam > 1e-10 * lam[-1])))
            r = min(r, keep)
            tr = np.ascontiguousarray(vec[:, ::-1][:, :r] / np.sqrt(lam[::-1][:r]))
            lines.append(repeat_bitwise(f"basis r={r}", lambda: (api.basis(blk, tr),), reps))
            qt = np.cos(np.arange(333)[:, None] * 0.01 * (1 + np.arange(r))[None, :])
            params, _ = api.snapshot_pass(blk, scaling=True)
            lines.append(repeat_bitwise(f"field r={r} nt_p=333",
                                        lambda: (api.reconstruct_field(blk, tr, qt, params),), reps))
            ctx.set_gram_order("reference")
            lines.append(repeat_bitwise("reference-order Gram", lambda: (api.local_gram(blk),), max(2, reps // 4)))
            ctx.set_gram_order("tensor")
            ctx.set_gram_reduce("nccl")
            blk.close()
    return lines


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    with api.DeviceContext(0) as ctx:
        nv, nx, nt, r = 2, 2500, 200, 12
        q = rng.standard_normal((nv * nx, nt)) + 1.0
        blk = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt, values=q)
        params, d = api.snapshot_pass(blk, scaling=True)  # stats, apply, DMMA Gram + reduce, unpack
        lam, vec = np.linalg.eigh(d)
        tr = np.ascontiguousarray(vec[:, ::-1][:, :r] / np.sqrt(lam[::-1][:r]))
        qhat = api.project_resident(ctx, tr)
        phi = api.basis(blk, tr)  # basis_dmma_kernel
        api.basis_rows(blk, tr, [0, 7, nv * nx - 1])
        qt = np.cos(np.arange(300)[:, None] * 0.01 * (1 + np.arange(r))[None, :])
        field = api.reconstruct_field(blk, tr, qt, params)  # field_dmma_kernel
        api.reconstruct_probes(blk, tr, qt, [api.Probe(0, 3), api.Probe(1, 2499)], params)
        api.eig_sym_desc(ctx)
        api.reduced_map(ctx, r)
        cfg = api.SearchConfig(api.logspace(1e-6, 1e2, 3), api.logspace(1e-6, 1e2, 3), 1.2, 2 * nt)
        try:
            api.grid_search(qhat[:4], cfg, ctx)
        except api.NoAdmissiblePairError:
            pass
        blk2 = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt)
        api.snapshot_pass_host(blk2, q, scaling=True)  # streamed: chunked H2D, per-variable Grams, combine
        ctx.set_gram_order("reference")
        api.snapshot_pass(blk2, scaling=False)  # gram_ref_kernel
        ctx.set_gram_order("tensor")
        api.stream_pass_synth(ctx, 2, api.RowRange(0, 3000), 64, seed=1, n_modes=4)
        blk.close()
        blk2.close()
        assert np.isfinite(field).all() and np.isfinite(phi).all()
    for line in stress(args.reps):
        print(line, flush=True)
    from paper_2504_14338_b200 import _lib

    lib = _lib.load()
    bad = lib.dopinf_b200_debug_guard_violations()
    print(f"guard violations: {bad}" + (" (guards off: set DOPINF_B200_GUARD_BYTES)" if bad < 0 else ""))
    if bad > 0:
        raise SystemExit(f"{bad} device buffers had their guard bytes overwritten")
    if bad == 0:  # positive control: one store past a buffer must be caught
        with api.DeviceContext(0) as ctx:
            ctx.debug_inject(_lib.INJECT_OOB_STORE)
            caught = lib.dopinf_b200_debug_guard_violations()
        print(f"positive control (one store past a buffer): {caught} violation(s) detected")
        if caught != 1:
            raise SystemExit("the guard check missed an injected out-of-bounds store")
    print("sanitize run ok")


if __name__ == "__main__":
    main()
