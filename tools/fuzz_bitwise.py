"""Randomised bit-identity fuzz of the device paths that claim the reference's
exact arithmetic, against the compiled reference (oracle/_ref) on the same
bytes (dev tool):
  rom_integrate       vs rom_search::integrate   (r 1..120: register, shared and cluster-DSMEM operator paths)
  reconstruct_probes  vs postprocess::reconstruct_probes
  project             vs pod::project

  python tools/fuzz_bitwise.py [--cases 120] [--seed 0]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle.cpu import Oracle, Reference  # noqa: E402
from paper_2504_14338_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=120)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    ref, o = Reference(), Oracle()
    fails = {"integrate": 0, "probes": 0, "project": 0}
    t0 = time.time()
    with api.DeviceContext(0) as ctx:
        for case in range(args.cases):
            rng = np.random.default_rng(args.seed * 100000 + case)
            # ---- integrate: contractive-ish random operators, some divergent
            r = int(rng.choice([1, 2, 3, 5, 8, 13, 20, 31, 40, 57, 64, 80, 97, 120]))
            d2 = r * (r + 1) // 2
            A = rng.standard_normal((r, r)) * (rng.uniform(0.2, 1.2) / np.sqrt(r))
            F = rng.standard_normal((r, d2)) * rng.uniform(0.0, 0.3) / r
            c = rng.standard_normal(r) * rng.uniform(0.0, 0.1)
            q0 = rng.standard_normal(r)
            steps = int(rng.integers(1, 400))
            want, fw = ref.integrate(A, F, c, q0, steps)
            got, fg = api.rom_integrate(ctx, A, F, c, q0, steps)
            fin = np.isfinite(want)
            if fw != fg or not np.array_equal(np.isfinite(got), fin) or not np.array_equal(got[fin], want[fin]):
                fails["integrate"] += 1
                print(f"FAIL integrate case {case}: r={r} steps={steps}", flush=True)
            # ---- probes on a random transformed block
            nv, nx, nt = int(rng.integers(1, 4)), int(rng.integers(5, 3000)), int(rng.integers(2, 200))
            rr = int(rng.integers(1, nt + 1))
            nt_p = int(rng.integers(1, 500))
            scaling = bool(rng.integers(2))
            q = rng.standard_normal((nv * nx, nt)) * rng.uniform(1e-2, 1e2) + rng.uniform(-5, 5)
            q[:, 0] += 1.0
            b = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt, values=q)
            params, dgram = api.snapshot_pass(b, scaling)
            tr = rng.standard_normal((nt, rr)) * 0.1
            qt = rng.standard_normal((nt_p, rr))
            n_pr = int(rng.integers(1, 40))
            var = rng.integers(0, nv, n_pr)
            idx = rng.integers(0, nx, n_pr)
            series = api.reconstruct_probes(b, tr, qt, [api.Probe(int(v), int(i)) for v, i in zip(var, idx)], params)
            want_s, owned = ref.reconstruct_probes(b.values, nv, 0, tr, qt, params.local_means,
                                                   params.scales if scaling else None, scaling, var, idx)
            if len(series) != n_pr or any(not np.array_equal(s.values, want_s[k]) for k, s in enumerate(series)):
                fails["probes"] += 1
                print(f"FAIL probes case {case}: nv={nv} nx={nx} nt={nt} r={rr} nt_p={nt_p}", flush=True)
            # ---- projection of the pass's D
            if not np.array_equal(api.project(tr, dgram, ctx), o.project(tr, dgram)):
                fails["project"] += 1
                print(f"FAIL project case {case}: nt={nt} r={rr}", flush=True)
            b.close()
    print(f"fuzz_bitwise: {args.cases} cases, failures {fails}, {time.time() - t0:.0f} s", flush=True)
    return 1 if any(fails.values()) else 0


if __name__ == "__main__":
    sys.exit(main())
