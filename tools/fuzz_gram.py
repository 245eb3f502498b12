"""Randomised snapshot-pass fuzz against the C oracle (dev tool; the committed
tests hold the pinned cases). Shapes span the Gram plan's regimes: one split,
many splits, the guided tail (n > 2T·768 rows), edge/diagonal tiles of every
width, n_vars 1-6, scaling on/off. Checks: means/scales/transformed block
bit-identical, Gram rel. Frobenius <= 1e-12 and bitwise symmetric, Q̂ bit-identical.

  python tools/fuzz_gram.py [--cases 200] [--seed 0]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from _helpers import oracle_pass  # noqa: E402
from oracle.cpu import Oracle  # noqa: E402
from paper_2504_14338_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    o = Oracle()
    worst, fails = 0.0, 0
    t0 = time.time()
    with api.DeviceContext(0) as ctx:
        for case in range(args.cases):
            rng = np.random.default_rng(args.seed * 100000 + case)
            regime = case % 4
            if regime == 0:      # small everything
                nv, nx, nt = int(rng.integers(1, 7)), int(rng.integers(1, 3000)), int(rng.integers(2, 300))
            elif regime == 1:    # many splits, mid K
                nv, nx, nt = int(rng.integers(1, 4)), int(rng.integers(10000, 40000)), int(rng.integers(100, 700))
            elif regime == 2:    # guided tail at small K (few tiles)
                nv, nx, nt = 1, int(rng.integers(200000, 600000)), int(rng.integers(2, 130))
            else:                # K around tile multiples
                nv = int(rng.integers(1, 3))
                nx = int(rng.integers(2000, 20000))
                nt = int(rng.choice([127, 128, 129, 255, 256, 257, 383, 384, 385, 511, 512, 513]))
            scaling = bool(rng.integers(2))
            q = rng.standard_normal((nv * nx, nt)) * rng.uniform(1e-3, 1e3) + rng.uniform(-10, 10)
            q[:, 0] += 1.0
            b = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt, values=q)
            params, d = api.snapshot_pass(b, scaling)
            full, means, scales, od = oracle_pass(o, q, nv, nx, 1, scaling)
            ok = np.array_equal(params.local_means, means) and np.array_equal(b.values, full)
            ok = ok and (not scaling or np.array_equal(params.scales, scales))
            err = float(np.linalg.norm(d - od) / np.linalg.norm(od))
            ok = ok and err <= 1e-12 and np.array_equal(d, d.T)
            r = int(rng.integers(1, nt + 1))
            tr = rng.standard_normal((nt, r))
            ok = ok and np.array_equal(api.project(tr, d, ctx), o.project(tr, d))
            worst = max(worst, err)
            b.close()
            if not ok:
                fails += 1
                print(f"FAIL case {case}: nv={nv} nx={nx} nt={nt} scaling={scaling} gram_err={err:.3e}", flush=True)
    print(f"fuzz: {args.cases} cases, {fails} failures, worst Gram rel. Frobenius {worst:.3e}, "
          f"{time.time() - t0:.0f} s", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
