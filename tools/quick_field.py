"""One C5 field reconstruction (dev tool for ncu): 4 x 262144 x 1200, r, nt_p = 2400.

  python tools/quick_field.py [--r 40] [--reps 1]
"""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_14338_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", type=int, default=40)
    ap.add_argument("--nt-p", type=int, default=2400)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    with api.DeviceContext(0) as ctx:
        b = api.LocalBlock(ctx, 4, api.RowRange(0, 262144), 1200)
        b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
        params, d = api.snapshot_pass(b, scaling=True)
        rng = np.random.default_rng(1)
        tr = rng.standard_normal((1200, args.r)) * 1e-3
        qt = rng.standard_normal((args.nt_p, args.r))
        for _ in range(args.reps):
            api.reconstruct_field(b, tr, qt, params, download=False)
            print(f"field_ms {ctx.stage_ms('field'):.3f}", flush=True)


if __name__ == "__main__":
    main()
