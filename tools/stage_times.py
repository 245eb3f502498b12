"""Per-stage device times of one resident snapshot pass (dev tool).

  python tools/stage_times.py [--workload c2|c1] [--reps 3]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_14338_b200 import api  # noqa: E402

WL = {"c2": (4, 262144, 1200, 40, 2, 1e-4), "c1": (2, 16384, 600, 20, 1, 1e-3)}
STAGES = ("stats", "apply", "gram", "gram_reduce", "unpack")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=sorted(WL))
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    nv, nx, nt, modes, seed, noise = WL[args.workload]
    with api.DeviceContext(0) as ctx:
        b = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt)
        for _ in range(args.reps):
            b.synth_oscillator(seed=seed, n_modes=modes, dt=1e-3, noise=noise)
            api.snapshot_pass(b, scaling=True)
            print(" ".join(f"{s}={ctx.stage_ms(s):.4f}" for s in STAGES), flush=True)


if __name__ == "__main__":
    main()
