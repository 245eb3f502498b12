"""Quick device-timed probe of the snapshot pass at a given config (dev tool)."""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2504_14338_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nvars", type=int, default=4)
    ap.add_argument("--nx", type=int, default=262144)
    ap.add_argument("--nt", type=int, default=1200)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--lowrank", action="store_true")
    ap.add_argument("--r", type=int, default=40)
    args = ap.parse_args()
    ctx = api.DeviceContext(0)
    b = api.LocalBlock(ctx, args.nvars, api.RowRange(0, args.nx), args.nt)
    t0 = time.time()
    if args.lowrank:
        b.synth_lowrank(seed=3, rank=50, amplitude=10.0)
    else:
        b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
    print(f"synth {time.time()-t0:.2f}s")
    n = args.nvars * args.nx
    K = args.nt
    import numpy as np
    for rep in range(args.reps):
        params, d = api.snapshot_pass(b, scaling=True)
        st = {s: ctx.stage_ms(s) for s in ("stats", "apply", "gram", "gram_reduce", "unpack", "download")}
        g = st["gram"]
        useful = n * K * (K + 1)
        print(f"rep {rep}: " + " ".join(f"{k}={v:.3f}ms" for k, v in st.items()) +
              f" | gram useful {useful/g/1e9:.2f} TFLOP/s, snapshot {8*n*K/g/1e6:.1f} GB/s"
              f" | transform {(24*n*K)/(st['stats']+st['apply'])/1e6:.1f} GB/s")
    tr = np.random.default_rng(0).standard_normal((K, args.r))
    for rep in range(2):
        phi = api.basis(b, tr, download=False)
        bm = ctx.stage_ms("basis")
        print(f"basis r={args.r}: {bm:.3f} ms  {2*n*K*args.r/bm/1e9:.2f} TFLOP/s  "
              f"{8*n*(K+args.r)/bm/1e6:.1f} GB/s")
    qh = api.project_resident(ctx, tr)
    print("project ms", ctx.stage_ms("project"), "launches", api.kernel_launches())


if __name__ == "__main__":
    main()
