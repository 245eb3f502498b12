"""Step IV grid search timing (dev tool; §8(f) row "OpInf grid search").

Q̂ from the config-2 snapshot pass (4 × 262144 × 1200, device eig, r modes),
then rom_search::grid_search with the reference's default 8 × 8 grid and
nt_p = 2K: the device version (all pairs) against the reference on a sample of
pairs (extrapolated per pair; the reference recomputes DhatᵀDhat per pair).

  python tools/grid_bench.py [--r 40] [--ref-pairs 2]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--r", type=int, default=40)
    ap.add_argument("--nt", type=int, default=1200)
    ap.add_argument("--ref-pairs", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    from paper_2504_14338_b200 import api

    ctx = api.DeviceContext(0)
    nt, r = args.nt, args.r
    b = api.LocalBlock(ctx, 4, api.RowRange(0, 262144), nt)
    b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
    api.snapshot_pass(b, True)
    api.eig_sym_desc(ctx, vectors=False)
    api.reduced_map(ctx, r, download=False)
    qhat = api.project_resident(ctx, None, r=r)
    cfg = api.SearchConfig(api.default_b1(), api.default_b2(), 1.2, 2 * nt)
    best = None
    rec = {"r": r, "nt": nt, "nt_p": 2 * nt, "pairs": 64}
    try:
        for _ in range(args.reps):
            t0 = time.perf_counter()
            out = api.grid_search(qhat, cfg, ctx)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        rec.update({"device_wall_s": round(best, 4), "device_rom_integrate_s": round(out.rom_seconds, 4),
                    "pair_opt": out.pair_opt, "train_err": out.train_err})
    except api.Error as e:
        rec["device_error"] = f"{type(e).__name__}: {e}"

    try:
        from oracle.cpu import Reference

        if Reference.available() and args.ref_pairs > 0:
            ref = Reference()
            b1 = np.array(cfg.b1[: args.ref_pairs])
            t0 = time.perf_counter()
            try:
                ref.grid_search(qhat, b1, np.array(cfg.b2[:1]), 1.2, 2 * nt)
            except RuntimeError as e:  # a 2-pair sample may have no admissible pair; the work is done
                rec["reference_sample_error"] = str(e)
            per_pair = (time.perf_counter() - t0) / args.ref_pairs
            rec.update({"reference_s_per_pair_1core": round(per_pair, 3),
                        "reference_64_pairs_1core_s": round(64 * per_pair, 1),
                        "reference_sample_pairs": args.ref_pairs})
    except Exception as e:  # noqa: BLE001 - dev tool
        rec["reference_error"] = str(e)
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
