"""Device vs reference grid search on the C2 Q̂ (dev tool): same pair? trajectory gap?"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    from paper_2504_14338_b200 import api
    from oracle.cpu import Reference

    r = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    ctx = api.DeviceContext(0)
    b = api.LocalBlock(ctx, 4, api.RowRange(0, 262144), 1200)
    b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
    api.snapshot_pass(b, True)
    api.eig_sym_desc(ctx, vectors=False)
    api.reduced_map(ctx, r, download=False)
    qhat = api.project_resident(ctx, None, r=r)
    cfg = api.SearchConfig(api.default_b1(), api.default_b2(), 1.2, 2400)
    out = api.grid_search(qhat, cfg, ctx)
    traj, pair, err = Reference().grid_search(qhat, np.array(cfg.b1), np.array(cfg.b2), 1.2, 2400)
    gap = np.linalg.norm(out.trajectory - traj) / np.linalg.norm(traj)
    # the reference against itself on Q̂ perturbed at the last bit: its own sensitivity
    q2 = qhat * (1.0 + 2.2e-16 * np.random.default_rng(0).standard_normal(qhat.shape))
    traj2, pair2, err2 = Reference().grid_search(q2, np.array(cfg.b1), np.array(cfg.b2), 1.2, 2400)
    self_gap = np.linalg.norm(traj2 - traj) / np.linalg.norm(traj)
    print(f"r={r} device pair {out.pair_opt} err {out.train_err:.6e} | reference pair {pair} err {err:.6e} | "
          f"trajectory rel {gap:.3e} | reference vs itself on a 1-ulp perturbed Q-hat: pair {pair2} "
          f"err {err2:.6e}, trajectory rel {self_gap:.3e}")


if __name__ == "__main__":
    main()
