"""Times (and, under ncu, exposes) the Step V field kernel at config-5 size:
1,048,576 rows, nt_p = 2400, r from argv (default 20); device-resident output."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_14338_b200 import api  # noqa: E402


def main():
    rs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "20").split(",")]
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    nv, nx, K, nt_p = 4, 262144, 1200, 2400
    with api.DeviceContext(0) as ctx:
        b = api.LocalBlock(ctx, nv, api.RowRange(0, nx), K)
        b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
        params, d = api.snapshot_pass(b, scaling=True)
        lam, vec = np.linalg.eigh(d)
        for r in rs:
            tr = np.ascontiguousarray(vec[:, ::-1][:, :r] / np.sqrt(lam[::-1][:r]))
            qt = np.random.default_rng(6).standard_normal((nt_p, r))
            ts = []
            for _ in range(reps):
                api.reconstruct_field(b, tr, qt, params, download=False)
                ts.append(ctx.stage_ms("field"))
            best = min(ts)
            n = nv * nx
            print(f"r={r} field best {best:.3f} ms  write {8 * n * nt_p / best / 1e6:.1f} GB/s  "
                  f"{2 * n * nt_p * r / best / 1e9:.2f} TFLOP/s  all {[round(t, 3) for t in ts]}")
        b.close()


if __name__ == "__main__":
    main()
