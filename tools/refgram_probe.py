"""Times the reference-order Gram (gram_ref.cu) on resident blocks: config 2
(4 x 262144 x 1200), config 1 (2 x 16384 x 600) and three single-variable
shapes at K = 256 / 512 / 2048 (dev tool)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_14338_b200 import api  # noqa: E402


def main():
    shapes = [(4, 262144, 1200), (2, 16384, 600), (1, 1048576, 256), (1, 1048576, 512), (1, 262144, 2048)]
    with api.DeviceContext(0) as ctx:
        ctx.set_gram_order("reference")
        for nv, nx, K in shapes:
            b = api.LocalBlock(ctx, nv, api.RowRange(0, nx), K)
            b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
            ts = []
            for _ in range(3):
                api.snapshot_pass(b, scaling=True)
                ts.append(ctx.stage_ms("gram"))
            n = nv * nx
            best = min(ts)
            print(f"{nv}x{nx}x{K}: reference-order Gram {best:.2f} ms, "
                  f"{n * K * (K + 1) / best / 1e9:.2f} TFLOP/s useful ({n * K * (K + 1) / best / 1e9 / 36.5:.1%} of DFMA peak)")
            b.close()


if __name__ == "__main__":
    main()
