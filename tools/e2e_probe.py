"""Where the e2e step's time goes (dev tool): snapshot_pass_host on C2 from pinned memory."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_14338_b200 import api, _lib  # noqa: E402


def main():
    ctx = api.DeviceContext(0)
    nv, nx, nt = 4, 262144, 1200
    b = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt)
    b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
    host = torch.empty((nv * nx, nt), dtype=torch.float64, pin_memory=True)
    assert _lib.load().dopinf_b200_block_download(b._h, _lib.dptr(host.numpy()), nt) == 0
    outs = {"d": torch.empty((nt, nt), dtype=torch.float64, pin_memory=True).numpy(),
            "means": torch.empty(nv * nx, dtype=torch.float64, pin_memory=True).numpy(),
            "scales": torch.empty(nv, dtype=torch.float64, pin_memory=True).numpy()}
    for rep in range(4):
        t0 = time.perf_counter()
        api.snapshot_pass_host(b, host.data_ptr(), scaling=True, out=outs, host_ld=nt)
        wall = (time.perf_counter() - t0) * 1e3
        print(f"rep {rep}: wall {wall:.1f} ms, stream {ctx.stage_ms('stream'):.1f} ms, "
              f"stream_gram {ctx.stage_ms('stream_gram'):.1f} ms, H2D-bound floor {8 * nv * nx * nt / 55.5e6:.1f} ms",
              flush=True)


if __name__ == "__main__":
    main()
