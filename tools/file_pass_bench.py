"""SNP1 file → device throughput (dev tool; §8(f) row "SNP1 load → device").

Writes a seeded oscillator snapshot file (the bench generator's bytes), then
times, with the page cache warm and (after posix_fadvise DONTNEED) cold:
  reference  data::read_block (oracle/_ref, ifstream)           host only
  b200       dopinf_b200_block_read (pinned ring + H2D)         file → HBM
  b200       dopinf_b200_snapshot_pass_file (read ‖ transform ‖ Gram)
and prints one JSON line per measurement.

  python tools/file_pass_bench.py [--vars 1] [--nx 262144] [--nt 1200] [--dir /tmp]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def drop(path):
    fd = os.open(path, os.O_RDONLY)
    try:
        os.fsync(fd)
        os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    finally:
        os.close(fd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--vars", type=int, default=1)
    ap.add_argument("--nx", type=int, default=262144)
    ap.add_argument("--nt", type=int, default=1200)
    ap.add_argument("--dir", default="/tmp")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()

    from paper_2504_14338_b200 import api

    ctx = api.DeviceContext(0)
    nv, nx, nt = args.vars, args.nx, args.nt
    gen = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt)
    gen.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
    q = gen.values
    gen.close()
    path = os.path.join(args.dir, f"dopinf_bench_{nv}x{nx}x{nt}.snp")
    header = api.SnapshotHeader(nv, nx, nt)
    api.write_snapshots(path, header, [q[j * nx:(j + 1) * nx] for j in range(nv)])
    payload = q.nbytes
    del q
    h = api.read_header(path)
    plan = api.partition_rows(nx, 1)
    ref = None
    try:
        from oracle.cpu import Reference

        if Reference.available():
            ref = Reference()
    except Exception:  # noqa: BLE001 - tool
        ref = None

    def timed(fn):
        t0 = time.perf_counter()
        out = fn()
        return time.perf_counter() - t0, out

    for cache in ("warm", "cold"):
        rows = {}
        for name, fn in [
            ("reference_read_block", (lambda: ref.read_block(path, 1, 0)) if ref else None),
            ("b200_block_read", lambda: api.read_block(path, plan, 0, h, ctx).close()),
            ("b200_snapshot_pass_file", lambda: api.snapshot_pass_file(path, plan, 0, h, ctx, True)[0].close()),
        ]:
            if fn is None:
                continue
            best = None
            for _ in range(args.reps):
                if cache == "cold":
                    drop(path)
                else:
                    fn()  # warm the page cache with this very read
                dt, _ = timed(fn)
                best = dt if best is None else min(best, dt)
            rows[name] = best
            print(json.dumps({"cache": cache, "what": name, "seconds": round(best, 4),
                              "gb_s": round(payload / best / 1e9, 2), "payload_gb": round(payload / 1e9, 3),
                              "shape": [nv, nx, nt], "threads": os.cpu_count()}), flush=True)
    os.remove(path)


if __name__ == "__main__":
    main()
