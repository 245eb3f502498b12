"""Device-timed sweep over the BASELINE.json configs on one B200 (dev tool; the
bench line itself is bench.py on config 2). Prints one JSON object per line
and writes them to gpurun_out/config_sweep.jsonl.

  c1   2 vars x 16384, K=600: snapshot pass (stage times)
  c3   1 var x 4194304, K in {256..4096}, N(0,1) + 10 x rank-50: Gram TFLOP/s per K
  c5   config-2 data, r in {20,40,80}: Phi_r = Q T_r and 1000 probe rows (basis_rows)
  c5f  config-2 data, r in {20,40,80}: field reconstruction (nt_p = 2400) + SNP1 field writer
  c4   8 vars x 4194304 per GPU, K=1500 (403 GB): streamed from a device ring
"""
import argparse
import os
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2504_14338_b200 import api  # noqa: E402

PEAK_FP64 = 37.1  # measured DMMA.8x8x4 peak (profiles/r01_fp64_peak.txt)
try:  # driver-written HBM copy bandwidth of this pool's B200s
    PEAK_HBM = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
except Exception:  # noqa: BLE001
    PEAK_HBM = 6551.4


def stages(ctx, names):
    return {n: round(ctx.stage_ms(n), 4) for n in names}


def emit(rec, out):
    line = json.dumps(rec)
    print(line, flush=True)
    out.write(line + "\n")


def tr_from(d, r):
    lam, vec = np.linalg.eigh(d)
    lam, vec = lam[::-1][:r], vec[:, ::-1][:, :r]
    return np.ascontiguousarray(vec / np.sqrt(np.maximum(lam, 1e-300)))


def run_c1(ctx, out):
    b = api.LocalBlock(ctx, 2, api.RowRange(0, 16384), 600)
    b.synth_oscillator(seed=1, n_modes=20, dt=1e-3, noise=1e-3)
    for rep in range(3):
        api.snapshot_pass(b, scaling=True)
    st = stages(ctx, ["stats", "apply", "gram", "gram_reduce", "unpack"])
    n, K = 32768, 600
    emit({"config": "c1", "n": n, "K": K, "stage_ms": st,
          "gram_tflops": round(n * K * (K + 1) / st["gram"] / 1e9, 3),
          "transform_gbs": round(24 * n * K / (st["stats"] + st["apply"]) / 1e6, 1)}, out)
    b.close()


def run_c3(ctx, out, ks):
    n = 4194304
    for K in ks:
        b = api.LocalBlock(ctx, 1, api.RowRange(0, n), K)
        b.synth_lowrank(seed=3, rank=50, amplitude=10.0)
        g = []
        for rep in range(3):
            api.snapshot_pass(b, scaling=True)
            g.append(ctx.stage_ms("gram"))
        best = min(g)
        st = stages(ctx, ["stats", "apply", "gram_reduce", "unpack"])
        emit({"config": "c3", "n": n, "K": K, "gram_ms": round(best, 3),
              "gram_tflops_useful": round(n * K * (K + 1) / best / 1e9, 3),
              "frac_of_dmma_peak": round(n * K * (K + 1) / best / 1e9 / PEAK_FP64, 4),
              "snapshot_gbs": round(8 * n * K / best / 1e6, 1), "other_stage_ms": st}, out)
        b.close()


def run_c5(ctx, out, rs, n_probes=1000):
    nv, nx, K = 4, 262144, 1200
    b = api.LocalBlock(ctx, nv, api.RowRange(0, nx), K)
    b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
    params, d = api.snapshot_pass(b, scaling=True)
    n = nv * nx
    rng = np.random.default_rng(5)
    probes = np.sort(rng.choice(n, size=n_probes, replace=False))
    for r in rs:
        tr = tr_from(d, r)
        ts = []
        for rep in range(3):
            api.basis(b, tr, download=False)
            ts.append(ctx.stage_ms("basis"))
        best = min(ts)
        flops = 2 * n * K * r
        byts = 8 * n * (K + r) + 8 * K * r
        t0 = time.perf_counter()
        rows = api.basis_rows(b, tr, probes)
        t_probe = time.perf_counter() - t0
        # the probes' series over the 2K horizon from a ROM trajectory (reconstruct_probes)
        qt = np.random.default_rng(r).standard_normal((2 * K, r)) * 1e-2
        plist = [api.Probe(int(p) // nx, int(p) % nx) for p in probes]
        t0 = time.perf_counter()
        series = api.reconstruct_probes(b, tr, qt, plist, params)
        t_series = time.perf_counter() - t0
        emit({"config": "c5", "n": n, "K": K, "r": r, "basis_ms": round(best, 3),
              "tflops": round(flops / best / 1e9, 3), "gbs": round(byts / best / 1e6, 1),
              "frac_fp64": round(flops / best / 1e9 / PEAK_FP64, 4), "frac_hbm": round(byts / best / 1e6 / PEAK_HBM, 4),
              "roofline_ms": round(max(flops / PEAK_FP64 / 1e9, byts / PEAK_HBM / 1e6), 3),
              "probe_rows": n_probes, "probe_basis_rows_wall_ms": round(t_probe * 1e3, 3),
              "probe_rows_shape": list(rows.shape), "probe_series_nt_p": 2 * K,
              "reconstruct_probes_wall_ms": round(t_series * 1e3, 3), "probe_series": len(series)}, out)
    b.close()


def run_c5_field(ctx, out, rs, nt_p=2400, write_dir="/tmp"):
    """Step V at config 5: field = s·(Q·T_r)·Q̃ᵀ + mean over all 1,048,576 rows and
    nt_p = 2K = 2400 (20 GB of output), device-resident; then the streamed SNP1
    field writer at r = 40, and the reference's reconstruct_field on a row sample."""
    nv, nx, K = 4, 262144, 1200
    b = api.LocalBlock(ctx, nv, api.RowRange(0, nx), K)
    b.synth_oscillator(seed=2, n_modes=40, dt=1e-3, noise=1e-4)
    params, d = api.snapshot_pass(b, scaling=True)
    n = nv * nx
    rng = np.random.default_rng(6)
    for r in rs:
        tr = tr_from(d, r)
        qt = rng.standard_normal((nt_p, r))
        ts = []
        for rep in range(3):
            api.reconstruct_field(b, tr, qt, params, download=False)
            ts.append(ctx.stage_ms("field"))
        best = min(ts)
        flops = 2 * n * nt_p * r
        byts = 8 * n * nt_p + 8 * n * r
        rec = {"config": "c5_field", "n": n, "K": K, "r": r, "nt_p": nt_p, "field_ms": round(best, 3),
               "basis_ms": round(ctx.stage_ms("basis"), 3), "tflops": round(flops / best / 1e9, 3),
               "write_gbs": round(8 * n * nt_p / best / 1e6, 1),
               "frac_fp64": round(flops / best / 1e9 / PEAK_FP64, 4),
               "frac_hbm": round(byts / best / 1e6 / PEAK_HBM, 4),
               "roofline_ms": round(max(flops / PEAK_FP64 / 1e9, byts / PEAK_HBM / 1e6), 3)}
        if r == 40:
            path = os.path.join(write_dir, "dopinf_field_rank0.snp1")
            t0 = time.perf_counter()
            api.write_field(b, tr, qt, params, [f"var{j}" for j in range(nv)], path)
            wall = time.perf_counter() - t0
            rec["write_field_wall_s"] = round(wall, 3)
            rec["write_field_gbs"] = round(8 * n * nt_p / wall / 1e9, 2)
            os.remove(path)
            try:
                from oracle.cpu import Reference

                if Reference.available():
                    sample = 8192
                    q = b.values[:sample]
                    t0 = time.perf_counter()
                    Reference().reconstruct_field(q, 1, tr, qt, params.local_means[:sample], params.scales[:1], True)
                    rs_ = time.perf_counter() - t0
                    rec["reference_sample_rows"] = sample
                    rec["reference_s_per_row"] = rs_ / sample
                    rec["reference_extrapolated_s"] = round(rs_ / sample * n, 1)
            except Exception as e:  # noqa: BLE001 - dev tool
                rec["reference_error"] = str(e)
        emit(rec, out)
    b.close()


def run_c4(ctx, out, r=68):
    """Config 4 per GPU: 8 vars x 4,194,304 points (33.5M rows), K = 1500, 60-mode
    oscillator with per-variable magnitudes 1e-2..1e5, scaling on, r = 68 —
    403 GB, streamed through a device ring (generated chunk by chunk)."""
    nv, nx, K = 8, 4194304, 1500
    amps = 10.0 ** np.linspace(-2, 5, nv)
    t0 = time.perf_counter()
    params, d = api.stream_pass_synth(ctx, nv, api.RowRange(0, nx), K, seed=4, n_modes=60, dt=1e-3, noise=1e-4,
                                      amps=amps, scaling=True)
    wall = time.perf_counter() - t0
    total = ctx.stage_ms("stream")
    gram = ctx.stage_ms("stream_gram")
    tr = tr_from(d, r)
    qhat = api.project_resident(ctx, tr)
    n = nv * nx
    emit({"config": "c4", "n_per_gpu": n, "K": K, "r": r, "bytes_per_gpu": 8 * n * K,
          "stream_total_ms": round(total, 1), "gram_ms_sum": round(gram, 1),
          "gram_tflops_useful": round(n * K * (K + 1) / gram / 1e9, 3),
          "pass_tflops_incl_generation": round(n * K * (K + 1) / total / 1e9, 3),
          "project_ms": round(ctx.stage_ms("project"), 3), "wall_s": round(wall, 2),
          "scales": [float(x) for x in params.scales], "qhat_shape": list(qhat.shape)}, out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c3,c5")
    ap.add_argument("--ks", default="256,512,1024,2048,4096")
    args = ap.parse_args()
    Path(ROOT / "gpurun_out").mkdir(exist_ok=True)
    with api.DeviceContext(0) as ctx, open(ROOT / "gpurun_out" / "config_sweep.jsonl", "w") as out:
        cfgs = args.configs.split(",")
        if "c1" in cfgs:
            run_c1(ctx, out)
        if "c3" in cfgs:
            run_c3(ctx, out, [int(k) for k in args.ks.split(",")])
        if "c5" in cfgs:
            run_c5(ctx, out, [20, 40, 80])
        if "c5f" in cfgs:
            run_c5_field(ctx, out, [20, 40, 80])
        if "c4" in cfgs:
            run_c4(ctx, out)


if __name__ == "__main__":
    main()
