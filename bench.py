#!/usr/bin/env python3
"""bench.py — the dOpInf snapshot pass (Steps II–III + projection) on B200.

Workload (BASELINE.json configs[1], the config the metric is quoted on):
4 state variables × 262,144 points (n = 1,048,576 rows), K = 1,200 fp64
snapshots from the seeded 40-mode damped-oscillator generator (noise 1e-4),
r = 40, rows strong-scaled over N GPUs with the reference's partition_rows.

One step = one pass of the hot path over the resident batch, through the C ABI:
center + global max-abs scales (MAX all-reduce) + scale, upper-triangle DMMA
Gram, cross-rank Gram reduction, D to the host (what the reference eig
consumes), Q̂ = T_rᵀ D and Q̂ to the host. The K×K eigensolve stays on the
reference path and is outside the step (T_r comes from the warm-up's D).

value  = useful FP64 flops per step (n·K·(K+1) Gram + 2·r·K² projection) ×
         steps ÷ device time (CUDA events on the pass's stream, max over ranks).
e2e    = the same through the C ABI from pinned HOST memory: every step
         uploads the raw batch, runs the pass, downloads D and Q̂.
--impl reference: the reference C++ implementation (oracle/_ref, compiled from
         /root/reference) on the box's host cores over a bounded row sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Gram+projection FP64 TFLOP/s & snapshot GB/s at 1/2/4/8 B200 vs roofline"
UNIT = "TFLOP/s"
# FP64 tensor-pipe (DMMA.8x8x4) peak measured on this pool's B200 by
# tools/microbench/fp64_peak.cu (profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json
# carries no FP64 figure and B200_PROFILING.md gives no FP64 fallback.
FP64_PEAK_TFLOPS = 37.1
WORKLOADS = {
    # name: n_vars, nx, nt, r, modes, noise
    "c2": dict(n_vars=4, nx=262144, nt=1200, r=40, modes=40, noise=1e-4, seed=2,
               name="config2: 4 vars x 262144 pts (n=1048576), K=1200, r=40, 40-mode oscillator"),
    "c1": dict(n_vars=2, nx=16384, nt=600, r=10, modes=20, noise=1e-3, seed=1,
               name="config1: 2 vars x 16384 pts (n=32768), K=600, r=10, 20-mode oscillator"),
}
CPU_SAMPLE_NX = 16384  # points per variable in the CPU sample (n_sample = n_vars * this)


def measured_peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:  # noqa: BLE001
        return {}


def ncu_traffic(workload: str):
    """dram read+write bytes per Gram launch from the committed ncu capture, if any."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        return json.loads(p.read_text())["gram"][workload]["dram_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        return None


# ---- clocks during the timed region ---------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait(timeout=5)
        self.file.flush()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in Path(self.file.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.file.name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---- CPU side (the reference, or the oracle port) ------------------------------------------------------
def numpy_oscillator(n_vars, nx, nt, modes, noise, seed, dt=1e-3):
    """Same generator family as the device one (same shapes and distributions;
    x ~ U[0,1), θ,φ ~ U[0,2π), ω ~ U[1,50), γ ~ U[0,0.5)) from numpy's PCG64."""
    rng = np.random.default_rng(seed)
    x = rng.random(nx)
    t = np.arange(nt) * dt
    j = np.arange(1, modes + 1)
    q = np.empty((n_vars * nx, nt))
    for v in range(n_vars):
        theta, phi = rng.uniform(0, 2 * np.pi, modes), rng.uniform(0, 2 * np.pi, modes)
        omega, gamma = rng.uniform(1, 50, modes), rng.uniform(0, 0.5, modes)
        a = np.sin(np.pi * np.outer(x, j) + theta)
        b = np.exp(-np.outer(gamma, t)) * np.cos(np.outer(omega, t) + phi[:, None])
        q[v * nx:(v + 1) * nx] = a @ b + noise * rng.standard_normal((nx, nt))
    return q


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def sample_rows(wl, nx_s):
    """The CPU sample: the first nx_s points of every variable of the workload,
    made by the same device generator as the GPU arm's batch (identical bytes:
    the generator is a pure function of seed, variable and global point), or,
    without a GPU, the numpy generator of the same family. Generation is
    outside every timed region. Returns (q, source)."""
    try:
        import torch

        if torch.cuda.is_available():
            from paper_2504_14338_b200 import api

            with api.DeviceContext(0) as ctx:
                blk = api.LocalBlock(ctx, wl["n_vars"], api.RowRange(0, nx_s), wl["nt"])
                blk.synth_oscillator(seed=wl["seed"], n_modes=wl["modes"], dt=1e-3, noise=wl["noise"])
                q = blk.values
                blk.close()
            return q, "the GPU arm's own bytes (device generator, first points of each variable)"
    except Exception:  # noqa: BLE001 - no GPU / no extension: same family from numpy
        pass
    return (numpy_oscillator(wl["n_vars"], nx_s, wl["nt"], wl["modes"], wl["noise"], wl["seed"]),
            "numpy generator of the same family (no GPU for the device generator)")


def cpu_pass(wl, steps, warmup, cores):
    """Time the reference's Steps II–III + project on a bounded row sample.
    Returns (tflops_per_s, seconds_per_step, kind, cores, sample_desc)."""
    from oracle.cpu import Oracle, Reference

    nv, nt, r = wl["n_vars"], wl["nt"], wl["r"]
    nx_s = min(CPU_SAMPLE_NX, wl["nx"])
    q, source = sample_rows(wl, nx_s)
    n_s = nv * nx_s
    flops = n_s * nt * (nt + 1) + 2 * r * nt * nt
    times = []
    if Reference.available():
        ref = Reference()
        kind, used = "reference", cores
        _, _, _, d, _ = ref.snapshot_pass(q, nv, nx_s, cores, True)
        _, tr = ref.eig_reduced_map(d, r)
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            _, _, _, d, secs = ref.snapshot_pass(q, nv, nx_s, cores, True)
            t1 = time.perf_counter()
            ref.project(tr, d)
            t2 = time.perf_counter()
            if i >= warmup:
                times.append(float(secs[0] + secs[1]) + (t2 - t1))
        sample = (f"{nv} vars x {nx_s} pts (n={n_s} of {nv * wl['nx']} rows), K={nt}, r={r}, bytes: {source}; "
                  f"reference center/compute_global_scales/scale_in_place + global_gram(local_gram) on {cores} "
                  f"in-process ranks (barrier-fenced stage times) + pod::project; OPENBLAS_NUM_THREADS=1; "
                  f"CPU {cpu_model()}; the rate is the sample's, extrapolated to the full batch (the work is "
                  f"linear in n at fixed K)")
    else:
        o = Oracle()
        kind, used = "port", 1
        nx_s = min(nx_s, 2048)  # one scalar thread: keep the sample to ~10-30 s
        q, source = sample_rows(wl, nx_s)
        n_s = nv * nx_s
        flops = n_s * nt * (nt + 1) + 2 * r * nt * nt
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            qc, _ = o.center(q)
            s, _ = o.reduce_scales(o.local_maxabs(qc, nv, nx_s)[None, :])
            d = o.gram(o.scale(qc, nv, nx_s, s))
            if i == 0:
                lam, vec = np.linalg.eigh(d)
                tr = vec[:, ::-1][:, :r] / np.sqrt(np.maximum(lam[::-1][:r], 1e-300))
            o.project(tr, d)
            if i >= warmup:
                times.append(time.perf_counter() - t0)
        sample = (f"{nv} vars x {nx_s} pts (n={n_s}), K={nt}, r={r}, bytes: {source}; C oracle port, 1 thread; "
                  f"CPU {cpu_model()}; rate extrapolated to the full batch (linear in n)")
    per_step = statistics.median(times)
    return flops / per_step / 1e12, per_step, kind, used, sample


def run_reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    value, per_step, kind, used, sample = cpu_pass(wl, args.steps, args.warmup, cores)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(per_step * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded damped-oscillator generator)",
        "config": {"workload": wl["name"], "sample_rows": wl["n_vars"] * min(CPU_SAMPLE_NX, wl["nx"]),
                   "rows_total": wl["n_vars"] * wl["nx"], "extrapolated": "rate of the row sample (linear in n)",
                   "cpu_model": cpu_model(), "parallelism": f"{used} host threads (in-process ranks)"},
        "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": used, "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm --------------------------------------------------------------------------------------------------
def tr_from(d, r):
    """T_r = U_r Λ_r^{-1/2} from a host eig (the reference path's job; any solver
    serves for timing the pass)."""
    lam, vec = np.linalg.eigh(d)
    lam, vec = lam[::-1][:r], vec[:, ::-1][:, :r]
    return np.ascontiguousarray(vec / np.sqrt(np.maximum(lam, 1e-300)))


def run_ours(args, wl):
    import torch

    from paper_2504_14338_b200 import api
    from paper_2504_14338_b200.distributed import (barrier, env_ranks, init_control_plane, max_over_ranks,
                                                   share_unique_id)

    rank, world, local = env_ranks()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    init_control_plane("gloo")
    uid = share_unique_id(rank) if world > 1 else None
    ctx = api.DeviceContext(local, rank, world, uid)
    torch.cuda.set_device(local)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    nv, nx, nt, r = wl["n_vars"], wl["nx"], wl["nt"], wl["r"]
    plan = api.partition_rows(nx, world)
    rr = plan[rank]
    block = api.LocalBlock(ctx, nv, rr, nt)
    block.synth_oscillator(seed=wl["seed"], n_modes=wl["modes"], dt=1e-3, noise=wl["noise"])
    n_total, n_local = nv * nx, nv * rr.count()
    flops_step = n_total * nt * (nt + 1) + 2 * r * nt * nt
    gram_flops_local = n_local * nt * (nt + 1)

    # Host results land in pinned buffers (D is what the reference eig reads).
    def pinned(*shape):
        return torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()

    outs = {"d": pinned(nt, nt), "means": pinned(n_local), "scales": pinned(nv)}
    qhat_out = pinned(r, nt)

    # warm-up (W steps); T_r from the first D (eig on the host: reference path)
    tr = None
    for _ in range(max(args.warmup, 1)):
        _, d = api.snapshot_pass(block, scaling=True, out=outs)
        if tr is None:
            tr = tr_from(d, r)
        api.project_resident(ctx, tr, out=qhat_out)

    barrier()
    torch.cuda.synchronize(local)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = api.kernel_launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gram_ms, stats_ms, apply_ms = [], [], []
    ev0.record(stream)
    for _ in range(args.steps):
        api.snapshot_pass(block, scaling=True, out=outs)
        gram_ms.append(ctx.stage_ms("gram"))
        stats_ms.append(ctx.stage_ms("stats"))
        apply_ms.append(ctx.stage_ms("apply"))
        api.project_resident(ctx, tr, out=qhat_out)
    ev1.record(stream)
    torch.cuda.synchronize(local)
    launches = api.kernel_launches() - launches0
    clk = clocks.stop()
    elapsed_ms = max_over_ranks(ev0.elapsed_time(ev1))
    barrier()

    value = flops_step * args.steps / (elapsed_ms * 1e-3) / 1e12
    ms_step = elapsed_ms / args.steps
    g_avg = statistics.mean(gram_ms)
    achieved = gram_flops_local / (g_avg * 1e-3) / 1e12
    t_avg = statistics.mean(stats_ms) + statistics.mean(apply_ms)
    hbm_peak = measured_peaks().get("hbm_gbs", 6447.5)
    transform_gbs = 24 * n_local * nt / (t_avg * 1e-3) / 1e9

    # ---- e2e: the same step from pinned HOST memory through the C ABI -----------------------------------------
    e2e = None
    if not args.no_e2e:
        block.synth_oscillator(seed=wl["seed"], n_modes=wl["modes"], dt=1e-3, noise=wl["noise"])
        host = torch.empty((n_local, nt), dtype=torch.float64, pin_memory=True)
        hv = host.numpy()
        from paper_2504_14338_b200 import _lib

        rc = _lib.load().dopinf_b200_block_download(block._h, _lib.dptr(hv), nt)
        assert rc == 0
        # W untimed warm-up steps here too: the first pass over a fresh pinned
        # buffer pays the IOMMU/page-table first touch (~80 ms at 10 GB)
        for _ in range(max(args.warmup, 1)):
            api.snapshot_pass_host(block, host.data_ptr(), scaling=True, out=outs, host_ld=nt)
            api.project_resident(ctx, tr, out=qhat_out)
        barrier()
        torch.cuda.synchronize(local)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            api.snapshot_pass_host(block, host.data_ptr(), scaling=True, out=outs, host_ld=nt)
            api.project_resident(ctx, tr, out=qhat_out)
        e1.record(stream)
        torch.cuda.synchronize(local)
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        e2e = {"value": round(flops_step * args.steps / (e2e_ms * 1e-3) / 1e12, 6), "unit": UNIT,
               "h2d_bytes_per_step": int(8 * n_total * nt + 8 * nt * r),
               "d2h_bytes_per_step": int(world * (8 * nt * nt + 8 * r * nt + 8 * n_local + 8 * nv)),
               "ms_per_step": round(e2e_ms / args.steps, 3),
               "path": "pinned host -> dopinf_b200_snapshot_pass_host (chunked H2D overlapped with "
                       "transform + Gram) -> dopinf_b200_project (D and Q̂ back to pinned host)"}
        del host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        value_c, per_step_c, kind, used, sample = cpu_pass(wl, steps=1, warmup=0, cores=os.cpu_count() or 1)
        cpu = {"value": round(value_c, 6), "unit": UNIT, "cores": used, "kind": kind, "sample": sample,
               "ms_per_step_sample": round(per_step_c * 1e3, 1)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded damped-oscillator generator on the device (BASELINE config 2)",
            "config": {"workload": wl["name"], "rows_total": n_total, "snapshots": nt, "r": r,
                       "parallelism": f"row-sharded x{world} (partition_rows), NCCL Gram reduction",
                       "l2": f"inputs larger than L2 ({8 * n_local * nt / 1e9:.1f} GB per GPU)",
                       "step": "center+scales(MAX)+scale, DMMA upper-triangle Gram, Gram reduction, D->host, "
                               "Q̂=T_rᵀD, Q̂->host; eig outside (reference path)"},
            "snapshot_gbs": round(8 * n_total * nt * args.steps / (elapsed_ms * 1e-3) / 1e9, 2),
            "roofline": {"bound": "tensor", "kernel": "gram_dmma_kernel", "achieved": round(achieved, 3),
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                         "traffic": ncu_traffic("c2" if nt == 1200 else "c1"),
                         "algorithmic": f"n_i*K*(K+1) = {gram_flops_local:.4g} flop per launch",
                         "peak_source": "measured DMMA.8x8x4 loop, tools/microbench/fp64_peak.cu "
                                        "(profiles/r01_fp64_peak.txt); no FP64 entry in MEASURED_PEAKS.json",
                         "avg_launch_ms": round(g_avg, 4)},
            "roofline_transform": {"bound": "hbm", "achieved": round(transform_gbs, 1), "peak": hbm_peak,
                                   "unit": "GB/s", "frac": round(transform_gbs / hbm_peak, 4),
                                   "algorithmic": "24*n_i*K bytes (stats read + apply read/write)",
                                   "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    block.close()
    ctx.close()
    return 0


# ---- config 1: the whole pipeline (Steps I-V) --------------------------------------------------------
def run_pipeline_workload(args):
    """BASELINE config 1 ("full dOpInf pipeline, single rank"): wall time of
    Steps I-V from an SNP1 file through the B200 chain (streamed file pass,
    device eigensolve, projection, device grid search, probes, streamed field
    file) beside the reference's pipeline::run on the same file, plus the
    device dsyevd against the reference's LAPACK dsyev at K = 600 and 1200.
    Prints one JSON line (a secondary workload: the bench metric line is
    config 2's)."""
    import torch

    from paper_2504_14338_b200 import api

    nv, nx, nt, r, nt_p = 2, 16384, 600, 10, 1200
    b1 = b2 = api.logspace(1e-6, 1e2, 8)
    probes = [(0, 0), (0, 5000), (1, 9999), (1, 16383)]
    work = Path(tempfile.mkdtemp(prefix="dopinf_c1_"))
    ctx = api.DeviceContext(0)
    gen = api.LocalBlock(ctx, nv, api.RowRange(0, nx), nt)
    gen.synth_oscillator(seed=1, n_modes=20, dt=1e-3, noise=1e-3)
    raw = gen.values
    gen.close()
    header = api.SnapshotHeader(nv, nx, nt, ["var0", "var1"])
    data = str(work / "c1.snp1")
    api.write_snapshots(data, header, [raw[:nx], raw[nx:]])
    plan = api.partition_rows(nx, 1)
    cfg = api.SearchConfig(b1, b2, 1.2, nt_p)
    pr = [api.Probe(v, i) for v, i in probes]

    def ours():
        t = [time.perf_counter()]
        blk, params, d = api.snapshot_pass_file(data, plan, 0, header, ctx, scaling=True)
        t.append(time.perf_counter())
        api.eig_sym_desc(ctx, vectors=False)
        api.reduced_map(ctx, r, download=False)
        api.project_resident(ctx, None, r=r)
        t.append(time.perf_counter())
        out = api.grid_search(None, cfg, ctx, r=r, nt=nt)
        t.append(time.perf_counter())
        api.reconstruct_probes(blk, None, out.trajectory, pr, params, r=r)
        api.write_field(blk, None, out.trajectory, params, header.var_names, str(work / "field_rank0.snp1"), r=r)
        t.append(time.perf_counter())
        blk.close()
        return np.diff(t), out

    for _ in range(max(args.warmup, 1)):
        ours()
    runs = [ours() for _ in range(args.steps)]
    st = np.median(np.array([x[0] for x in runs]), axis=0)
    pair = runs[-1][1].pair_opt
    line = {"workload": "config1-pipeline: 2 vars x 16384 pts, K=600, r=10, 8x8 (b1, b2) in [1e-6, 1e2], "
                        "nt_p=1200, 4 probes, field file",
            "metric": "dOpInf pipeline wall time, Steps I-V from an SNP1 file", "unit": "s",
            "higher_is_better": False, "steps": args.steps, "warmup": args.warmup,
            "value": round(float(st.sum()), 4),
            "stages_s": {"file+transform+gram (I-III)": round(float(st[0]), 4),
                         "eig+reduced_map+project (III)": round(float(st[1]), 4),
                         "grid_search (IV)": round(float(st[2]), 4),
                         "probes+field file (V)": round(float(st[3]), 4)},
            "chain": "snapshot_pass_file -> eig_sym_desc (cuSOLVER dsyevd) -> reduced_map -> project -> "
                     "grid_search (device) -> reconstruct_probes -> write_field", "pair": list(pair)}
    # the device eigensolve against the reference's dsyev at K = 600 (this D) and 1200 (config 2's)
    eig = {}
    from oracle.cpu import Reference

    have_ref = Reference.available()
    ref = Reference() if have_ref else None
    for K, (nvk, nxk, modes, noise, seed) in ((600, (2, 16384, 20, 1e-3, 1)), (1200, (4, 262144, 40, 1e-4, 2))):
        blk = api.LocalBlock(ctx, nvk, api.RowRange(0, nxk), K)
        blk.synth_oscillator(seed=seed, n_modes=modes, dt=1e-3, noise=noise)
        _, d = api.snapshot_pass(blk, scaling=True)
        blk.close()
        times = []
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            api.eig_sym_desc(ctx, vectors=True)
            times.append(time.perf_counter() - t0)
        eig[f"K={K}"] = {"device_dsyevd_s": round(min(times), 4)}
        if ref is not None:
            t0 = time.perf_counter()
            ref.eig_reduced_map(d, 10)
            eig[f"K={K}"]["reference_dsyev_s"] = round(time.perf_counter() - t0, 4)
    line["eig"] = eig
    if ref is not None:
        for workers in (1, os.cpu_count() or 1):
            t0 = time.perf_counter()
            stages, res = ref.pipeline_run(data, work / f"ref_w{workers}", workers, r, True, b1, b2, 1.2, nt_p, probes)
            line[f"reference_pipeline_run_workers{workers}"] = {
                "wall_s": round(time.perf_counter() - t0, 4),
                "stages_s": dict(zip(["load", "transform", "gram_reduce", "eig_project", "search", "postprocess"],
                                     [round(float(x), 4) for x in stages])),
                "pair": [res[1], res[2]]}
        line["reference_kind"] = "compiled reference (oracle/_ref), OPENBLAS_NUM_THREADS=1 as its CLI"
    ctx.close()
    import shutil

    shutil.rmtree(work, ignore_errors=True)
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS) + ["c1-pipeline"], default="c2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.workload == "c1-pipeline":
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        return run_pipeline_workload(args)
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        return run_reference_arm(args, wl)
    return run_ours(args, wl)


if __name__ == "__main__":
    sys.exit(main())
