"""Summarise ncu outputs into profiles/ (dev tool).

  python tools/ncu_summary.py launches <launches.csv>     per-kernel share of device time
  python tools/ncu_summary.py full <report.ncu-rep>       key metrics per profiled kernel
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_active_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory_throughput_%"),
    ("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "registers"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem_ld_bank_conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem_ld_wavefronts"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[i]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot = {}
    for r in rows[i + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        tot.setdefault(name, []).append(float(r[vi].replace(",", "")))
    allt = sum(sum(v) for v in tot.values())
    out = [f"{'kernel':34s} {'launches':>8s} {'total_ms':>10s} {'avg_ms':>9s} {'share':>6s}"]
    for name, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
        out.append(f"{name:34s} {len(v):8d} {sum(v) / 1e6:10.3f} {sum(v) / len(v) / 1e6:9.4f} {sum(v) / allt:6.3f}")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    idx = {k: i for i, k in enumerate(h)}
    out = []
    for d in data:
        out.append("---- " + d[idx["Kernel Name"]][:110])
        for key, label in KEYS:
            if key in idx:
                out.append(f"  {label:26s} {d[idx[key]]:>16s} {units[idx[key]]}")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
