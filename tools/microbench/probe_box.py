"""Probe the GPU box: host cores, GPU, cuBLAS FP64 DGEMM/DSYRK-class throughput via torch.

Plumbing only: sets the FP64 denominator next to tools/microbench/fp64_peak.cu.
"""
import os
import subprocess
import time

import torch


def main():
    print("nproc", os.cpu_count())
    try:
        print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:800])
    except Exception as e:  # noqa: BLE001
        print("lscpu failed", e)
    print(subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout)
    dev = torch.device("cuda:0")
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(2):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(5):
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"cuBLAS DGEMM n={n}: {best:.3f} ms {2*n**3/(best*1e-3)/1e12:.2f} TFLOP/s")
    # Gram-shaped: Q^T Q with tall Q (cuBLAS DGEMM on the TN shape)
    for (rows, k) in ((1048576, 1200), (4194304, 512)):
        q = torch.randn(rows, k, dtype=torch.float64, device=dev)
        for _ in range(2):
            q.t() @ q
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            e0.record()
            q.t() @ q
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"cuBLAS QtQ rows={rows} K={k}: {best:.3f} ms executed {2*rows*k*k/(best*1e-3)/1e12:.2f} TFLOP/s"
              f" useful(nK(K+1)) {rows*k*(k+1)/(best*1e-3)/1e12:.2f}")
        del q
        torch.cuda.empty_cache()
    # host<->device copy rates (pinned)
    h = torch.empty(1 << 28, dtype=torch.float64).pin_memory()
    d = torch.empty(1 << 28, dtype=torch.float64, device=dev)
    for _ in range(2):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"H2D pinned {h.numel()*8/(t1-t0)/1e9:.1f} GB/s  D2H pinned {h.numel()*8/(t2-t1)/1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
