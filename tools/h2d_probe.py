import torch, time
n = 1 << 30
h = torch.empty(n // 8, dtype=torch.float64).pin_memory()
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
for chunk_mb in (64, 256, 1024):
    c = chunk_mb << 20
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record()
        for rep in range(4):
            for off in range(0, n, c):
                d.view(torch.uint8)[off:off+c].copy_(h.view(torch.uint8)[off:off+c], non_blocking=True)
        e1.record()
    torch.cuda.synchronize()
    print(f"H2D chunk {chunk_mb} MB: {4*n/ (e0.elapsed_time(e1)*1e-3)/1e9:.1f} GB/s")
# two streams concurrently
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0=time.perf_counter()
half = n // 2
for rep in range(4):
    with torch.cuda.stream(s1):
        d.view(torch.uint8)[:half].copy_(h.view(torch.uint8)[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        d.view(torch.uint8)[half:].copy_(h.view(torch.uint8)[half:], non_blocking=True)
torch.cuda.synchronize(); print(f"H2D 2 streams: {4*n/(time.perf_counter()-t0)/1e9:.1f} GB/s")
# 2-D copies as the streamed pass issues them: 32768 rows x 9600 B (K = 1200), equal pitches
import ctypes
cudart = ctypes.CDLL("libcudart.so.12") if False else None
rows, width = 32768, 9600
nbytes = rows * width
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
hv = h.view(torch.uint8)[: 3 * nbytes].view(3 * rows, width)
dv = d.view(torch.uint8)[: 3 * nbytes].view(3 * rows, width)
with torch.cuda.stream(s):
    e0.record()
    for rep in range(4):
        for k in range(3):
            dv[k * rows:(k + 1) * rows].copy_(hv[k * rows:(k + 1) * rows], non_blocking=True)
    e1.record()
torch.cuda.synchronize()
print(f"H2D 315 MB row blocks (torch, contiguous): {12 * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
