import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from pathlib import Path
from oracle.cpu import Oracle
from paper_2504_14338_b200 import api
G = np.load('/root/repo/tests/golden/reference_vectors.npz')
o = Oracle()
ctx = api.DeviceContext(0)
for i in range(20):
    m, nt, rk = (int(v) for v in G["sweep_meta"][i])
    rng = o.rng(1000 + i)
    q = rng.matrix(m, nt) if rk == 0 else o.matmul(rng.matrix(m, rk), rng.matrix(rk, nt))
    tr = G[f"sweep_{i}_tr"]
    b = api.LocalBlock(ctx, 1, api.RowRange(0, m), nt, values=q)
    phi = api.basis(b, tr)
    ref = o.matmul(q, tr)
    err = np.linalg.norm(phi - ref) / np.linalg.norm(ref)
    colerr = np.linalg.norm(phi - ref, axis=0) / np.linalg.norm(ref, axis=0)
    print(i, m, nt, rk, tr.shape[1], f"{err:.2e}", f"max col {colerr.max():.2e}", f"|tr| {np.abs(tr).max():.2e}", f"|phi| {np.abs(ref).max():.2e}")
