"""Shared test helpers: the reference data flow of Steps II-III over p ranks,
restated with the CPU oracle (test infrastructure)."""
import numpy as np


def slices(q, n_vars, nx, plan):
    nt = q.shape[1]
    out = []
    for b, e in plan:
        parts = [q[j * nx + b: j * nx + e] for j in range(n_vars)]
        out.append(np.concatenate(parts).reshape(-1, nt) if parts else np.zeros((0, nt)))
    return out


def oracle_pass(oracle, q, n_vars, nx, p, scaling=True):
    """Steps II-III over p ranks with the oracle, the reference's data flow
    (pipeline.cpp:270-280; MAX and ascending-rank SUM as comm_inprocess.cpp)."""
    plan = oracle.partition_rows(nx, p)
    blocks = slices(q, n_vars, nx, plan)
    cent = [oracle.center(b) for b in blocks]
    scales = None
    if scaling:
        per_rank = np.stack([oracle.local_maxabs(c, n_vars, e - b) for (c, _), (b, e) in zip(cent, plan)])
        scales, bad = oracle.reduce_scales(per_rank)
        assert bad == -1
        cent = [(oracle.scale(c, n_vars, e - b, scales), m) for (c, m), (b, e) in zip(cent, plan)]
    d = oracle.allreduce_sum(np.stack([oracle.gram(c) for c, _ in cent]))
    full = np.empty_like(q)
    means = np.empty(q.shape[0])
    for (c, m), (b, e) in zip(cent, plan):
        nxi = e - b
        for j in range(n_vars):
            full[j * nx + b: j * nx + e] = c[j * nxi:(j + 1) * nxi]
            means[j * nx + b: j * nx + e] = m[j * nxi:(j + 1) * nxi]
    return full, means, scales, d
