"""Generate tests/golden/reference_vectors.npz from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref, i.e. /root/reference at build
time):  python tests/golden/make_golden.py

Inputs are the reference's own seeded streams (synth::Rng, synth.cpp:15-34)
for the shapes its tests use — not stored: tests regenerate them with the
oracle's restated Rng, which tests/test_oracle_pins.py pins bit-for-bit to the
reference's — and outputs are what the reference's functions return on them
(oracle/ref_bench.cpp calls the reference API unchanged):

  transform_*   test_transform.cpp:52-150 shapes, Steps II on p in {1,2,3}
  gram_*        test_linalg.cpp:40-62 / test_pod.cpp:30-56 shapes, p in {1,2,4}
  sweep_*       acceptance.cpp:202-236 20-shape sweep (seeds 1000+i): D (p=1
                and p=7), eigenvalues and T_r from eig_sym_desc/reduced_map,
                Q̂ = project(T_r, D), Φ_r rows (basis_rows)
  pipeline_*    a small oscillator dataset through Steps II-IV (grid search)
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.cpu import Reference  # noqa: E402

SWEEP = [(500, 50, 0), (350, 40, 0), (500, 13, 0), (120, 30, 0), (64, 24, 0), (57, 23, 0), (200, 50, 0),
         (480, 36, 0), (33, 20, 0), (100, 12, 0), (450, 48, 0), (77, 31, 0), (500, 50, 5), (300, 30, 3),
         (120, 40, 10), (64, 16, 1), (500, 24, 8), (90, 45, 12), (250, 50, 2), (48, 12, 4)]


def rng_matrix(ref, seed, rows, cols, skip=0):
    """Rows × cols normals from Rng(seed) after `skip` draws (helpers.hpp:14-18)."""
    v = ref.normals(seed, skip + rows * cols)[skip:]
    return v.reshape(rows, cols)


def main():
    ref = Reference()
    assert ref.backend() == "avx2", ref.backend()
    out = {}

    # Step II on the reference's test shapes (var count, nx, nt, seed).
    for tag, (nv, nx, nt, seed) in {"t12": (1, 20, 7, 12), "t8": (2, 15, 11, 8), "t21": (2, 12, 9, 21),
                                    "t77": (3, 40, 33, 77)}.items():
        q = rng_matrix(ref, seed, nv * nx, nt)
        for p in (1, 2, 3):
            if p > nx:
                continue
            qt, means, scales, d, _ = ref.snapshot_pass(q, nv, nx, p, True)
            out[f"transform_{tag}_p{p}_q"] = qt
            out[f"transform_{tag}_p{p}_means"] = means
            out[f"transform_{tag}_p{p}_scales"] = scales
            out[f"transform_{tag}_p{p}_gram"] = d
        qc, mc = ref.center(q)
        out[f"transform_{tag}_centered"] = qc
        out[f"transform_{tag}_center_means"] = mc
    out["transform_meta"] = np.array([[1, 20, 7, 12], [2, 15, 11, 8], [2, 12, 9, 21], [3, 40, 33, 77]])

    # Gram on test_pod / test_linalg shapes.
    for tag, (m, k, seed) in {"g41": (20, 6, 41), "g5": (13, 7, 5), "g73": (30, 8, 73), "g6": (26, 20, 6)}.items():
        q = rng_matrix(ref, seed, m, k)
        for p in (1, 2, 4):
            out[f"gram_{tag}_p{p}"] = ref.global_gram(q, p)

    # acceptance.cpp sweep.
    for i, (m, nt, rk) in enumerate(SWEEP):
        seed = 1000 + i
        if rk == 0:
            q = rng_matrix(ref, seed, m, nt)
        else:
            allv = ref.normals(seed, m * rk + rk * nt)
            q = ref.matmul(allv[: m * rk].reshape(m, rk), allv[m * rk:].reshape(rk, nt))
        d1 = ref.global_gram(q, 1)
        d7 = ref.global_gram(q, 7)
        # numerical rank from the singular values of q (acceptance.cpp:218-222 uses thin_svd);
        # the Gram's round-off eigenvalues (~1e-16 λ1) would over-count it.
        sigma = np.linalg.svd(q, compute_uv=False)
        numerical_rank = int(np.sum(sigma > 1e-8 * sigma[0]))
        r = min(max(numerical_rank, 1), 10)
        lam, tr = ref.eig_reduced_map(d1, r)
        out[f"sweep_{i}_gram_p1"] = d1
        out[f"sweep_{i}_gram_p7"] = d7
        out[f"sweep_{i}_lambda"] = lam
        out[f"sweep_{i}_tr"] = tr
        out[f"sweep_{i}_qhat"] = ref.project(tr, d1)
        sel = np.arange(0, m, max(1, m // 9), dtype=np.uintp)
        out[f"sweep_{i}_basis_sel"] = sel.astype(np.int64)
        out[f"sweep_{i}_basis_rows"] = ref.basis_rows(q, tr, sel)
    out["sweep_meta"] = np.array(SWEEP)

    # Steps II-IV on a small seeded dataset (Q̂ → grid search → ROM trajectory).
    nv, nx, nt, r = 2, 64, 40, 4
    q = rng_matrix(ref, 4242, nv * nx, nt) * 1e-2
    tgrid = np.arange(nt) * 0.05
    for v in range(nv):
        for mode in range(3):
            q[v * nx:(v + 1) * nx] += np.outer(np.sin((mode + 1) * np.pi * np.linspace(0, 1, nx) + v),
                                               np.exp(-0.1 * (mode + 1) * tgrid) *
                                               np.cos((mode + 2) * tgrid + mode))
    qt, means, scales, d, _ = ref.snapshot_pass(q, nv, nx, 1, True)
    lam, tr = ref.eig_reduced_map(d, r)
    qhat = ref.project(tr, d)
    b1 = np.logspace(-6, 2, 4)
    b2 = np.logspace(-6, 2, 4)
    traj, pair, err = ref.grid_search(qhat, b1, b2, 1.2, 2 * nt)
    out.update({"pipeline_input": q, "pipeline_q": qt, "pipeline_gram": d, "pipeline_lambda": lam,
                "pipeline_tr": tr, "pipeline_qhat": qhat, "pipeline_traj": traj,
                "pipeline_pair_err": np.array([pair[0], pair[1], err]), "pipeline_meta": np.array([nv, nx, nt, r])})

    path = Path(__file__).with_name("reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size / 1e6:.2f} MB, {len(out)} arrays)")


if __name__ == "__main__":
    main()
