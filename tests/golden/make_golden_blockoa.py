"""Golden fixture for the reference-semantics generator,
generated from the UNMODIFIED reference build (oracle/_ref) in this container:

  chip_default.npz — configs/default.json (default_run_config, run_config.cpp:273-291):
    field_digest of every floorplan group's k field and basis power map
    (build_floorplans / rasterize_*, chip.cpp:180-306), the first 4 samples'
    normalised weights (draw_weights, pipeline.cpp:136-152), and the full
    generate_blockoa result summarised: block-CG iterations, floorplan ids,
    residuals, per-sample L2 norms of u and q, and u / q of samples 0, 1, 499.

Run: python tests/golden/make_golden_blockoa.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference, build_reference  # noqa: E402


def main():
    build_reference()
    ref = Reference()
    grid, n_data, n_basis, n_k, seed = (24, 24, 12), 500, 50, 5, 1
    eta = n_basis // n_k
    bc = [(0, 50.0, 0.0)] * 4 + [(1, 3e4, 50.0)] * 2
    k, q = ref.chip_fields(grid, n_k, eta, seed)
    kd = np.array([ref.field_digest(grid, f) for f in k], np.uint64)
    qd = np.array([ref.field_digest(grid, f) for f in q], np.uint64)
    w = ref.draw_weights(n_basis, seed, 4)
    d = ref.generate_blockoa(grid, n_data, n_basis, n_k, seed, bc, ("uniform", -0.01, 0.01), 1e-9,
                             50000)
    keep = np.array([0, 1, 499])
    np.savez_compressed(
        os.path.join(HERE, "chip_default.npz"), grid=np.array(grid), n_data=n_data,
        n_basis=n_basis, n_k=n_k, seed=seed, k_digest=kd, q_digest=qd, weights=w,
        iterations=d["iterations"], floorplan_id=d["floorplan_id"], residual=d["residual"],
        u_norm=np.linalg.norm(d["u"], axis=1), q_norm=np.linalg.norm(d["q"], axis=1), keep=keep,
        u=d["u"][keep], q=d["q"][keep])


if __name__ == "__main__":
    main()
