"""Generate the golden fixtures in tests/golden from the UNMODIFIED reference.

Run in the build container (needs /root/reference and oracle/_ref):

    python tests/golden/make_golden.py

Inputs come from the product's seeded host generator (bk.synth_chip, pinned in
DESIGN.md §Inputs; a SHA-256 of the input bytes is stored so generator drift is
caught). Every output array is computed by oracle/_ref/libblockoa_ref.so — the
reference core compiled from /root/reference/proj/core/src — through its public
API (assemble, apply_block, block_cg, combine_from_weights, operator_action,
relative_residual). Config 4 (non-uniform dz) is not expressible in the
reference's GridSpec and has no reference golden.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_2510_23221_b200 as bk  # noqa: E402
from oracle.oracle import Reference, build_reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, config, nx, ny, nz, s, N, stored sample indices)
PIPELINE_CASES = [
    ("c1_full", 1, 64, 64, 1, 8, 256, [0, 1, 127, 255]),
    ("c2_reduced", 2, 48, 48, 1, 16, 64, [0, 31, 63]),
    ("c3_reduced", 3, 16, 16, 8, 32, 32, [0, 17, 31]),
    ("c5_reduced", 5, 8, 8, 16, 64, 16, [0, 15]),
]


def input_digest(inp) -> str:
    h = hashlib.sha256()
    for a in (inp.k, inp.q_basis, inp.coef):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def grid_tuple(g):
    return (g.nx, g.ny, g.nz, g.lx, g.ly, g.lz)


def main():
    build_reference()
    ref = Reference()

    # --- SPEC.md:128 known answer: 3x3x3, unit spacing, k=1, Dirichlet 0
    op = ref.assemble((3, 3, 3, 3.0, 3.0, 3.0), np.ones(27), [(0, 0.0, 0.0)] * 6)
    rp, col, val, g, vol = ref.csr(op)
    np.savez(os.path.join(OUT, "kat_3x3x3.npz"), row_ptr=rp, col=col, val=val, g=g, vol=vol)

    # --- mixed boundary operator (all three face kinds) + apply_block
    rng = np.random.default_rng(20251023)
    grid = (7, 5, 4, 7e-3, 5e-3, 0.6e-3)
    k = rng.uniform(1.0, 400.0, 7 * 5 * 4)
    bc = [(0, 50.0, 0.0), (1, 30.0, 20.0), (2, 0.0, 0.0), (0, 10.0, 0.0), (1, 1e2, 25.0),
          (1, 1e4, 25.0)]
    op = ref.assemble(grid, k, bc)
    rp, col, val, g, vol = ref.csr(op)
    xs = {s: rng.standard_normal((140, s)) for s in (1, 4, 7, 16)}
    ys = {s: ref.apply_block(op, xs[s]) for s in xs}
    np.savez(os.path.join(OUT, "mixed_operator.npz"), grid=np.array(grid), k=k,
             bc_kind=np.array([f[0] for f in bc]), bc_a=np.array([f[1] for f in bc]),
             bc_b=np.array([f[2] for f in bc]), row_ptr=rp, col=col, val=val, g=g, vol=vol,
             **{f"x{s}": xs[s] for s in xs}, **{f"y{s}": ys[s] for s in ys})

    # --- pipeline goldens on BASELINE-config inputs
    for name, cfg, nx, ny, nz, s, N, keep in PIPELINE_CASES:
        inp = bk.synth_chip(cfg, nx, ny, nz, s, N)
        op = ref.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
        B = np.stack([ref.rhs_from_power(op, inp.q_basis[:, t]) for t in range(s)], axis=1)
        X, rep = ref.block_cg(op, B, 1e-12, 100000, 1)
        T, Q, R = ref.combine_action(op, X, inp.coef, threads=os.cpu_count() or 1)
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"), config=cfg, shape=np.array([nx, ny, nz, s, N]),
            input_sha256=input_digest(inp), X=X, iterations=rep["iterations"],
            matvec_count=rep["matvec_count"], final_rel_residual=rep["final_rel_residual"],
            converged=rep["converged"], keep=np.array(keep), T=T[keep], Q=Q[keep], resid=R)
        print(f"{name}: n={inp.grid.cell_count()} s={s} N={N} iters={rep['iterations']} "
              f"max resid={R.max():.2e}")


def c2_full_meta(ref):
    """Reference block-CG iteration count on the full BASELINE config-2 chip
    (chip 0): bench.py's reference arm times a capped number of iterations and
    scales by this count."""
    import time

    inp = bk.synth_chip(*bk.CONFIGS[2])
    op = ref.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    B = np.stack([ref.rhs_from_power(op, inp.q_basis[:, t]) for t in range(16)], axis=1)
    t0 = time.perf_counter()
    X, rep = ref.block_cg(op, B, 1e-12, 100000, 1)
    wall = time.perf_counter() - t0
    np.savez(os.path.join(OUT, "c2_full_meta.npz"), input_sha256=input_digest(inp),
             iterations=rep["iterations"], matvec_count=rep["matvec_count"],
             final_rel_residual=rep["final_rel_residual"], converged=rep["converged"],
             solve_wall_s=wall, X_colnorm=np.linalg.norm(X, axis=0),
             X_checksum=np.array([X.sum(), np.abs(X).sum()]))
    print(f"c2_full: iters={rep['iterations']} wall={wall:.1f}s")


if __name__ == "__main__":
    main()
    if "--c2-full" in sys.argv:
        c2_full_meta(Reference())
