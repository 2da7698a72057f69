"""Full-size golden fixtures for BASELINE configs 3, 4 and 5.

TEST INFRASTRUCTURE. Run in the build container (needs oracle/_ref, i.e.
/root/reference at build time); every array is computed by the UNMODIFIED
reference core (oracle/_ref/libblockoa_ref.so) through its public API, except
config 4, whose per-layer dz the reference GridSpec cannot express — it uses
the pinned C restatement (oracle/liboracle.so, itself pinned to the reference
in tests/test_oracle.py). Inputs come from the checker-side generator
(orc_synth_chip, bitwise the product's bk_synth_chip); a SHA-256 of the input
bytes is stored so generator drift is caught.

The full solutions (33 MB for C3, 2.1 GB for C5) are too large to commit, so a
fixture keeps: the full column 2-norms of X, X on a fixed sample of cells
(rows), the solver reports, and for a few samples T and q on the same cells
(T = X C by the reference's combine_from_weights, q by its operator_action,
pipeline.cpp:187-251, evaluated on the full grid).

    python tests/golden/make_golden_full.py c3          # block_cg 1e-12, ~70 s
    python tests/golden/make_golden_full.py c4          # oracle, 1e-10
    python tests/golden/make_golden_full.py c5-capped   # block_cg m = 1, 2, 3 (~4 min)
    python tests/golden/make_golden_full.py c5-cg [W]   # per-column cg 1e-12, W workers (hours)
    python tests/golden/make_golden_full.py c5-pack     # fixture from the c5-cg results
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
WORK = os.environ.get("BK_GOLDEN_WORK", "/tmp/bk_golden_c5")
N_ROWS = 8192
MAX_ITER_CG = 20000
SAMPLES = [0, 1, 2499, 4999]


def digest(ch) -> str:
    h = hashlib.sha256()
    for a in (ch.k, ch.q_basis, ch.coef):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def sample_rows(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([rng.integers(0, n, N_ROWS), [0, n - 1]]))
    return rows.astype(np.int64)


def rhs(ref, op, ch):
    s = ch.q_basis.shape[1]
    B = np.empty_like(ch.q_basis)
    for j in range(s):
        B[:, j] = ref.rhs_from_power(op, np.ascontiguousarray(ch.q_basis[:, j]))
    return B


def tq_on_rows(ref, op, X, coef, samples, rows, threads=8):
    """T, q of `samples` on `rows` through the reference's combine_from_weights
    and operator_action (full grid), plus the per-sample residual."""
    basis = ref.basis(op, X)
    T, Q, R = [], [], []
    for j in samples:
        t, q, r = basis.combine_action(coef, j, j + 1, threads=1)
        T.append(t[0][rows])
        Q.append(q[0][rows])
        R.append(r[0])
    return np.array(T), np.array(Q), np.array(R)


def c3():
    o, ref = Oracle(), Reference()
    ch = o.synth_chip(3, 128, 128, 8, 32, 5000, chip_id=0)
    op = ref.assemble(ch.grid, ch.k, ch.bc)
    B = rhs(ref, op, ch)
    t = time.time()
    X, rep = ref.block_cg(op, B, 1e-12, 100000, 1)
    dt = time.time() - t
    n = op.n
    rows = sample_rows(n, 3)
    T, Q, R = tq_on_rows(ref, op, X, ch.coef, SAMPLES, rows)
    np.savez_compressed(os.path.join(OUT, "c3_full.npz"), rows=rows, x_rows=X[rows],
                        x_norms=np.linalg.norm(X, axis=0), iterations=rep["iterations"],
                        matvec_count=rep["matvec_count"], final_rel_residual=rep["final_rel_residual"],
                        converged=rep["converged"], samples=np.array(SAMPLES), t_rows=T, q_rows=Q,
                        resid=R, tol=1e-12, seconds=dt, input_sha256=digest(ch),
                        shape=np.array([128, 128, 8, 32, 5000]))
    print("c3", rep["iterations"], dt, rep["converged"].all())


def c4():
    o = Oracle()
    out = {}
    for chip in (0, 4):
        ch = o.synth_chip(4, 128, 128, 4, 16, 8, chip_id=chip)
        op = o.assemble(ch.grid, ch.k, ch.bc, dz=ch.dz)
        B = o.rhs_from_power(op, ch.q_basis)
        X, rep = o.block_cg(op, B, 1e-10, 5000, 1)
        T, Q, R = o.combine_action(op, X, ch.coef)
        rows = sample_rows(op.n, 40 + chip)
        out.update({f"chip{chip}_{k}": v for k, v in dict(
            rows=rows, x_rows=X[rows], x_norms=np.linalg.norm(X, axis=0),
            iterations=rep["iterations"], matvec_count=rep["matvec_count"],
            final_rel_residual=rep["final_rel_residual"], converged=rep["converged"],
            t_rows=T[:, rows], q_rows=Q[:, rows], resid=R, input_sha256=digest(ch)).items()})
        print("c4 chip", chip, rep["iterations"], rep["converged"].all(),
              float(np.max(rep["final_rel_residual"])))
    np.savez_compressed(os.path.join(OUT, "c4_full.npz"), tol=1e-10, **out)


def c5_inputs(o, ref):
    ch = o.synth_chip(5, 512, 512, 16, 64, 5000, chip_id=0)
    op = ref.assemble(ch.grid, ch.k, ch.bc)
    return ch, op


def c5_capped():
    o, ref = Oracle(), Reference()
    ch, op = c5_inputs(o, ref)
    B = rhs(ref, op, ch)
    rows = sample_rows(op.n, 5)
    out = {"rows": rows, "input_sha256": digest(ch), "tol": 1e-10}
    for m in (1, 2, 3):
        t = time.time()
        X, rep = ref.block_cg(op, B, 1e-10, m, 1)
        out[f"m{m}_x_rows"] = X[rows]
        out[f"m{m}_x_norms"] = np.linalg.norm(X, axis=0)
        out[f"m{m}_matvec_count"] = rep["matvec_count"]
        out[f"m{m}_iterations"] = rep["iterations"]
        print("c5 capped m", m, time.time() - t, flush=True)
    np.savez_compressed(os.path.join(OUT, "c5_capped.npz"), **out)


def _cg_worker(args):
    cols, tol = args
    o, ref = Oracle(), Reference()
    k = np.load(os.path.join(WORK, "k.npy"))
    meta = json.load(open(os.path.join(WORK, "meta.json")))
    op = ref.assemble(tuple(meta["grid"]), k, [tuple(f) for f in meta["bc"]])
    for j in cols:
        xp = os.path.join(WORK, f"x_{j:02d}.npy")
        if os.path.exists(xp):
            continue
        b = np.load(os.path.join(WORK, f"b_{j:02d}.npy"))
        t = time.time()
        x, rep = ref.cg(op, b, tol, MAX_ITER_CG, 1)
        rep = {kk: (float(v) if not isinstance(v, (bool, int)) else v) for kk, v in rep.items()}
        rep["seconds"] = time.time() - t
        np.save(xp + ".tmp.npy", x)
        os.replace(xp + ".tmp.npy", xp)
        json.dump(rep, open(os.path.join(WORK, f"rep_{j:02d}.json"), "w"))
        print("column", j, rep, flush=True)


def c5_cg(workers: int, tol: float = 1e-11):
    """Per-column reference cg (solvers.cpp:82-171) of the full C5 basis, the
    SURVEY §8(c) golden for config 5 (resumable; results in $BK_GOLDEN_WORK).
    tol 1e-11, not 1e-12: a lone C5 column, like a C2 one (tests/test_oracle.py),
    plateaus around 1e-12 in fp64, where the reference cg runs to max_iter
    (measured: 1 of 6 columns reached 1e-12 within ~35 minutes); 1e-11 is
    still ten times tighter than the GPU's pinned 1e-10."""
    from multiprocessing import Pool

    os.makedirs(WORK, exist_ok=True)
    if not os.path.exists(os.path.join(WORK, "meta.json")):
        o, ref = Oracle(), Reference()
        ch, op = c5_inputs(o, ref)
        B = rhs(ref, op, ch)
        np.save(os.path.join(WORK, "k.npy"), ch.k)
        for j in range(64):
            np.save(os.path.join(WORK, f"b_{j:02d}.npy"), np.ascontiguousarray(B[:, j]))
        np.save(os.path.join(WORK, "coef.npy"), ch.coef)
        json.dump({"grid": list(ch.grid), "bc": [list(f) for f in ch.bc], "sha256": digest(ch),
                   "tol": tol}, open(os.path.join(WORK, "meta.json"), "w"))
        del B, ch
    cols = [list(range(w, 64, workers)) for w in range(workers)]
    with Pool(workers) as p:
        p.map(_cg_worker, [(c, tol) for c in cols])


def c5_pack():
    o, ref = Oracle(), Reference()
    meta = json.load(open(os.path.join(WORK, "meta.json")))
    k = np.load(os.path.join(WORK, "k.npy"))
    op = ref.assemble(tuple(meta["grid"]), k, [tuple(f) for f in meta["bc"]])
    n = op.n
    X = np.empty((n, 64))
    reps = []
    for j in range(64):
        X[:, j] = np.load(os.path.join(WORK, f"x_{j:02d}.npy"))
        reps.append(json.load(open(os.path.join(WORK, f"rep_{j:02d}.json"))))
    coef = np.load(os.path.join(WORK, "coef.npy"))
    rows = sample_rows(n, 5)
    T, Q, R = tq_on_rows(ref, op, X, coef, SAMPLES, rows)
    np.savez_compressed(os.path.join(OUT, "c5_full_cg.npz"), rows=rows, x_rows=X[rows],
                        x_norms=np.linalg.norm(X, axis=0),
                        iterations=np.array([r["iterations"] for r in reps]),
                        final_rel_residual=np.array([r["final_rel_residual"] for r in reps]),
                        converged=np.array([r["converged"] for r in reps]),
                        seconds=np.array([r["seconds"] for r in reps]),
                        samples=np.array(SAMPLES), t_rows=T, q_rows=Q, resid=R,
                        tol=meta["tol"], input_sha256=meta["sha256"])
    print("packed", [r["iterations"] for r in reps])


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "c3":
        c3()
    elif what == "c4":
        c4()
    elif what == "c5-capped":
        c5_capped()
    elif what == "c5-cg":
        c5_cg(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    elif what == "c5-pack":
        c5_pack()
    else:
        raise SystemExit(__doc__)
