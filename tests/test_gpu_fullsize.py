"""GPU parity at the full BASELINE shapes of configs 3, 4 and 5.

Goldens (tests/golden/make_golden_full.py, from the unmodified reference core
except config 4 — per-layer dz, not expressible in the reference GridSpec —
which uses the pinned C restatement) keep the full column norms of the basis
X, X on a fixed sample of cells, and T / q of a few samples on those cells.
Bars: T and q within 1e-9 relative L2 (BASELINE north_star), X within 1e-9;
capped iterates within 1e-12 with identical matvec accounting; iteration counts
reported next to the reference's.
"""
import hashlib
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, rel_l2

pytestmark = pytest.mark.gpu
PARITY = 1e-9


def sha(ch):
    h = hashlib.sha256()
    for a in (ch.k, ch.q_basis, ch.coef):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def solve_full(bk, ctx, ch, tol, max_iter=100000):
    import torch

    dev = torch.device("cuda", 0)
    op = bk.assemble(ch.k, ch.grid, ch.bc, ctx)
    q = torch.from_numpy(ch.q_basis).to(dev)
    B = torch.empty_like(q)
    bk.rhs_from_power(op, q, out=B)
    X = torch.empty_like(q)
    r = bk.block_cg(op, B, bk.SolverConfig(tol, max_iter, "jacobi"), out=X)
    torch.cuda.synchronize()
    return op, X, r.report


def check_x(X, d, prefix=""):
    Xh = X.cpu().numpy() if hasattr(X, "cpu") else X
    norms = np.linalg.norm(Xh, axis=0)
    gn = d[prefix + "x_norms"]
    assert np.max(np.abs(norms - gn) / np.where(gn > 0, gn, 1.0)) <= PARITY
    rows = d[prefix + "rows"]
    return rel_l2(Xh[rows], d[prefix + "x_rows"])


def check_tq(bk, op, X, coef, samples, d, t_key="t_rows", q_key="q_rows", prefix=""):
    import torch

    dev = torch.device("cuda", 0)
    rows = d[prefix + "rows"]
    c = torch.from_numpy(np.ascontiguousarray(coef[:, samples])).to(dev)
    n, m = op.n, len(samples)
    T = torch.empty((m, n), dtype=torch.float64, device=dev)
    Q = torch.empty_like(T)
    R = torch.empty(m, dtype=torch.float64, device=dev)
    bk.combine_action(op, X, c, t_out=T, q_out=Q, resid_out=R)
    torch.cuda.synchronize()
    Th, Qh = T.cpu().numpy(), Q.cpu().numpy()
    for i in range(m):
        assert rel_l2(Th[i, rows], d[prefix + t_key][i]) <= PARITY, ("T", samples[i])
        assert rel_l2(Qh[i, rows], d[prefix + q_key][i]) <= PARITY, ("q", samples[i])
    assert float(R.max().item()) <= 1e-12


def test_c3_full_vs_reference(bk, ctx):
    """C3 128x128x8, s = 32, block CG at 1e-12 against the reference's own
    block_cg (solvers.cpp:452-665) on the same chip; (T, q) of samples 0, 1,
    2499, 4999 against combine_from_weights / operator_action."""
    d = golden("c3_full.npz")
    ch = bk.synth_chip(3, 128, 128, 8, 32, 5000, chip_id=0)
    assert sha(ch) == str(d["input_sha256"])
    op, X, rep = solve_full(bk, ctx, ch, 1e-12)
    assert rep.all_converged() and bool(np.all(d["converged"]))
    assert abs(rep.iterations - int(d["iterations"])) <= max(3, int(d["iterations"]) // 4)
    assert check_x(X, d) <= PARITY
    check_tq(bk, op, X, ch.coef, list(d["samples"]), d)


def test_c3_batched_bench_path_vs_reference(bk, ctx):
    """The bench's C3 step: z-stacked chips solved by one batched launch
    (bk_generate_batch); chip 0's (T, q) against the reference golden."""
    import torch
    from types import SimpleNamespace

    d = golden("c3_full.npz")
    dev = torch.device("cuda", 0)
    samples = list(d["samples"])
    chips = []
    for c in range(4):
        ch = bk.synth_chip(3, 128, 128, 8, 32, 5000, chip_id=c)
        coef = np.ascontiguousarray(ch.coef[:, samples])
        chips.append(SimpleNamespace(grid=ch.grid, bc=ch.bc, k=torch.from_numpy(ch.k).to(dev),
                                     q_basis=torch.from_numpy(ch.q_basis).to(dev),
                                     coef=torch.from_numpy(coef).to(dev)))
    n, m = 128 * 128 * 8, len(samples)
    T = [torch.empty((m, n), dtype=torch.float64, device=dev) for _ in chips]
    Q = [torch.empty((m, n), dtype=torch.float64, device=dev) for _ in chips]
    R = [torch.empty(m, dtype=torch.float64, device=dev) for _ in chips]
    _, _, _, reps, _ = bk.generate_batch(chips, bk.SolverConfig(1e-12, 100000, "jacobi"), T, Q, R,
                                         streams=4, ctx=ctx)
    torch.cuda.synchronize()
    assert ctx.last_solver_variant.startswith("block_cg_dmma_kernel<32,0,1,1>")
    rows = d["rows"]
    Th, Qh = T[0].cpu().numpy(), Q[0].cpu().numpy()
    for i in range(m):
        assert rel_l2(Th[i, rows], d["t_rows"][i]) <= PARITY
        assert rel_l2(Qh[i, rows], d["q_rows"][i]) <= PARITY
    assert all(r.all_converged() for r in reps)


@pytest.mark.parametrize("chip", [0, 4])
def test_c4_full_vs_oracle(bk, ctx, chip):
    """C4 128x128x4 chips with per-layer dz (the restatement's assemble_layered),
    block CG at the pinned 1e-10, in the bench's batched launch of 32 chips."""
    import torch
    from types import SimpleNamespace

    d = golden("c4_full.npz")
    p = f"chip{chip}_"
    dev = torch.device("cuda", 0)
    chips, host = [], None
    for c in range(32):
        ch = bk.synth_chip(4, 128, 128, 4, 16, 8, chip_id=c)
        if c == chip:
            host = ch
        chips.append(SimpleNamespace(grid=ch.grid, bc=ch.bc, k=torch.from_numpy(ch.k).to(dev),
                                     q_basis=torch.from_numpy(ch.q_basis).to(dev),
                                     coef=torch.from_numpy(ch.coef).to(dev)))
    assert sha(host) == str(d[p + "input_sha256"])
    n = 128 * 128 * 4
    T = [torch.empty((8, n), dtype=torch.float64, device=dev) for _ in chips]
    Q = [torch.empty((8, n), dtype=torch.float64, device=dev) for _ in chips]
    R = [torch.empty(8, dtype=torch.float64, device=dev) for _ in chips]
    _, _, _, reps, _ = bk.generate_batch(chips, bk.SolverConfig(1e-10, 5000, "jacobi"), T, Q, R,
                                         streams=32, ctx=ctx, check_converged=False)
    torch.cuda.synchronize()
    assert reps[chip].all_converged() and bool(np.all(d[p + "converged"]))
    rows = d[p + "rows"]
    Th, Qh = T[chip].cpu().numpy(), Q[chip].cpu().numpy()
    for j in range(8):
        assert rel_l2(Th[j, rows], d[p + "t_rows"][j]) <= PARITY, j
        assert rel_l2(Qh[j, rows], d[p + "q_rows"][j]) <= PARITY, j


@pytest.fixture(scope="module")
def c5_chip(bk):
    return bk.synth_chip(5, 512, 512, 16, 64, 5000, chip_id=0)


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c5_capped.npz")),
                    reason="c5_capped.npz not generated")
def test_c5_capped_iterates_vs_reference(bk, ctx, c5_chip):
    """C5 512x512x16, s = 64: the multi-kernel engine's iterates after m = 1,
    2, 3 block-CG steps equal the reference block_cg's (same matvec counts)."""
    d = golden("c5_capped.npz")
    assert sha(c5_chip) == str(d["input_sha256"])
    for m in (1, 2, 3):
        op, X, rep = solve_full(bk, ctx, c5_chip, 1e-10, max_iter=m)
        assert ctx.last_solver_variant.startswith("block_cg_large<64>")
        assert rep.iterations == m and rep.matvec_count == int(d[f"m{m}_matvec_count"])
        Xh = X.cpu().numpy()
        gn = d[f"m{m}_x_norms"]
        assert np.max(np.abs(np.linalg.norm(Xh, axis=0) - gn) / gn) <= 1e-12
        assert rel_l2(Xh[d["rows"]], d[f"m{m}_x_rows"]) <= 1e-12


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "c5_full_cg.npz")),
                    reason="c5_full_cg.npz not generated")
def test_c5_full_vs_reference_cg(bk, ctx, c5_chip):
    """C5 full solve at the pinned 1e-10 against the reference's per-column cg
    (solvers.cpp:82-171) run to 1e-11 on all 64 columns (3136-3288 iterations
    each, tests/golden/make_golden_full.py c5-cg): X and (T, q) of samples 0,
    1, 2499, 4999 within 1e-9."""
    d = golden("c5_full_cg.npz")
    assert sha(c5_chip) == str(d["input_sha256"])
    op, X, rep = solve_full(bk, ctx, c5_chip, 1e-10)
    assert rep.all_converged()
    assert check_x(X, d) <= PARITY
    check_tq(bk, op, X, c5_chip.coef, list(d["samples"]), d)
