"""GPU parity tests: the sm_100a path (through the C ABI) against the reference
golden fixtures and the CPU oracle on the same seeded inputs.

Bars: integer structure bitwise; stencil coefficients, apply_block,
rhs_from_power, and combine/action (given the same X) bitwise; block-CG
solutions within 1e-9 relative L2 (Krylov reduction order differs); full-chain
(T, q) within 1e-9 relative L2; every sample residual <= 1e-12.
"""
import numpy as np
import pytest

from conftest import golden, grid_tuple, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-12
PARITY = 1e-9


def cfg_jacobi(max_iter=100000):
    import paper_2510_23221_b200 as bk
    return bk.SolverConfig(TOL, max_iter, "jacobi")


# ----------------------------------------------------------------- discretization
def test_kat_3x3x3_bitwise(bk, ctx):
    d = golden("kat_3x3x3.npz")
    op = bk.assemble(np.ones(27), bk.GridSpec(3, 3, 3, 3.0, 3.0, 3.0),
                     bk.BoundarySpec.uniform_dirichlet(0.0), ctx)
    for a, b in zip(op.csr(), (d["row_ptr"], d["col"], d["val"], d["g"], d["vol"])):
        assert a.dtype == b.dtype and np.array_equal(a, b)


def test_mixed_operator_and_apply_bitwise(bk, ctx):
    d = golden("mixed_operator.npz")
    faces = []
    for kd, a, b in zip(d["bc_kind"], d["bc_a"], d["bc_b"]):
        faces.append(bk.Dirichlet(a) if kd == 0 else bk.Robin(a, b) if kd == 1 else bk.Adiabatic())
    gr = d["grid"]
    grid = bk.GridSpec(int(gr[0]), int(gr[1]), int(gr[2]), gr[3], gr[4], gr[5])
    op = bk.assemble(d["k"], grid, bk.BoundarySpec(faces), ctx)
    for a, key in zip(op.csr(), ("row_ptr", "col", "val", "g", "vol")):
        assert np.array_equal(a, d[key]), key
    for s in (1, 4, 7, 16):
        x = d[f"x{s}"]
        assert np.array_equal(op.apply_block(x), d[f"y{s}"]), s


def test_operator_from_reference_csr(bk, ctx):
    """bk_operator_from_csr on the reference's own assembled CSR (golden): the
    same operator bitwise as bk_assemble, so block_cg(const CsrMatrix&) is a
    drop-in."""
    d = golden("mixed_operator.npz")
    faces = [bk.Dirichlet(a) if kd == 0 else bk.Robin(a, b) if kd == 1 else bk.Adiabatic()
             for kd, a, b in zip(d["bc_kind"], d["bc_a"], d["bc_b"])]
    gr = d["grid"]
    grid = bk.GridSpec(int(gr[0]), int(gr[1]), int(gr[2]), gr[3], gr[4], gr[5])
    op = bk.operator_from_csr(grid, d["row_ptr"], d["col"], d["val"], d["g"], d["vol"], ctx)
    for a, key in zip(op.csr(), ("row_ptr", "col", "val", "g", "vol")):
        assert np.array_equal(a, d[key]), key
    for s in (1, 4, 7, 16):
        assert np.array_equal(op.apply_block(d[f"x{s}"]), d[f"y{s}"]), s
    ref = bk.assemble(d["k"], grid, bk.BoundarySpec(faces), ctx)
    B = np.random.default_rng(3).uniform(0.0, 1.0, (grid.cell_count(), 8))
    r1, r2 = bk.block_cg(op, B, cfg_jacobi()), bk.block_cg(ref, B, cfg_jacobi())
    assert np.array_equal(r1.x, r2.x) and r1.report.iterations == r2.report.iterations


def test_operator_from_csr_nonuniform_layers_and_rejects(bk, ctx, oracle):
    inp = bk.synth_chip(4, 20, 12, 4, 16, 2, chip_id=3)
    g = inp.grid
    o = oracle.assemble(grid_tuple(g), inp.k, inp.bc.as_tuples(), dz=g.dz)
    row_ptr, col, val, gg, vol = oracle.csr(o)
    op = bk.operator_from_csr(g, row_ptr, col, val, gg, vol, ctx)
    ref = bk.assemble(inp.k, g, inp.bc, ctx)
    B = oracle.rhs_from_power(o, inp.q_basis)
    assert np.array_equal(bk.block_cg(op, B, cfg_jacobi()).x, bk.block_cg(ref, B, cfg_jacobi()).x)
    T1, Q1, _ = bk.combine_action(op, B, inp.coef)
    T2, Q2, _ = bk.combine_action(ref, B, inp.coef)
    assert np.array_equal(T1, T2) and np.array_equal(Q1, Q2)
    bad = val.copy()
    p = int(np.flatnonzero(col[row_ptr[5]:row_ptr[6]] == 6)[0]) + int(row_ptr[5])
    bad[p] *= 1.0 + 1e-15  # A[5][6] != A[6][5]
    with pytest.raises(bk.InvalidSpecError):
        bk.operator_from_csr(g, row_ptr, col, bad, gg, vol, ctx)
    wrong = bk.GridSpec(g.nx * 2, g.ny // 2, g.nz, g.lx, g.ly, g.lz, dz=g.dz)
    with pytest.raises(bk.InvalidSpecError):
        bk.operator_from_csr(wrong, row_ptr, col, val, gg, vol, ctx)
    v2 = vol.copy()
    v2[7] *= 2.0
    with pytest.raises(bk.InvalidSpecError):
        bk.operator_from_csr(g, row_ptr, col, val, gg, v2, ctx)


@pytest.mark.parametrize("case", [(1, 32, 32, 1, 8), (2, 48, 40, 1, 16), (3, 16, 16, 8, 32),
                                  (4, 24, 16, 4, 16), (5, 8, 8, 16, 64)])
def test_assemble_apply_rhs_bitwise_vs_oracle(bk, ctx, oracle, case):
    inp = bk.synth_chip(*case, 4)
    g = inp.grid
    op = bk.assemble(inp.k, g, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(g), inp.k, inp.bc.as_tuples(), dz=g.dz)
    for a, b in zip(op.csr(), oracle.csr(o)):
        assert np.array_equal(a, b)
    x = np.random.default_rng(1).standard_normal((g.cell_count(), 5))
    assert np.array_equal(op.apply_block(x), oracle.apply_block(o, x))
    assert np.array_equal(bk.rhs_from_power(op, inp.q_basis), oracle.rhs_from_power(o, inp.q_basis))
    b = oracle.rhs_from_power(o, inp.q_basis)
    assert np.array_equal(bk.power_from_rhs(op, b), oracle.power_from_rhs(o, b))


def test_assemble_into_reuses_and_matches(bk, ctx):
    """bk_assemble_into: re-assembling another chip into an existing operator
    (buffers reused) gives bitwise the freshly assembled operator."""
    a = bk.synth_chip(3, 24, 20, 8, 8, 2, chip_id=0)
    b = bk.synth_chip(3, 24, 20, 8, 8, 2, chip_id=1)
    op = bk.assemble(a.k, a.grid, a.bc, ctx)
    h = op.h.value
    op2 = bk.assemble(b.k, b.grid, b.bc, ctx, out=op)
    assert op2 is op and op.h.value == h
    fresh = bk.assemble(b.k, b.grid, b.bc, ctx)
    for x, y in zip(op.csr(), fresh.csr()):
        assert np.array_equal(x, y)


def test_operator_action_center_indicator(bk, ctx):
    """q = center column of A (27-cell, g = 0, unit volumes)."""
    op = bk.assemble(np.ones(27), bk.GridSpec(3, 3, 3, 3.0, 3.0, 3.0),
                     bk.BoundarySpec.uniform_dirichlet(0.0), ctx)
    x = np.zeros((27, 1))
    x[13, 0] = 1.0
    T, Q, R = bk.combine_action(op, x, np.ones((1, 1)))
    assert Q[0, 13] == 6.0 and all(Q[0, i] == -1.0 for i in (4, 10, 12, 14, 16, 22))
    assert R[0] == 0.0 and T[0, 13] == 1.0


# ----------------------------------------------------------------- solver
@pytest.mark.parametrize("name", ["c1_full", "c2_reduced", "c3_reduced", "c5_reduced"])
def test_block_cg_vs_reference_golden(bk, ctx, oracle, name):
    d = golden(f"{name}.npz")
    cfg, (nx, ny, nz, s, N) = int(d["config"]), d["shape"].tolist()
    inp = bk.synth_chip(cfg, nx, ny, nz, s, N)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    B = bk.rhs_from_power(op, inp.q_basis)
    r = bk.block_cg(op, B, cfg_jacobi())
    assert r.report.all_converged()
    assert np.all(r.report.final_rel_residual <= TOL)
    assert rel_l2(r.x, d["X"]) <= PARITY
    ref_it = int(d["iterations"])
    assert abs(r.report.iterations - ref_it) <= max(3, ref_it // 10)
    # independent check of the GPU solution with the oracle's CSR apply
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    res = np.linalg.norm(B - oracle.apply_block(o, r.x), axis=0) / np.linalg.norm(B, axis=0)
    assert np.all(res <= 1.5 * TOL)


def test_block_cg_matches_oracle_iterates(bk, ctx, oracle):
    """Capped iteration counts: GPU iterate after m steps == oracle iterate."""
    inp = bk.synth_chip(3, 16, 16, 8, 32, 4)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    B = oracle.rhs_from_power(o, inp.q_basis)
    for m in (1, 2, 5, 13):
        r = bk.block_cg(op, B, cfg_jacobi(m))
        X, rep = oracle.block_cg(o, B, TOL, m, 1)
        assert r.report.iterations == rep["iterations"] == m
        assert r.report.matvec_count == rep["matvec_count"]
        assert not r.report.converged.any() and not rep["converged"].any()
        assert rel_l2(r.x, X) <= 1e-12
        assert np.allclose(r.report.final_rel_residual, rep["final_rel_residual"], rtol=1e-9)


def test_block_cg_nonuniform_stack_vs_oracle(bk, ctx, oracle):
    """BASELINE config 4 (per-chip non-uniform dz; not expressible in the
    reference GridSpec) against the oracle restatement."""
    for chip in (0, 1):
        inp = bk.synth_chip(4, 32, 32, 4, 16, 8, chip_id=chip)
        op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
        o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples(), dz=inp.grid.dz)
        B = oracle.rhs_from_power(o, inp.q_basis)
        r = bk.block_cg(op, B, cfg_jacobi())
        X, rep = oracle.block_cg(o, B, TOL, 100000, 1)
        assert r.report.all_converged() and rep["converged"].all()
        assert rel_l2(r.x, X) <= PARITY


def test_block_cg_duplicate_and_zero_columns(bk, ctx, oracle):
    """SPEC.md:211 duplicate columns (rank-deficient block -> pivoted Cholesky
    path) and zero right-hand sides (x = 0, converged, solvers.cpp:478-485)."""
    inp = bk.synth_chip(1, 24, 24, 1, 8, 1)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    B = oracle.rhs_from_power(o, inp.q_basis)
    B[:, 3] = B[:, 1]
    B[:, 5] = 0.0
    r = bk.block_cg(op, B, cfg_jacobi())
    X, rep = oracle.block_cg(o, B, TOL, 100000, 1)
    assert r.report.all_converged() and rep["converged"].all()
    assert np.all(r.x[:, 5] == 0.0) and r.report.final_rel_residual[5] == 0.0
    assert rel_l2(r.x, X) <= PARITY
    assert rel_l2(r.x[:, 3], r.x[:, 1]) <= 10 * TOL


def test_s1_and_odd_widths(bk, ctx, oracle):
    """s = 1 equals CG; widths padded to the kernel width."""
    inp = bk.synth_chip(1, 24, 20, 1, 8, 1)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    B = oracle.rhs_from_power(o, inp.q_basis)
    b = np.ascontiguousarray(B[:, 0])
    x, rc = oracle.cg(o, b, TOL, 100000, 1)
    r = bk.block_cg(op, b[:, None].copy(), cfg_jacobi())
    assert rel_l2(r.x[:, 0], x) <= 10 * TOL and r.report.converged[0] == rc["converged"]
    for s in (3, 5, 11):
        Bs = np.ascontiguousarray(B[:, :min(s, 8)]) if s <= 8 else np.ascontiguousarray(
            np.concatenate([B, B[:, : s - 8] * 0.5 + 1e-3 * B[:, 1: s - 7]], axis=1))
        r = bk.block_cg(op, Bs, cfg_jacobi())
        X, rep = oracle.block_cg(o, Bs, TOL, 100000, 1)
        assert r.report.all_converged() and rel_l2(r.x, X) <= PARITY


def test_block_cg_deterministic(bk, ctx):
    inp = bk.synth_chip(2, 64, 64, 1, 16, 1)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    B = bk.rhs_from_power(op, inp.q_basis)
    r1 = bk.block_cg(op, B, cfg_jacobi())
    r2 = bk.block_cg(op, B, cfg_jacobi())
    assert np.array_equal(r1.x, r2.x) and r1.report.iterations == r2.report.iterations


def test_errors_map_to_reference_exceptions(bk, ctx):
    grid = bk.GridSpec(4, 4, 1, 1e-3, 1e-3, 1e-4)
    bc = bk.BoundarySpec.uniform_dirichlet(0.0)
    k = np.ones(16)
    with pytest.raises(bk.NonPositiveConductivityError):
        bk.assemble(np.where(np.arange(16) == 5, -1.0, 1.0), grid, bc, ctx)
    with pytest.raises(bk.NonPositiveHtcError):
        bk.assemble(k, grid, bk.BoundarySpec([bk.Robin(0.0, 1.0)] + [bk.Dirichlet()] * 5), ctx)
    with pytest.raises(bk.InvalidSpecError):
        bk.assemble(np.ones(0), bk.GridSpec(0, 4, 1, 1, 1, 1), bc, ctx)
    with pytest.raises(bk.DimensionMismatchError):
        bk.assemble(np.ones(15), grid, bc, ctx)
    op = bk.assemble(k, grid, bc, ctx)
    with pytest.raises(bk.InvalidConfigError):
        bk.block_cg(op, np.ones((16, 2)), bk.SolverConfig(1.5, 10, "jacobi"))
    with pytest.raises(bk.InvalidConfigError):
        bk.block_cg(op, np.ones((16, 2)), bk.SolverConfig(1e-9, 0, "jacobi"))
    with pytest.raises(bk.DimensionMismatchError):
        bk.block_cg(op, np.ones((15, 2)), cfg_jacobi())
    with pytest.raises(bk.EmptyBasisError):
        bk.combine_action(op, np.ones((16, 0)), np.ones((0, 3)))


# ----------------------------------------------------------------- combine + action
@pytest.mark.parametrize("name", ["c1_full", "c2_reduced", "c3_reduced", "c5_reduced"])
def test_combine_action_bitwise_vs_reference_golden(bk, ctx, name):
    """Given the reference's X, T and q equal the reference's bit for bit."""
    d = golden(f"{name}.npz")
    cfg, (nx, ny, nz, s, N) = int(d["config"]), d["shape"].tolist()
    inp = bk.synth_chip(cfg, nx, ny, nz, s, N)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    T, Q, R = bk.combine_action(op, d["X"], inp.coef)
    keep = d["keep"]
    assert np.array_equal(T[keep], d["T"]) and np.array_equal(Q[keep], d["Q"])
    assert np.allclose(R, d["resid"], rtol=1e-6, atol=1e-17) and np.max(R) <= TOL


def test_combine_action_bitwise_vs_oracle_odd_shapes(bk, ctx, oracle):
    # widths 5 and 20 run on the padded 8 / 32 kernels: only the real s rows of
    # C may be read
    # single-plane grids with S = 32 / 64 (two / four TMA panels per plane),
    # odd nx (the cell-pair path's unpaired last column), 3D with S = 64
    for case, N in (((1, 37, 29, 1, 8), 19), ((3, 33, 17, 8, 32), 21), ((4, 20, 9, 4, 16), 8),
                    ((1, 37, 29, 1, 5), 19), ((3, 16, 12, 8, 20), 33),
                    ((1, 41, 23, 1, 20), 37), ((1, 35, 9, 1, 40), 18), ((3, 19, 21, 8, 64), 17)):
        inp = bk.synth_chip(*case, N)
        g = inp.grid
        op = bk.assemble(inp.k, g, inp.bc, ctx)
        o = oracle.assemble(grid_tuple(g), inp.k, inp.bc.as_tuples(), dz=g.dz)
        X = np.random.default_rng(2).uniform(0, 50, (g.cell_count(), case[4]))
        coef = inp.coef.copy()
        coef[0, 3] = 0.0      # zero weights are skipped in the reference
        coef[:, 5] = 0.0
        T, Q, R = bk.combine_action(op, X, coef)
        To, Qo, Ro = oracle.combine_action(o, X, coef)
        assert np.array_equal(T, To) and np.array_equal(Q, Qo)
        assert np.allclose(R, Ro, rtol=1e-6, atol=1e-17)


# ----------------------------------------------------------------- full chain
@pytest.mark.parametrize("name", ["c1_full", "c2_reduced", "c3_reduced", "c5_reduced"])
def test_generate_chip_vs_reference_golden(bk, ctx, name):
    d = golden(f"{name}.npz")
    cfg, (nx, ny, nz, s, N) = int(d["config"]), d["shape"].tolist()
    inp = bk.synth_chip(cfg, nx, ny, nz, s, N)
    T, Q, R, rep, tim = bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef,
                                         cfg_jacobi(), ctx=ctx)
    keep = d["keep"]
    for j, kk in enumerate(keep):
        assert rel_l2(T[kk], d["T"][j]) <= PARITY
        assert rel_l2(Q[kk], d["Q"][j]) <= PARITY
    assert np.max(R) <= TOL and rep.all_converged()
    assert tim.basis_solve_s > 0 and tim.total_s >= tim.basis_solve_s


def test_generate_chip_nonuniform_vs_oracle(bk, ctx, oracle):
    inp = bk.synth_chip(4, 32, 32, 4, 16, 8, chip_id=7)
    T, Q, R, rep, _ = bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef,
                                       cfg_jacobi(), ctx=ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples(), dz=inp.grid.dz)
    X, _ = oracle.block_cg(o, oracle.rhs_from_power(o, inp.q_basis), TOL, 100000, 1)
    To, Qo, Ro = oracle.combine_action(o, X, inp.coef)
    assert rel_l2(T, To) <= PARITY and rel_l2(Q, Qo) <= PARITY and np.max(R) <= TOL


def test_generate_chip_host_and_device_pointers_agree(bk, ctx):
    import torch

    inp = bk.synth_chip(2, 64, 64, 1, 16, 40)
    T1, Q1, R1, rep1, _ = bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef,
                                           cfg_jacobi(), ctx=ctx)
    dev = torch.device("cuda", 0)
    n, N = inp.grid.cell_count(), 40
    Td = torch.empty((N, n), dtype=torch.float64, device=dev)
    Qd = torch.empty_like(Td)
    Rd = torch.empty(N, dtype=torch.float64, device=dev)
    bk.generate_chip(inp.grid, torch.from_numpy(inp.k).to(dev), inp.bc,
                     torch.from_numpy(inp.q_basis).to(dev), torch.from_numpy(inp.coef).to(dev),
                     cfg_jacobi(), t_out=Td, q_out=Qd, resid_out=Rd, ctx=ctx)
    torch.cuda.synchronize()
    assert np.array_equal(Td.cpu().numpy(), T1) and np.array_equal(Qd.cpu().numpy(), Q1)
    assert np.array_equal(Rd.cpu().numpy(), R1)


def test_generate_chip_host_outputs_chunked(bk, ctx):
    """Host output buffers are drained in sample chunks overlapped with the
    combine (64 samples per chunk at 256 x 256): 150 samples = 3 chunks, the
    last one partial; identical to the device-pointer call."""
    import torch

    inp = bk.synth_chip(2, 256, 256, 1, 16, 150)
    n, N = inp.grid.cell_count(), 150
    pin = lambda *shape: torch.empty(shape, dtype=torch.float64).pin_memory()  # noqa: E731
    Th, Qh, Rh = pin(N, n), pin(N, n), pin(N)
    bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef, cfg_jacobi(),
                     t_out=Th, q_out=Qh, resid_out=Rh, ctx=ctx)
    dev = torch.device("cuda", 0)
    Td = torch.empty((N, n), dtype=torch.float64, device=dev)
    Qd = torch.empty_like(Td)
    Rd = torch.empty(N, dtype=torch.float64, device=dev)
    bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef, cfg_jacobi(),
                     t_out=Td, q_out=Qd, resid_out=Rd, ctx=ctx)
    torch.cuda.synchronize()
    assert torch.equal(Td.cpu(), Th) and torch.equal(Qd.cpu(), Qh) and torch.equal(Rd.cpu(), Rh)
    T2, Q2, R2, _, _ = bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef,
                                        cfg_jacobi(), ctx=ctx)  # pageable numpy outputs
    assert np.array_equal(T2, Th.numpy()) and np.array_equal(Q2, Qh.numpy())


@pytest.mark.slow
def test_full_size_c2_properties(bk, ctx, oracle):
    """BASELINE config 2 at full size: size-independent properties against the
    oracle (the full oracle pipeline takes minutes): per-column true residual of
    the GPU basis via the oracle CSR, X column norms vs the reference's own
    full solve (tests/golden/c2_full_meta.npz), sampled (T, q) bitwise equal to
    the oracle's combine/action on the GPU basis, every sample residual."""
    import torch

    d = golden("c2_full_meta.npz")
    inp = bk.synth_chip(*bk.CONFIGS[2])
    n, s, N = inp.grid.cell_count(), 16, 2048
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    B = bk.rhs_from_power(op, inp.q_basis)
    r = bk.block_cg(op, B, cfg_jacobi())
    assert r.report.all_converged()
    res = np.linalg.norm(B - oracle.apply_block(o, r.x), axis=0) / np.linalg.norm(B, axis=0)
    assert np.all(res <= 1.5 * TOL)
    assert np.allclose(np.linalg.norm(r.x, axis=0), d["X_colnorm"], rtol=PARITY)
    assert abs(r.report.iterations - int(d["iterations"])) <= int(d["iterations"]) // 10
    dev = torch.device("cuda", 0)
    Td = torch.empty((N, n), dtype=torch.float64, device=dev)
    Qd = torch.empty_like(Td)
    Rd = torch.empty(N, dtype=torch.float64, device=dev)
    bk.combine_action(op, r.x, inp.coef, t_out=Td, q_out=Qd, resid_out=Rd)
    torch.cuda.synchronize()
    pick = [0, 1, 777, 2047]
    To, Qo, Ro = oracle.combine_action(o, r.x, inp.coef[:, pick].copy())
    assert np.array_equal(Td[pick].cpu().numpy(), To)
    assert np.array_equal(Qd[pick].cpu().numpy(), Qo)
    assert float(Rd.max()) <= TOL
    # determinism of the whole chain
    T2, Q2, R2, rep2, _ = bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef,
                                           cfg_jacobi(), ctx=ctx)
    T3, Q3, R3, rep3, _ = bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef,
                                           cfg_jacobi(), ctx=ctx)
    assert np.array_equal(T2, T3) and np.array_equal(Q2, Q3)
    assert rel_l2(T2[pick], To) <= PARITY and rel_l2(Q2[pick], Qo) <= PARITY


def test_launch_counter_and_native_library_loaded(bk, ctx):
    import os

    before = ctx.launch_count
    inp = bk.synth_chip(1, 16, 16, 1, 8, 4)
    bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef, cfg_jacobi(), ctx=ctx)
    assert ctx.launch_count > before
    maps = open("/proc/self/maps").read()
    assert os.path.basename(bk.library_path()) in maps


def test_generate_batch_matches_per_chip(bk, ctx, oracle):
    """Config 4 batch path. streams = 1 (and host outputs with more streams):
    chips one after another, bitwise the single-chip runs. streams = K with
    device outputs: groups of K chips z-stacked and solved by one cooperative
    launch, chip k on 1/K of the SMs — bitwise the single-chip run given the
    same SM share (same CTA ranges and reduction order). Oracle parity."""
    import torch

    chips = [bk.synth_chip(4, 32, 24, 4, 16, 8, chip_id=c) for c in range(5)]
    for streams in (1, 2):  # host outputs: sequential
        T, Q, R, reps, tim = bk.generate_batch(chips, cfg_jacobi(), streams=streams, ctx=ctx)
        assert len(reps) == 5 and all(r.all_converged() for r in reps)
        assert tim.total_s > 0 and tim.iterations_total == sum(r.iterations for r in reps)
        for c, ch in enumerate(chips):
            T1, Q1, R1, rep1, _ = bk.generate_chip(ch.grid, ch.k, ch.bc, ch.q_basis, ch.coef,
                                                   cfg_jacobi(), ctx=ctx)
            assert np.array_equal(T[c], T1) and np.array_equal(Q[c], Q1)
    o = oracle.assemble(grid_tuple(chips[2].grid), chips[2].k, chips[2].bc.as_tuples(),
                        dz=chips[2].grid.dz)
    X, _ = oracle.block_cg(o, oracle.rhs_from_power(o, chips[2].q_basis), TOL, 100000, 1)
    To, Qo, _ = oracle.combine_action(o, X, chips[2].coef)
    assert rel_l2(T[2], To) <= PARITY and rel_l2(Q[2], Qo) <= PARITY
    # batched pipeline: 5 chips in groups of 3 (3 + 2), device outputs
    dev = torch.device("cuda", 0)
    n, N = chips[0].grid.cell_count(), 8
    Td = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in chips]
    Qd = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in chips]
    Rd = [torch.empty(N, dtype=torch.float64, device=dev) for _ in chips]
    _, _, _, reps, tim = bk.generate_batch(chips, cfg_jacobi(), t_out=Td, q_out=Qd, resid_out=Rd,
                                           streams=3, ctx=ctx)
    torch.cuda.synchronize()
    assert all(r.all_converged() for r in reps)
    for c, ch in enumerate(chips):
        sub = bk.Context(0)
        bk.set_cg_sm_budget(sub, sub_budget(3 if c < 3 else 2))
        T1, Q1, R1, rep1, _ = bk.generate_chip(ch.grid, ch.k, ch.bc, ch.q_basis, ch.coef,
                                               cfg_jacobi(), ctx=sub)
        assert reps[c].iterations == rep1.iterations
        assert np.array_equal(Td[c].cpu().numpy(), T1) and np.array_equal(Qd[c].cpu().numpy(), Q1)


def test_generate_batch_stacked_2d_vs_oracle(bk, ctx, oracle):
    """Batched pipeline on 2D chips (C2-like, resident solver): every chip
    within tolerance of the oracle."""
    import torch

    chips = [bk.synth_chip(2, 48, 40, 1, 16, 12, chip_id=c) for c in range(4)]
    dev = torch.device("cuda", 0)
    n, N = chips[0].grid.cell_count(), 12
    Td = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in chips]
    Qd = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in chips]
    Rd = [torch.empty(N, dtype=torch.float64, device=dev) for _ in chips]
    _, _, _, reps, _ = bk.generate_batch(chips, cfg_jacobi(), t_out=Td, q_out=Qd, resid_out=Rd,
                                         streams=4, ctx=ctx)
    torch.cuda.synchronize()
    for c, ch in enumerate(chips):
        o = oracle.assemble(grid_tuple(ch.grid), ch.k, ch.bc.as_tuples())
        X, _ = oracle.block_cg(o, oracle.rhs_from_power(o, ch.q_basis), TOL, 100000, 1)
        To, Qo, _ = oracle.combine_action(o, X, ch.coef)
        assert reps[c].all_converged()
        assert rel_l2(Td[c].cpu().numpy(), To) <= PARITY and rel_l2(Qd[c].cpu().numpy(), Qo) <= PARITY


def sub_budget(streams):
    import torch

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    return max(1, sms // streams)


@pytest.mark.parametrize("case", [(2, 64, 48, 1, 16), (1, 48, 40, 1, 8)])
def test_block_cg_row_ring_path_vs_oracle(bk, ctx, oracle, case):
    """Single-plane chips outside resident mode run phase 1 through the TMA row
    ring, with X += P alpha deferred to phase 3 (S = 16): capped iterates equal
    the oracle's, a full solve converges to it."""
    inp = bk.synth_chip(*case, 4)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    B = oracle.rhs_from_power(o, inp.q_basis)
    with ctx.options(no_resident=1):
        for m in (1, 2, 7):
            r = bk.block_cg(op, B, cfg_jacobi(m))
            X, rep = oracle.block_cg(o, B, TOL, m, 1)
            assert r.report.iterations == m and r.report.matvec_count == rep["matvec_count"]
            assert rel_l2(r.x, X) <= 1e-12
        r = bk.block_cg(op, B, cfg_jacobi())
    X, rep = oracle.block_cg(o, B, TOL, 100000, 1)
    assert r.report.all_converged() and rel_l2(r.x, X) <= PARITY


@pytest.mark.parametrize("case", [(1, 32, 32, 1, 8), (2, 40, 36, 1, 16), (3, 16, 16, 8, 32),
                                  (4, 24, 20, 4, 16)])
def test_block_cg_multikernel_path_vs_oracle(bk, ctx, oracle, case):
    """The one-kernel-per-phase engine (used for s > 32 / large grids and by the
    slab decomposition) forced on small cases: same solution as the oracle."""
    inp = bk.synth_chip(*case, 4)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples(), dz=inp.grid.dz)
    B = oracle.rhs_from_power(o, inp.q_basis)
    with ctx.options(force_large=1):
        r = bk.block_cg(op, B, cfg_jacobi())
        X, rep = oracle.block_cg(o, B, TOL, 100000, 1)
        assert r.report.all_converged() and rep["converged"].all()
        assert rel_l2(r.x, X) <= PARITY
        assert abs(r.report.iterations - rep["iterations"]) <= max(3, rep["iterations"] // 10)
        for m in (1, 3):
            rm = bk.block_cg(op, B, cfg_jacobi(m))
            Xm, repm = oracle.block_cg(o, B, TOL, m, 1)
            assert rm.report.iterations == m and rm.report.matvec_count == repm["matvec_count"]
            assert rel_l2(rm.x, Xm) <= 1e-12


@pytest.mark.parametrize("case", [(5, 48, 40, 16, 64), (3, 16, 16, 8, 32), (1, 32, 32, 1, 8)])
def test_block_cg_graph_loop_bitwise(bk, ctx, oracle, case):
    """Device-driven iterations (option graph_loop: the iteration as a CUDA
    graph body under a while-node, verifications handed back to the host) give
    bitwise the host-driven engine's X and report, full solve and capped."""
    inp = bk.synth_chip(*case, 4)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples(), dz=inp.grid.dz)
    B = oracle.rhs_from_power(o, inp.q_basis)
    for m in (1, 2, 7, 100000):
        cfg = cfg_jacobi(m) if m < 100000 else cfg_jacobi()
        with ctx.options(force_large=1):
            h = bk.block_cg(op, B, cfg)
        with ctx.options(force_large=1, graph_loop=1):
            g = bk.block_cg(op, B, cfg)
        assert np.array_equal(h.x, g.x), m
        assert h.report.iterations == g.report.iterations
        assert h.report.matvec_count == g.report.matvec_count
        assert np.array_equal(h.report.final_rel_residual, g.report.final_rel_residual)
    X, rep = oracle.block_cg(o, B, TOL, 100000, 1)
    assert g.report.all_converged() and rel_l2(g.x, X) <= PARITY


@pytest.mark.parametrize("case", [(5, 48, 40, 16, 64), (3, 16, 16, 8, 32), (2, 40, 36, 1, 16)])
def test_block_cg_lookahead_bitwise(bk, ctx, oracle, case):
    """The default lookahead loop of the multi-kernel engine (iteration m + 1
    enqueued with gated kernels before the host reads iteration m's control
    word) gives bitwise the synchronous loop's X and report: capped runs, and
    full solves through every verification."""
    inp = bk.synth_chip(*case, 4)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    o = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples(), dz=inp.grid.dz)
    B = oracle.rhs_from_power(o, inp.q_basis)
    for m in (1, 2, 7, 100000):
        cfg = cfg_jacobi(m) if m < 100000 else cfg_jacobi()
        with ctx.options(force_large=1, no_lookahead=1):
            h = bk.block_cg(op, B, cfg)
        with ctx.options(force_large=1):
            g = bk.block_cg(op, B, cfg)
        assert np.array_equal(h.x, g.x), m
        assert h.report.iterations == g.report.iterations
        assert h.report.matvec_count == g.report.matvec_count
        assert np.array_equal(h.report.final_rel_residual, g.report.final_rel_residual)
        assert np.array_equal(h.report.converged, g.report.converged)
    X, rep = oracle.block_cg(o, B, TOL, 100000, 1)
    assert g.report.all_converged() and rel_l2(g.x, X) <= PARITY


@pytest.mark.parametrize("case", [(5, 48, 40, 16, 64, 2), (5, 40, 36, 16, 64, 2)])
@pytest.mark.parametrize("nslabs", [2, 3])
def test_slab_lookahead_bitwise(bk, ctx, nslabs, case):
    """dd_block_cg's lookahead loop (BK_DD_GATED steps, asynchronous control
    reads) is bitwise its synchronous loop, with virtual ranks on one GPU."""
    import torch

    from paper_2510_23221_b200 import dd

    inp = bk.synth_chip(*case)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    dev = torch.device("cuda", 0)
    q = torch.from_numpy(inp.q_basis).to(dev)
    B = torch.empty_like(q)
    bk.rhs_from_power(op, q, out=B)
    parts = dd.partition_rows(inp.grid.ny, nslabs)
    for cfg in (cfg_jacobi(3), cfg_jacobi()):
        Xs, rs = dd.solve_decomposed(bk, ctx, op, B, cfg, parts, lookahead=False)
        Xl, rl = dd.solve_decomposed(bk, ctx, op, B, cfg, parts, lookahead=True)
        torch.cuda.synchronize()
        assert torch.equal(Xs, Xl)
        assert rs.iterations == rl.iterations and rs.matvec_count == rl.matvec_count
        assert np.array_equal(rs.final_rel_residual, rl.final_rel_residual)
    assert rl.all_converged()


@pytest.mark.parametrize("case", [(5, 48, 40, 16, 64, 2), (5, 40, 36, 16, 64, 2)])
@pytest.mark.parametrize("nslabs", [1, 2, 3])
def test_slab_decomposition_matches_single_gpu(bk, ctx, nslabs, case):
    """y-slab decomposition (config 5 structure: s = 64) with virtual ranks on
    one GPU (dd.LocalComm): same solution as the single-GPU solve; one slab is
    bitwise the single-GPU multi-kernel engine — on 16-aligned x the slab steps
    run the same warp-specialised sweeps with X deferred to the P update
    (bk_dd_deferred_x), otherwise the per-run sweeps with X in phase 2."""
    import torch

    from paper_2510_23221_b200 import dd

    inp = bk.synth_chip(*case)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    dev = torch.device("cuda", 0)
    q = torch.from_numpy(inp.q_basis).to(dev)
    B = torch.empty_like(q)
    bk.rhs_from_power(op, q, out=B)
    torch.cuda.synchronize()
    deferred = bool(bk._load().bk_dd_deferred_x(op.h, 64))
    assert deferred == (inp.grid.nx % 16 == 0)
    ref_ws = bk.block_cg(op, B.cpu().numpy(), cfg_jacobi())
    with ctx.options(no_ws_update=1, no_ws_spmm=1):
        ref_pr = bk.block_cg(op, B.cpu().numpy(), cfg_jacobi())
    assert rel_l2(ref_ws.x, ref_pr.x) <= PARITY
    ref = ref_ws if deferred else ref_pr
    parts = dd.partition_rows(inp.grid.ny, nslabs)
    X, rep = dd.solve_decomposed(bk, ctx, op, B, cfg_jacobi(), parts)
    torch.cuda.synchronize()
    Xh = X.cpu().numpy()
    assert rep.all_converged() and ref.report.all_converged()
    if nslabs == 1:
        assert np.array_equal(Xh, ref.x) and rep.iterations == ref.report.iterations
        assert rep.matvec_count == ref.report.matvec_count
    else:
        assert rel_l2(Xh, ref.x) <= PARITY
        assert abs(rep.iterations - ref.report.iterations) <= max(3, ref.report.iterations // 10)


# ------------------------------------------------------ device-side synthesis
@pytest.mark.parametrize("case", [(1, 40, 32, 1, 8, 6), (2, 48, 40, 1, 16, 5), (3, 24, 20, 8, 32, 4),
                                  (4, 32, 24, 4, 16, 8), (5, 16, 16, 16, 64, 3)])
def test_synth_chip_device_matches_host(bk, ctx, case):
    """the device generator evaluates the host generator's plan.
    Geometry, boundary, coefficients and the tile / layer k are bitwise; the
    blob maps and the lognormal k differ only through CUDA exp vs libm."""
    h = bk.synth_chip(*case, chip_id=5)
    d = bk.synth_chip_device(*case, chip_id=5, ctx=ctx)
    assert (h.grid.nx, h.grid.ny, h.grid.nz, h.grid.lz) == (d.grid.nx, d.grid.ny, d.grid.nz, d.grid.lz)
    assert h.bc.as_tuples() == d.bc.as_tuples()
    assert np.array_equal(h.coef, d.coef.cpu().numpy())
    kd, qd = d.k.cpu().numpy(), d.q_basis.cpu().numpy()
    if case[0] in (1, 2, 4):
        assert np.array_equal(h.k, kd)
    else:
        assert np.max(np.abs(kd - h.k) / h.k) <= 1e-15
    assert np.max(np.abs(qd - h.q_basis)) <= 1e-14 * np.max(np.abs(h.q_basis))
    assert np.array_equal(qd == 0.0, h.q_basis == 0.0)


def test_generate_from_device_synthesis(bk, ctx):
    """A config-4 chip generated straight from device-synthesised inputs:
    within tolerance of the host-synthesised chip's outputs."""
    import torch

    h = bk.synth_chip(4, 32, 24, 4, 16, 8, chip_id=2)
    d = bk.synth_chip_device(4, 32, 24, 4, 16, 8, chip_id=2, ctx=ctx)
    Th, Qh, Rh, reph, _ = bk.generate_chip(h.grid, h.k, h.bc, h.q_basis, h.coef, cfg_jacobi(), ctx=ctx)
    n = d.grid.cell_count()
    Td = torch.empty((8, n), dtype=torch.float64, device="cuda")
    Qd = torch.empty_like(Td)
    Rd = torch.empty(8, dtype=torch.float64, device="cuda")
    _, _, _, repd, _ = bk.generate_chip(d.grid, d.k, d.bc, d.q_basis, d.coef, cfg_jacobi(),
                                        t_out=Td, q_out=Qd, resid_out=Rd, ctx=ctx)
    torch.cuda.synchronize()
    assert repd.all_converged()
    assert rel_l2(Td.cpu().numpy(), Th) <= PARITY and rel_l2(Qd.cpu().numpy(), Qh) <= PARITY


@pytest.mark.parametrize("case,nslabs", [((5, 48, 40, 16, 64, 21), 1), ((5, 48, 40, 16, 64, 21), 3),
                                         ((3, 32, 24, 8, 32, 11), 2)])
def test_slab_local_combine_matches_global(bk, ctx, case, nslabs):
    """Config-5 multi-GPU outputs without gathering X: one X-halo exchange, then
    every slab forms all samples on its own rows (bk_dd_combine_action). Given
    the same X, each slab's T and q are bitwise the global kernel's rows; the
    per-sample residual from the summed (num, den) partials matches."""
    import torch

    from paper_2510_23221_b200 import dd

    inp = bk.synth_chip(*case)
    g = inp.grid
    op = bk.assemble(inp.k, g, inp.bc, ctx)
    dev = torch.device("cuda", 0)
    S = case[4]
    q = torch.from_numpy(inp.q_basis).to(dev)
    B = torch.empty_like(q)
    bk.rhs_from_power(op, q, out=B)
    X = torch.empty_like(q)
    bk.block_cg(op, B, cfg_jacobi(60), out=X)
    coef = torch.from_numpy(inp.coef).to(dev)
    N, n = inp.coef.shape[1], g.cell_count()
    T = torch.empty((N, n), dtype=torch.float64, device=dev)
    Q, R = torch.empty_like(T), torch.empty(N, dtype=torch.float64, device=dev)
    bk.combine_action(op, X, coef, t_out=T, q_out=Q, resid_out=R)
    slabs = dd.make_slabs(bk, ctx, op, S, dd.partition_rows(g.ny, nslabs))
    for sl in slabs:
        sl.load_x(X)
    Tl = [torch.full((N, sl.cells()), float("nan"), dtype=torch.float64, device=dev) for sl in slabs]
    Ql = [torch.full_like(t, float("nan")) for t in Tl]
    Rl = [torch.empty(N, dtype=torch.float64, device=dev) for _ in slabs]
    dd.slab_outputs(slabs, dd.LocalComm(), coef, Tl, Ql, Rl)
    torch.cuda.synchronize()
    Tg = T.cpu().numpy().reshape(N, g.nz, g.ny, g.nx)
    Qg = Q.cpu().numpy().reshape(N, g.nz, g.ny, g.nx)
    for sl, t, qq, r in zip(slabs, Tl, Ql, Rl):
        ts = t.cpu().numpy().reshape(N, g.nz, sl.nyl, g.nx)
        qs = qq.cpu().numpy().reshape(N, g.nz, sl.nyl, g.nx)
        assert np.array_equal(ts, Tg[:, :, sl.y0:sl.y0 + sl.nyl, :])
        assert np.array_equal(qs, Qg[:, :, sl.y0:sl.y0 + sl.nyl, :])
        rr, RR = r.cpu().numpy(), R.cpu().numpy()
        assert np.max(np.abs(rr - RR) / np.maximum(RR, 1e-300)) <= 1e-12


def test_measure_fp64_peak(bk, ctx):
    """bk_measure_fp64_peak (bench.py's live roofline denominator): a plausible
    B200 FP64 tensor rate, sustained not above burst."""
    burst, sustained = ctx.measure_fp64_peak(0.5)
    assert 20.0 < burst < 60.0, burst
    assert 0.5 * burst < sustained <= 1.02 * burst, (burst, sustained)


def test_generate_batch_64_chips_per_launch(bk, ctx, oracle):
    """bench.py's config-1 step: 64 chips z-stacked in ONE launch (2 CTAs per
    chip). The 64 solve reports (37 KiB) come back through the mapped-memory
    read in pieces — a 32 KiB cap there once made this configuration fail."""
    import torch

    chips = [bk.synth_chip(1, 16, 16, 1, 8, 4, chip_id=c) for c in range(64)]
    dev = torch.device("cuda", 0)
    n, N = chips[0].grid.cell_count(), 4
    Td = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in chips]
    Qd = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in chips]
    Rd = [torch.empty(N, dtype=torch.float64, device=dev) for _ in chips]
    _, _, _, reps, _ = bk.generate_batch(chips, cfg_jacobi(), t_out=Td, q_out=Qd, resid_out=Rd,
                                         streams=64, ctx=ctx)
    torch.cuda.synchronize()
    assert "chips=64" in ctx.last_solver_variant, ctx.last_solver_variant
    assert len(reps) == 64 and all(r.all_converged() for r in reps)
    for c in (0, 37, 63):
        ch = chips[c]
        o = oracle.assemble(grid_tuple(ch.grid), ch.k, ch.bc.as_tuples())
        X, orep = oracle.block_cg(o, oracle.rhs_from_power(o, ch.q_basis), TOL, 100000, 1)
        To, Qo, _ = oracle.combine_action(o, X, ch.coef)
        assert rel_l2(Td[c].cpu().numpy(), To) <= PARITY and rel_l2(Qd[c].cpu().numpy(), Qo) <= PARITY
