"""CPU tests: pin the oracle restatement (oracle/blockoa_oracle.c) to the
reference — golden fixtures from the unmodified reference, the reference itself
compiled from source (oracle/_ref, when present) and the SPEC.md examples."""
import hashlib
import zlib

import numpy as np
import pytest

from conftest import golden, grid_tuple, rel_l2

TOL = 1e-12


def csr_dense(rp, col, val, n):
    A = np.zeros((n, n))
    for i in range(n):
        for p in range(rp[i], rp[i + 1]):
            A[i, col[p]] = val[p]
    return A


# ----------------------------------------------------------------- assembly
def test_kat_3x3x3_center_row(oracle):
    """center row (4,-1)(10,-1)(12,-1)(13,6)(14,-1)(16,-1)(22,-1)."""
    op = oracle.assemble((3, 3, 3, 3.0, 3.0, 3.0), np.ones(27), [(0, 0.0, 0.0)] * 6)
    rp, col, val, g, vol = oracle.csr(op)
    row = list(zip(col[rp[13]:rp[14]].tolist(), val[rp[13]:rp[14]].tolist()))
    assert row == [(4, -1.0), (10, -1.0), (12, -1.0), (13, 6.0), (14, -1.0), (16, -1.0),
                   (22, -1.0)]
    # corner: 3 interior faces (1 each) + 3 Dirichlet half-cell faces (2 each)
    assert val[rp[0]:rp[1]][0] == 9.0
    kat = golden("kat_3x3x3.npz")
    for a, b in zip((rp, col, val, g, vol), (kat["row_ptr"], kat["col"], kat["val"], kat["g"],
                                             kat["vol"])):
        assert np.array_equal(a, b)


def test_mixed_operator_bitwise_vs_reference_golden(oracle):
    d = golden("mixed_operator.npz")
    bc = list(zip(d["bc_kind"].tolist(), d["bc_a"].tolist(), d["bc_b"].tolist()))
    op = oracle.assemble(tuple(d["grid"][:3].astype(int)) + tuple(d["grid"][3:]), d["k"], bc)
    rp, col, val, g, vol = oracle.csr(op)
    assert np.array_equal(rp, d["row_ptr"]) and np.array_equal(col, d["col"])
    assert np.array_equal(val, d["val"]) and np.array_equal(g, d["g"])
    assert np.array_equal(vol, d["vol"])
    A = csr_dense(rp, col, val, op.n)
    assert np.array_equal(A, A.T)  # SPEC.md:160 symmetric bitwise
    assert np.all(np.diag(A) > 0) and np.all(A - np.diag(np.diag(A)) <= 0)
    for s in (1, 4, 7, 16):
        y = oracle.apply_block(op, d[f"x{s}"])
        assert np.array_equal(y, d[f"y{s}"]), s


@pytest.mark.parametrize("shape", [(5, 4, 3), (9, 1, 1), (1, 7, 2), (6, 6, 1)])
@pytest.mark.parametrize("bcset", ["dirichlet", "robin", "adiabatic_mix"])
def test_assemble_oracle_vs_reference(oracle, reference, shape, bcset):
    rng = np.random.default_rng(zlib.crc32(repr((shape, bcset)).encode()))
    nx, ny, nz = shape
    grid = (nx, ny, nz, 1e-3 * nx, 2e-3 * ny, 0.3e-3 * nz)
    k = rng.uniform(1.0, 400.0, nx * ny * nz)
    bc = {"dirichlet": [(0, 50.0, 0.0)] * 6,
          "robin": [(1, 1e3, 25.0)] * 6,
          "adiabatic_mix": [(2, 0, 0), (2, 0, 0), (0, 30.0, 0), (2, 0, 0), (1, 1e2, 20.0),
                            (1, 1e4, 0.0)]}[bcset]
    a = oracle.csr(oracle.assemble(grid, k, bc))
    b = reference.csr(reference.assemble(grid, k, bc))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_nonuniform_dz_reduces_to_reference_when_equal(oracle, reference):
    rng = np.random.default_rng(3)
    k = rng.uniform(1, 400, 6 * 5 * 4)
    bc = [(2, 0, 0)] * 4 + [(1, 1e2, 0.0), (1, 1e4, 0.0)]
    grid = (6, 5, 4, 6e-3, 5e-3, 0.8e-3)
    a = oracle.csr(oracle.assemble(grid, k, bc, dz=[0.2e-3] * 4))
    b = reference.csr(reference.assemble(grid, k, bc))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_nonuniform_dz_series_conductance(oracle):
    """z-face between layers of different thickness = area/(da/2ka + db/2kb)."""
    k = np.array([2.0, 300.0])
    op = oracle.assemble((1, 1, 2, 1e-3, 1e-3, 3e-4), k, [(2, 0, 0)] * 6, dz=[1e-4, 2e-4])
    rp, col, val, g, vol = oracle.csr(op)
    gz = 1e-6 / (1e-4 / 4.0 + 2e-4 / 600.0)
    assert val[1] == -gz and val[2] == -gz
    assert np.allclose(vol, [1e-10, 2e-10], rtol=0, atol=1e-25)


def test_errors(oracle):
    from oracle.oracle import CheckerError

    with pytest.raises(CheckerError) as e:
        oracle.assemble((2, 2, 1, 1, 1, 1), np.array([1, 1, 0, 1.0]), [(0, 0, 0)] * 6)
    assert e.value.code == 4
    with pytest.raises(CheckerError) as e:
        oracle.assemble((2, 2, 1, 1, 1, 1), np.ones(4), [(1, 0.0, 0)] + [(0, 0, 0)] * 5)
    assert e.value.code == 5


def test_rhs_power_roundtrip(oracle):
    """power_from_rhs(rhs_from_power(q)) = q within 1e-14 (unit
    volumes, so V q and the lift g are of comparable size; with physical
    volumes ~1e-11 m^3 the round trip is limited by the cancellation g/(V q))."""
    rng = np.random.default_rng(5)
    op = oracle.assemble((7, 6, 3, 7.0, 6.0, 3.0), rng.uniform(1, 400, 126),
                         [(0, 50.0, 0)] * 4 + [(1, 1e4, 25.0)] * 2)
    q = rng.uniform(-1e6, 1e6, 126)
    back = oracle.power_from_rhs(op, oracle.rhs_from_power(op, q))
    assert np.max(np.abs(back - q) / np.abs(q)) <= 1e-14


# ----------------------------------------------------------------- solvers
def diag_csr(d):
    n = len(d)
    return np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.asarray(d, float)


def test_cg_diag23(oracle):
    """cg(diag(2,3), (2,3)) -> (1,1) in <= 2 iterations."""
    op = oracle.op_from_csr(*diag_csr([2.0, 3.0]))
    x, rep = oracle.cg(op, np.array([2.0, 3.0]), 1e-12, 100, 0)
    assert np.allclose(x, [1.0, 1.0], rtol=1e-14) and rep["iterations"] <= 2 and rep["converged"]


def test_cg_diag23_reference(reference):
    x, rep = reference.cg_csr(*diag_csr([2.0, 3.0]), np.array([2.0, 3.0]), 1e-12, 100, 0)
    assert np.allclose(x, [1.0, 1.0], rtol=1e-14) and rep["iterations"] <= 2


def test_block_cg_duplicate_columns(oracle):
    """duplicate columns: both solved, rank-deficient block handled."""
    op = oracle.op_from_csr(*diag_csr([2.0, 3.0]))
    B = np.array([[2.0, 2.0], [3.0, 3.0]])
    X, rep = oracle.block_cg(op, B, 1e-12, 100, 0)
    assert np.allclose(X, 1.0, rtol=1e-13) and rep["converged"].all()


def random_spd_csr(n, seed):
    rng = np.random.default_rng(seed)
    M = rng.standard_normal((n, n))
    A = M @ M.T + n * np.eye(n)
    rp = np.arange(0, n * n + 1, n, dtype=np.int64)
    col = np.tile(np.arange(n, dtype=np.int32), n)
    return A, rp, col, A.ravel().copy()


def test_random_spd_block_vs_cg(oracle):
    """100x100 SPD, s=5: every column within 10*tol of cg and
    block iterations <= max single-RHS iterations."""
    A, rp, col, val = random_spd_csr(100, 11)
    op = oracle.op_from_csr(rp, col, val)
    B = np.random.default_rng(12).standard_normal((100, 5))
    X, rep = oracle.block_cg(op, B, 1e-10, 1000, 0)
    its = []
    for j in range(5):
        x, r = oracle.cg(op, np.ascontiguousarray(B[:, j]), 1e-10, 1000, 0)
        its.append(r["iterations"])
        assert rel_l2(X[:, j], x) <= 10 * 1e-10
    assert rep["iterations"] <= max(its)
    xd = np.linalg.solve(A, B)
    assert rel_l2(X, xd) <= 100 * 1e-10  # SPEC.md:226 dense-oracle equivalence


def test_random_spd_reference_agrees(oracle, reference):
    A, rp, col, val = random_spd_csr(60, 21)
    B = np.random.default_rng(22).standard_normal((60, 4))
    X1, r1 = oracle.block_cg(oracle.op_from_csr(rp, col, val), B, 1e-10, 1000, 0)
    X2, r2 = reference.block_cg_csr(rp, col, val, B, 1e-10, 1000, 0)
    assert rel_l2(X1, X2) < 1e-9 and abs(r1["iterations"] - r2["iterations"]) <= 2


def test_s1_block_equals_cg(oracle):
    """s = 1 degenerates to CG."""
    rng = np.random.default_rng(7)
    op = oracle.assemble((8, 7, 3, 8e-3, 7e-3, 0.3e-3), rng.uniform(10, 150, 168),
                         [(2, 0, 0)] * 5 + [(1, 1e3, 0.0)])
    b = rng.uniform(0, 1e-3, 168)
    X, rb = oracle.block_cg(op, b[:, None].copy(), 1e-12, 10000, 1)
    x, rc = oracle.cg(op, b, 1e-12, 10000, 1)
    assert rel_l2(X[:, 0], x) <= 10 * 1e-12 and rb["converged"][0] == rc["converged"]


def test_cg_error_bound(oracle):
    assert oracle.cg_error_bound(100, 1, 1) == pytest.approx(1.6363636363636365, rel=1e-15)
    assert oracle.cg_error_bound(4, 2, 1) == pytest.approx(2.0 / 9.0, rel=1e-15)
    assert oracle.cg_error_bound(1, 5, 3) == 0.0
    from oracle.oracle import CheckerError
    with pytest.raises(CheckerError):
        oracle.cg_error_bound(0.5, 1, 1)


def test_operator_action_center_indicator(oracle):
    """27-cell, g = 0, unit volumes: q = center column of A."""
    op = oracle.assemble((3, 3, 3, 3.0, 3.0, 3.0), np.ones(27), [(0, 0.0, 0.0)] * 6)
    x = np.zeros(27)
    x[13] = 1.0
    T, Q, R = oracle.combine_action(op, x[:, None].copy(), np.ones((1, 1)))
    assert Q[0, 13] == 6.0 and all(Q[0, i] == -1.0 for i in (4, 10, 12, 14, 16, 22))
    assert R[0] == 0.0


def test_manufactured_second_order(oracle):
    """manufactured solution, second-order convergence."""
    errs = []
    for m in (8, 16, 32):
        L = 1.0
        h = L / m
        c = (np.arange(m) + 0.5) * h
        X, Y, Z = np.meshgrid(c, c, c, indexing="ij")
        u = np.sin(np.pi * X) * np.sin(np.pi * Y) * np.sin(np.pi * Z)
        q = 3 * np.pi ** 2 * u
        uf = u.transpose(2, 1, 0).ravel()  # flat = ix + nx*(iy + ny*iz)
        qf = q.transpose(2, 1, 0).ravel()
        op = oracle.assemble((m, m, m, L, L, L), np.ones(m ** 3), [(0, 0.0, 0.0)] * 6)
        b = oracle.rhs_from_power(op, qf)
        x, rep = oracle.cg(op, b, 1e-12, 10000, 1)
        errs.append(np.max(np.abs(x - uf)))
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.0 <= r1 <= 5.0 and 3.0 <= r2 <= 5.0, errs


# ----------------------------------------------------------------- pipeline goldens
@pytest.mark.parametrize("name", ["c1_full", "c2_reduced", "c3_reduced", "c5_reduced"])
def test_pipeline_oracle_vs_reference_golden(oracle, bk, name):
    d = golden(f"{name}.npz")
    cfg, (nx, ny, nz, s, N) = int(d["config"]), d["shape"].tolist()
    inp = bk.synth_chip(cfg, nx, ny, nz, s, N)
    h = hashlib.sha256()
    for a in (inp.k, inp.q_basis, inp.coef):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == str(d["input_sha256"]), "input generator drifted"
    op = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    B = oracle.rhs_from_power(op, inp.q_basis)
    X, rep = oracle.block_cg(op, B, TOL, 100000, 1)
    assert rep["converged"].all() and d["converged"].all()
    assert rel_l2(X, d["X"]) <= 1e-9
    assert abs(rep["iterations"] - int(d["iterations"])) <= max(3, int(d["iterations"]) // 10)
    keep = d["keep"]
    T, Q, R = oracle.combine_action(op, d["X"], inp.coef)
    # same X -> combine + action bitwise equal to the reference
    assert np.array_equal(T[keep], d["T"]) and np.array_equal(Q[keep], d["Q"])
    assert np.max(R) <= 1e-12 and np.max(d["resid"]) <= 1e-12


def test_rng_bit_exact(oracle, bk):
    for tag, idx in (("chip", 0), ("basis", 17), ("coef", 0)):
        seed = bk.derive_seed(1, tag, idx)
        assert seed == oracle.derive_seed(1, tag, idx)
        assert np.array_equal(bk.rng_u64(seed, 257), oracle.rng_u64(seed, 257))
        assert np.array_equal(bk.rng_normal(seed, 257), oracle.rng_normal(seed, 257))
        assert np.array_equal(bk.rng_uniform(seed, 2, 8, 257), oracle.rng_uniform(seed, 2, 8, 257))


def test_rng_bit_exact_reference(reference, bk):
    seed = bk.derive_seed(1, "lognormal", 0)
    assert seed == reference.derive_seed(1, "lognormal", 0)
    assert np.array_equal(bk.rng_normal(seed, 1001), reference.rng_normal(seed, 1001))
    assert np.array_equal(bk.rng_u64(seed, 99), reference.rng_u64(seed, 99))


def test_block_cg_deterministic(oracle, bk):
    inp = bk.synth_chip(1, 32, 32, 1, 8, 4)
    op = oracle.assemble(grid_tuple(inp.grid), inp.k, inp.bc.as_tuples())
    B = oracle.rhs_from_power(op, inp.q_basis)
    X1, r1 = oracle.block_cg(op, B, TOL, 10000, 1)
    X2, r2 = oracle.block_cg(op, B, TOL, 10000, 1)
    assert np.array_equal(X1, X2) and r1["iterations"] == r2["iterations"]


def test_reference_block_cg_breaks_down_with_shared_lift(reference, bk):
    """Documented pin: with a non-zero ambient on the Robin
    faces every RHS is dominated by the shared lift g; the reference block CG
    then fails to converge (this is why the BASELINE inputs use u_inf = 0)."""
    inp = bk.synth_chip(4, 32, 32, 4, 16, 1)
    bc = [(k, a, 25.0 if k == 1 else b) for (k, a, b) in inp.bc.as_tuples()]
    dz = inp.grid.dz
    assert dz is not None
    # uniform-dz stand-in so the reference can assemble it
    g = (32, 32, 4, inp.grid.lx, inp.grid.ly, 4 * float(np.mean(dz)))
    op = reference.assemble(g, inp.k, bc)
    B = np.stack([reference.rhs_from_power(op, inp.q_basis[:, t]) for t in range(16)], axis=1)
    X, rep = reference.block_cg(op, B, TOL, 400, 1)
    assert not rep["converged"].all()
    bc0 = [(k, a, 0.0) for (k, a, b) in bc]
    op0 = reference.assemble(g, inp.k, bc0)
    B0 = np.stack([reference.rhs_from_power(op0, inp.q_basis[:, t]) for t in range(16)], axis=1)
    X0, rep0 = reference.block_cg(op0, B0, TOL, 400, 1)
    assert rep0["converged"].all()


@pytest.mark.parametrize("case", [(1, 64, 64, 1, 8, 256), (2, 48, 40, 1, 16, 12),
                                  (3, 24, 20, 8, 32, 7), (4, 32, 24, 4, 16, 8),
                                  (5, 32, 16, 16, 64, 5), (2, 256, 256, 1, 16, 2048)])
def test_oracle_synth_bitwise_product_synth(oracle, bk, case):
    """The checker-side input generator (orc_synth_chip, used by bench.py's
    reference arm so it never loads the product) draws bitwise the same chip as
    the product's host generator bk_synth_chip, for every BASELINE config."""
    for chip_id in (0, 7):
        o = oracle.synth_chip(*case, chip_id=chip_id)
        p = bk.synth_chip(*case, chip_id=chip_id)
        g = p.grid
        assert o.grid == (g.nx, g.ny, g.nz, g.lx, g.ly, g.lz)
        assert (o.dz is None) == (g.dz is None)
        if o.dz is not None:
            assert np.array_equal(o.dz, g.dz)
        assert o.bc == tuple(p.bc.as_tuples())
        for a, b in ((o.k, p.k), (o.q_basis, p.q_basis), (o.coef, p.coef)):
            assert a.shape == b.shape and np.array_equal(a, b)


def test_reference_cg_stalls_at_fp64_floor_on_c2_direct_columns(reference, oracle):
    """SURVEY §8(f4) direct baseline: a lone C2 sample column (power map
    Q c_j) does not reach rel_tol 1e-12 under the reference's own cg
    (solvers.cpp:82-171) either — it plateaus at ~1.2e-12 (measured: still
    unconverged after 100000 iterations) — so the GPU direct-CG leg stopping
    at max_iter on these columns is the reference's behaviour, not a bug."""
    ch = oracle.synth_chip(2, 256, 256, 1, 16, 2, chip_id=0)
    op = reference.assemble(ch.grid, ch.k, ch.bc)
    b = reference.rhs_from_power(op, ch.q_basis @ ch.coef[:, 0])
    _, rep = reference.cg(op, b, 1e-12, 5000, 1)
    assert not rep["converged"] and rep["iterations"] == 5000
    assert 1e-12 < rep["final_rel_residual"] < 2e-12


@pytest.mark.parametrize("name,case", [("c3_full.npz", (3, 128, 128, 8, 32, 5000, 0)),
                                       ("c4_full.npz", (4, 128, 128, 4, 16, 8, 0)),
                                       ("c4_full.npz", (4, 128, 128, 4, 16, 8, 4)),
                                       ("c5_capped.npz", (5, 512, 512, 16, 64, 5000, 0)),
                                       ("c5_full_cg.npz", (5, 512, 512, 16, 64, 5000, 0))])
def test_full_size_golden_inputs_match_generator(oracle, name, case):
    """The full-size goldens were computed on the generator's current bytes."""
    d = golden(name)
    ch = oracle.synth_chip(*case[:6], chip_id=case[6])
    h = hashlib.sha256()
    for a in (ch.k, ch.q_basis, ch.coef):
        h.update(np.ascontiguousarray(a).tobytes())
    key = "input_sha256" if name != "c4_full.npz" else f"chip{case[6]}_input_sha256"
    assert h.hexdigest() == str(d[key])
