"""Dataset sink and validation against the reference's own
dataset_io.cpp (oracle/_ref):

CPU: field_digest bit-exact (product, oracle, reference); datasets written by
our writer match the reference's write_dataset for the same samples (payloads
byte-identical, manifest text identical up to the bundled json library's
integer-array layout) and are read back by the reference; our
reader accepts the reference's files; error behaviour (ExistsError,
CorruptManifestError, SizeMismatchError, staged-directory cleanup).

GPU: bk_residuals vs the reference relative_residual (host-staged and device
inputs, several staging chunks, zero-denominator edges); a chip generated on
the GPU, drained from HBM into a dataset by the writer, validates with the
reference's validate_dataset and with ours (same verdicts, residuals within
1e-10 relative); digest tampering fails in both."""
import json
import os
import re

import numpy as np
import pytest

from conftest import grid_tuple


def _bc(bk):
    return bk.BoundarySpec([bk.Dirichlet(20.0), bk.Adiabatic(), bk.Robin(50.0, 25.0),
                            bk.Adiabatic(), bk.Adiabatic(), bk.Robin(1e3, 25.0)])


def _samples(grid, n_data, seed=0, groups=2):
    rng = np.random.default_rng(seed)
    n = grid.cell_count()
    ks = [rng.uniform(1.0, 400.0, n) for _ in range(groups)]
    ids = [j * groups // n_data for j in range(n_data)]
    k = np.stack([ks[i] for i in ids])
    q = rng.uniform(0.0, 1e6, (n_data, n))
    u = rng.uniform(20.0, 90.0, (n_data, n))
    return k, q, u, [100 + i for i in ids]


def _inline_int_arrays(text):
    """The nlohmann/json this image bundles (cudnn_frontend's copy of 3.11.3,
    used to build oracle/_ref because the reference's vendor/ is absent) is
    patched to print integer arrays on one line; upstream 3.11.3, which the
    reference pins and our writer follows, prints one element per line."""
    pat = re.compile(r"\[\n(?:[ ]+-?\d+,\n)*[ ]+-?\d+\n[ ]*\]")
    return pat.sub(lambda m: "[" + ",".join(re.findall(r"-?\d+", m.group(0))) + "]", text)


def _files(d):
    return {f: open(os.path.join(d, f), "rb").read()
            for f in ("manifest.json", "k.bin", "q.bin", "u.bin")}


# ---------------------------------------------------------------- CPU
def test_field_digest_bit_exact(bk, oracle, reference):
    rng = np.random.default_rng(3)
    for dims in ((1, 1, 1), (7, 5, 3), (64, 64, 1), (33, 17, 4)):
        v = rng.uniform(-1e3, 1e3, int(np.prod(dims)))
        g = bk.GridSpec(*dims)
        d = bk.field_digest(v, g)
        assert d == oracle.field_digest(dims, v) == reference.field_digest(dims, v)
    # shape is part of the digest
    v = rng.uniform(0, 1, 12)
    assert bk.field_digest(v, bk.GridSpec(3, 4, 1)) != bk.field_digest(v, bk.GridSpec(4, 3, 1))


def test_oracle_relative_residual_bit_exact(oracle, reference):
    # pins the rounding the GPU residual kernel must reproduce per cell:
    # CsrMatrix::apply and norm2 uncontracted, rhs_from_power contracted
    rng = np.random.default_rng(9)
    grid = (20, 16, 3, 0.01, 0.008, 0.001)
    bc = [(0, 20.0, 0.0), (2, 0.0, 0.0), (1, 50.0, 25.0), (2, 0.0, 0.0), (2, 0.0, 0.0),
          (1, 1e3, 25.0)]
    k = rng.uniform(1.0, 400.0, 960)
    oo, rr = oracle.assemble(grid, k, bc), reference.assemble(grid, k, bc)
    for _ in range(20):
        u, q = rng.uniform(20.0, 90.0, 960), rng.uniform(0.0, 1e6, 960)
        assert oracle.relative_residual(oo, u, q) == reference.relative_residual(rr, u, q)


def test_writer_byte_identical_to_reference(bk, reference, tmp_path):
    grid = bk.GridSpec(12, 9, 3, 0.012, 0.009, 0.00045)
    k, q, u, ids = _samples(grid, 7)
    bc = _bc(bk)
    digests = []
    for i in sorted(set(ids)):
        digests.append((i, bk.field_digest(k[ids.index(i)], grid)))
    timings = bk.ManifestTimings(1.25, 0.0625, 3e-5, 0.0, 1.5e15, 431, 6897)
    m = bk.DatasetManifest(method="blockoa", n_data=7, master_seed=1, floorplan_ids=ids,
                           floorplan_digests=digests, timings=timings,
                           residual_tol_claimed=1e-12, tool_version="blockoa-0.1.0",
                           requested_n_data=9, dropped_count=2)
    ours = tmp_path / "ours"
    summ = bk.write_dataset(bk.Dataset(grid, bc, k, q, u, m), str(ours))
    assert summ.n_data == 7 and summ.payload_bytes_per_file == 7 * grid.cell_count() * 8
    ref = tmp_path / "ref"
    st = reference.write_dataset(ref, grid_tuple(grid), bc.as_tuples(), k, q, u, ids,
                                 master_seed=1, digests=digests,
                                 timings=(1.25, 0.0625, 3e-5, 0.0, 1.5e15), counters=(431, 6897),
                                 requested=9, dropped=2)
    assert st == 0
    a, b = _files(ours), _files(ref)
    for f in ("k.bin", "q.bin", "u.bin"):
        assert a[f] == b[f], f
    ma, mb = a["manifest.json"].decode(), b["manifest.json"].decode()
    assert json.loads(ma) == json.loads(mb)
    # text identical up to the bundled json library's integer-array layout
    # (float formatting, key order, indentation, trailing newline all equal)
    assert _inline_int_arrays(ma) == mb
    # and the reference reads ours back
    st, dims, ext, rk, rq, ru, rids = reference.read_dataset(ours)
    assert st == 0 and dims == (12, 9, 3)
    assert np.array_equal(rk, k) and np.array_equal(rq, q) and np.array_equal(ru, u)
    assert list(rids) == ids
    assert not [p for p in os.listdir(tmp_path) if ".tmp-" in p]


def test_reader_reads_reference_dataset(bk, reference, tmp_path):
    grid = bk.GridSpec(8, 6, 2, 1.0, 0.75, 0.25)
    k, q, u, ids = _samples(grid, 5, seed=1)
    bc = _bc(bk)
    d = tmp_path / "ref"
    assert reference.write_dataset(d, grid_tuple(grid), bc.as_tuples(), k, q, u, ids,
                                   master_seed=7) == 0
    ds = bk.read_dataset(str(d))
    assert (ds.grid.nx, ds.grid.ny, ds.grid.nz) == (8, 6, 2)
    assert ds.manifest.n_data == 5 and ds.manifest.master_seed == 7
    assert ds.manifest.floorplan_ids == ids
    assert np.array_equal(ds.k, k) and np.array_equal(ds.q, q) and np.array_equal(ds.u, u)
    # adiabatic faces come back as the reference's Robin{1e-300, 0}
    assert ds.bc.faces[1] == bk.Robin(1e-300, 0.0)
    assert ds.bc.faces[0] == bk.Dirichlet(20.0)


def test_exists_overwrite_and_abort(bk, reference, tmp_path):
    grid = bk.GridSpec(4, 4, 1)
    k, q, u, ids = _samples(grid, 2, seed=2, groups=1)
    m = bk.DatasetManifest(n_data=2, floorplan_ids=ids)
    ds = bk.Dataset(grid, _bc(bk), k, q, u, m)
    d = str(tmp_path / "ds")
    bk.write_dataset(ds, d)
    with pytest.raises(bk.ExistsError):
        bk.write_dataset(ds, d)
    # the reference agrees (ExistsError = status 10)
    assert reference.write_dataset(d, grid_tuple(grid), _bc(bk).as_tuples(), k, q, u, ids) == 10
    ds.u = u + 1.0
    bk.write_dataset(ds, d, overwrite=True)
    assert np.array_equal(bk.read_dataset(d).u, u + 1.0)
    # an uncommitted writer leaves nothing behind
    e = str(tmp_path / "aborted")
    with bk.DatasetWriter(e, grid, _bc(bk)) as w:
        w.append(k[0], q[:1], u[:1], 5)
    assert not os.path.exists(e)
    assert not [p for p in os.listdir(tmp_path) if ".tmp-" in p]
    with pytest.raises(bk.DimensionMismatchError):
        with bk.DatasetWriter(e, grid, _bc(bk)) as w:
            w.append(k[0], q[:1, :5], u[:1], 5)


def test_reader_errors_match_reference(bk, reference, tmp_path):
    grid = bk.GridSpec(5, 4, 1)
    k, q, u, ids = _samples(grid, 3, seed=4, groups=1)
    good = str(tmp_path / "good")
    bk.write_dataset(bk.Dataset(grid, _bc(bk), k, q, u,
                                bk.DatasetManifest(n_data=3, floorplan_ids=ids)), good)

    def variant(name, edit=None, truncate=None, drop=None):
        d = tmp_path / name
        os.makedirs(d)
        for f, data in _files(good).items():
            if f == drop:
                continue
            if f == "manifest.json" and edit:
                j = json.loads(data)
                edit(j)
                data = json.dumps(j).encode()
            if f == truncate:
                data = data[:-8]
            open(d / f, "wb").write(data)
        return str(d)

    cases = [
        (variant("nomanifest", drop="manifest.json"), bk.CorruptManifestError, 11),
        (variant("badver", edit=lambda j: j.update(format_version=2)), bk.CorruptManifestError, 11),
        (variant("nokey", edit=lambda j: j.pop("tool_version")), bk.CorruptManifestError, 11),
        (variant("ids", edit=lambda j: j.update(floorplan_ids=[1])), bk.CorruptManifestError, 11),
        (variant("bctype", edit=lambda j: j["bc"]["xlo"].update(type="neumann")),
         bk.CorruptManifestError, 11),
        (variant("short", truncate="q.bin"), bk.SizeMismatchError, 12),
        (variant("missing", drop="u.bin"), bk.SizeMismatchError, 12),
    ]
    for d, exc, code in cases:
        with pytest.raises(exc):
            bk.read_dataset(d)
        assert reference.read_dataset(d)[0] == code, d


# ---------------------------------------------------------------- GPU
def _c1_chip(bk, nx=64, ny=64, N=64):
    ins = bk.synth_chip(1, nx, ny, 1, 8, N, master_seed=1, chip_id=0)
    return ins


@pytest.mark.gpu
def test_residuals_vs_reference(bk, ctx, reference):
    import torch

    grid = bk.GridSpec(40, 30, 5, 0.01, 0.0075, 0.001)
    rng = np.random.default_rng(5)
    k = rng.uniform(1.0, 400.0, grid.cell_count())
    bc = _bc(bk)
    op = bk.assemble(k, grid, bc, ctx)
    rop = reference.assemble(grid_tuple(grid), k, bc.as_tuples())
    N = 21
    u = rng.uniform(20.0, 90.0, (N, grid.cell_count()))
    q = rng.uniform(0.0, 1e6, (N, grid.cell_count()))
    want = np.array([reference.relative_residual(rop, u[j], q[j]) for j in range(N)])
    got_host = bk.relative_residual(op, u, q)
    got_dev = bk.relative_residual(op, torch.from_numpy(u).cuda(), torch.from_numpy(q).cuda())
    assert np.array_equal(got_host, got_dev)
    np.testing.assert_allclose(got_host, want, rtol=1e-12, atol=0)
    assert bk.relative_residual(op, u[3], q[3]) == got_host[3]
    # zero denominator (b = 0): 0 for u = 0, +inf otherwise (discretize.cpp:283-284)
    gz = bk.GridSpec(6, 5, 2)
    bz = bk.BoundarySpec.uniform_dirichlet(0.0)
    opz = bk.assemble(np.ones(gz.cell_count()), gz, bz, ctx)
    zero = np.zeros((2, gz.cell_count()))
    uz = zero.copy()
    uz[1, 7] = 1.0
    r = bk.relative_residual(opz, uz, zero)
    assert r[0] == 0.0 and np.isinf(r[1])


@pytest.mark.gpu
def test_residuals_several_staging_chunks(bk, ctx, reference):
    # 160 samples of 65,536 cells = 2 x 80 MiB of host input: two 128 MiB
    # pinned chunks (U and Q of 64 samples each ... ) through the overlap path
    grid = bk.GridSpec(256, 256, 1, 0.01, 0.01, 1.5e-4)
    rng = np.random.default_rng(6)
    k = rng.uniform(10.0, 150.0, grid.cell_count())
    bc = bk.BoundarySpec([bk.Adiabatic()] * 5 + [bk.Robin(1e3, 25.0)])
    op = bk.assemble(k, grid, bc, ctx)
    rop = reference.assemble(grid_tuple(grid), k, bc.as_tuples())
    N = 160
    u = rng.uniform(20.0, 90.0, (N, grid.cell_count()))
    q = rng.uniform(0.0, 1e6, (N, grid.cell_count()))
    got = bk.relative_residual(op, u, q)
    idx = [0, 1, 63, 64, 127, 128, 129, 159]
    want = np.array([reference.relative_residual(rop, u[j], q[j]) for j in idx])
    np.testing.assert_allclose(got[idx], want, rtol=1e-12, atol=0)


@pytest.mark.gpu
def test_generated_chip_to_dataset_validates(bk, ctx, reference, tmp_path):
    import torch

    ins = _c1_chip(bk)
    cfg = bk.SolverConfig(1e-12, 100000, "jacobi")
    n, N = ins.grid.cell_count(), ins.coef.shape[1]
    T = torch.empty((N, n), dtype=torch.float64, device="cuda")
    Q = torch.empty_like(T)
    R = torch.empty(N, dtype=torch.float64, device="cuda")
    ins2 = bk.synth_chip(1, 64, 64, 1, 8, 32, master_seed=1, chip_id=1)
    T2 = torch.empty((32, n), dtype=torch.float64, device="cuda")
    Q2 = torch.empty_like(T2)
    R2 = torch.empty(32, dtype=torch.float64, device="cuda")
    bk.generate_chip(ins.grid, ins.k, ins.bc, ins.q_basis, ins.coef, cfg, T, Q, R, ctx=ctx)
    bk.generate_chip(ins2.grid, ins2.k, ins2.bc, ins2.q_basis, ins2.coef, cfg, T2, Q2, R2,
                     ctx=ctx)
    d = str(tmp_path / "c1")
    with bk.DatasetWriter(d, ins.grid, ins.bc, master_seed=1, ctx=ctx) as w:
        w.append(torch.from_numpy(ins.k).cuda(), Q, T, 0)
        w.append(ins2.k, Q2, T2, 1)
        w.commit(bk.ManifestTimings(basis_solve_s=0.01))
    ds = bk.read_dataset(d)
    assert ds.manifest.n_data == N + 32
    assert np.array_equal(ds.u[:N], T.cpu().numpy()) and np.array_equal(ds.q[N:], Q2.cpu().numpy())
    assert np.array_equal(ds.k[N + 5], ins2.k)
    st, p, f, mx, rres = reference.validate_dataset(d, 1e-12)
    assert st == 0 and (p, f) == (N + 32, 0)
    ours = bk.validate_dataset(d, 1e-12, ctx)
    assert (ours.pass_count, ours.fail_count) == (p, f)
    # residuals ~1e-16: the per-cell r_i are bitwise the reference's, only the
    # two norms are summed in another order
    np.testing.assert_allclose(ours.residuals, rres, rtol=1e-10, atol=0)
    np.testing.assert_allclose(ours.max_residual, mx, rtol=1e-10)
    # against the pipeline's own per-sample residual as well
    assert np.all(ours.residuals <= 1e-12)

    # tamper with chip 1's digest: its samples fail with +inf in both
    j = json.load(open(os.path.join(d, "manifest.json")))
    j["floorplan_digests"][1]["k_digest"] ^= 1
    open(os.path.join(d, "manifest.json"), "w").write(json.dumps(j))
    st, p, f, mx, rres = reference.validate_dataset(d, 1e-12)
    ours = bk.validate_dataset(d, 1e-12, ctx)
    assert st == 0 and (p, f) == (N, 32) and np.isinf(mx)
    assert (ours.pass_count, ours.fail_count) == (p, f) and np.isinf(ours.max_residual)
    assert np.all(np.isinf(ours.residuals[N:])) and np.all(np.isinf(rres[N:]))


@pytest.mark.gpu
def test_writer_device_drain_several_chunks(bk, ctx, tmp_path):
    import torch

    # 300 x 65,536 doubles = 150 MiB per field: two pinned chunks per field
    grid = bk.GridSpec(256, 256, 1)
    n = grid.cell_count()
    g = torch.Generator(device="cuda").manual_seed(0)
    Q = torch.rand((300, n), dtype=torch.float64, device="cuda", generator=g)
    T = torch.rand((300, n), dtype=torch.float64, device="cuda", generator=g)
    k = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) + 1.0
    d = str(tmp_path / "big")
    with bk.DatasetWriter(d, grid, bk.BoundarySpec.uniform_dirichlet(0.0), ctx=ctx) as w:
        w.append(k, Q, T, 3)
        w.commit()
    ds = bk.read_dataset(d)
    assert np.array_equal(ds.q, Q.cpu().numpy()) and np.array_equal(ds.u, T.cpu().numpy())
    assert np.array_equal(ds.k[299], k.cpu().numpy())
    assert ds.manifest.floorplan_digests == [(3, bk.field_digest(k, grid))]
