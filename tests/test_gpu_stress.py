"""Race / bounds stress on the hand-synchronised kernels (compute-sanitizer is
closed on this GPU pool: runs under it have left GPUs needing a reset, so the
pool refuses it — see profiles/r2_sanitizer.md).

Every output buffer is poisoned with NaN before each run and each kernel
variant is run repeatedly: a missed write leaves a NaN, a race (a TMA ring
slot refilled early, a group barrier passed early, a stale P row) changes bits
between runs. The kernels use no floating-point atomics and fixed-order
reductions, so repeated runs must agree bit for bit.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REPS = 4


def dev_chips(bk, cases):
    import torch
    from types import SimpleNamespace

    dev = torch.device("cuda", 0)
    out = []
    for c in cases:
        ch = bk.synth_chip(*c)
        out.append(SimpleNamespace(grid=ch.grid, bc=ch.bc, k=torch.from_numpy(ch.k).to(dev),
                                   q_basis=torch.from_numpy(ch.q_basis).to(dev),
                                   coef=torch.from_numpy(ch.coef).to(dev)))
    return out


def batch_runs(bk, ctx, cases, streams, tol=1e-12, it=100000, reps=REPS, **opts):
    import torch

    chips = dev_chips(bk, cases)
    dev = torch.device("cuda", 0)
    n, N = chips[0].grid.cell_count(), int(chips[0].coef.shape[1])
    outs = []
    with ctx.options(**opts):
        for _ in range(reps):
            T = [torch.full((N, n), float("nan"), dtype=torch.float64, device=dev) for _ in chips]
            Q = [torch.full((N, n), float("nan"), dtype=torch.float64, device=dev) for _ in chips]
            R = [torch.full((N,), float("nan"), dtype=torch.float64, device=dev) for _ in chips]
            bk.generate_batch(chips, bk.SolverConfig(tol, it, "jacobi"), T, Q, R, streams=streams,
                              ctx=ctx, check_converged=False)
            torch.cuda.synchronize()
            outs.append([(t.cpu().numpy(), q.cpu().numpy(), r.cpu().numpy())
                         for t, q, r in zip(T, Q, R)])
        variant = ctx.last_solver_variant
    for o in outs:
        for c in o:
            for arr in c:
                assert not np.isnan(arr).any(), variant
    for rep, o in enumerate(outs[1:], 1):
        for chip, (a, b) in enumerate(zip(o, outs[0])):
            for name, x, y in zip("TQR", a, b):
                bad = np.argwhere(x != y)
                assert bad.size == 0, (variant, f"rep {rep} chip {chip} {name}: {len(bad)} differ, "
                                                f"first at {bad[0].tolist()}")
    return variant


@pytest.mark.parametrize("cases,streams,opts,expect", [
    ([(2, 64, 48, 1, 16, 24, 1, c) for c in range(6)], 6, {"no_resident": 1},
     "block_cg_dmma_kernel<16,0,1,1> ring"),
    ([(2, 48, 40, 1, 16, 24, 1, c) for c in range(8)], 8, {}, "block_cg_dmma_kernel<16,1,1,0>"),
    ([(3, 32, 24, 8, 32, 20, 1, c) for c in range(3)], 3, {}, "block_cg_dmma_kernel<32,0,1,1>"),
    # deferred X, 3D, few cells per CTA: the true-residual sweep reads X halo
    # cells of up to ~12 other CTAs (a CTA-only barrier after the deferred X
    # update let it see stale ones; fixed with a group barrier)
    ([(3, 32, 24, 8, 32, 20, 1, c) for c in range(6)], 6, {"reps": 8},
     "block_cg_dmma_kernel<32,0,1,1>"),
    ([(4, 32, 24, 4, 16, 8, 1, c) for c in range(8)], 8, {"no_resident": 1},
     "block_cg_dmma_kernel<16,0,1,0>"),
    ([(2, 64, 48, 1, 16, 40, 1, c) for c in range(4)], 4, {"comb_one_role": 1},
     "block_cg_dmma_kernel<16,1,1,0>"),
])
def test_batched_solve_and_combine_repeatable(bk, ctx, cases, streams, opts, expect):
    variant = batch_runs(bk, ctx, cases, streams, **opts)
    assert variant.startswith(expect), variant


@pytest.mark.parametrize("opts", [{}, {"spmm_band": 1}, {"spmm_band": 2}, {"spmm_teams": 1},
                                  {"graph_loop": 1}, {"no_ws_update": 1, "no_ws_spmm": 1}])
def test_multikernel_s64_repeatable(bk, ctx, opts):
    """The S = 64 engine (warp-specialised TMA sweeps by default: y-banded
    role-split stencil sweep, producer-less update, register-resident control
    solves) on a reduced config-5 chip, every sweep variant: X bitwise equal
    over repeated solves, no NaN left."""
    import torch

    inp = bk.synth_chip(5, 48, 40, 16, 64, 2)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    dev = torch.device("cuda", 0)
    q = torch.from_numpy(inp.q_basis).to(dev)
    B = torch.empty_like(q)
    bk.rhs_from_power(op, q, out=B)
    xs = []
    with ctx.options(**opts):
        for _ in range(REPS):
            X = torch.full_like(q, float("nan"))
            r = bk.block_cg(op, B, bk.SolverConfig(1e-10, 40, "jacobi"), out=X)
            torch.cuda.synchronize()
            xs.append(X.cpu().numpy())
        variant = ctx.last_solver_variant
    assert r.report.iterations == 40
    assert not np.isnan(xs[0]).any()
    for x in xs[1:]:
        assert np.array_equal(x, xs[0]), variant


def test_stream_pipeline_repeatable(bk, ctx):
    ch = bk.synth_chip(3, 24, 20, 8, 32, 45)
    got = []
    for _ in range(3):
        acc = {}

        def sink(chip, j0, T, Q, R):
            acc[(chip, j0)] = (T.copy(), Q.copy(), R.copy())

        bk.generate_stream([ch, ch, ch], bk.SolverConfig(1e-12, 100000, "jacobi"), sink=sink,
                           chunk=8, ctx=ctx)
        got.append(acc)
    for acc in got[1:]:
        assert acc.keys() == got[0].keys()
        for key in acc:
            for a, b in zip(acc[key], got[0][key]):
                assert np.array_equal(a, b)


@pytest.mark.parametrize("cases,streams,opts", [
    ([(3, 32, 24, 8, 32, 20, 1, c) for c in range(6)], 6, {}),                    # 3D, S = 32
    ([(2, 64, 48, 1, 16, 24, 1, c) for c in range(6)], 6, {"no_resident": 1}),    # 2D row ring
])
def test_deferred_x_bitwise_the_phase2_update(bk, ctx, cases, streams, opts):
    """X += P alpha placed in phase 3 (deferred, the default for S = 32 and the
    row ring) or in phase 2 (option no_defer_x) is the same DMMA chain per
    element, so iterations, T and q must agree bit for bit. The deferred form
    reads X halo cells of other CTAs in a verification right after updating X:
    with only a CTA barrier there, a borderline column restarted instead of
    freezing and the two forms (and repeated runs) differed."""
    import torch

    chips = dev_chips(bk, cases)
    dev = torch.device("cuda", 0)
    n, N = chips[0].grid.cell_count(), int(chips[0].coef.shape[1])
    res = {}
    for name, extra in (("deferred", {}), ("phase2", {"no_defer_x": 1})):
        with ctx.options(**opts, **extra):
            T = [torch.full((N, n), float("nan"), dtype=torch.float64, device=dev) for _ in chips]
            Q = [torch.full((N, n), float("nan"), dtype=torch.float64, device=dev) for _ in chips]
            R = [torch.full((N,), float("nan"), dtype=torch.float64, device=dev) for _ in chips]
            _, _, _, reps, _ = bk.generate_batch(chips, bk.SolverConfig(1e-12, 100000, "jacobi"),
                                                 T, Q, R, streams=streams, ctx=ctx,
                                                 check_converged=False)
            torch.cuda.synchronize()
            res[name] = (ctx.last_solver_variant, [r.iterations for r in reps],
                         [r.matvec_count for r in reps], [t.cpu().numpy() for t in T],
                         [q.cpu().numpy() for q in Q])
    vd, vp = res["deferred"][0], res["phase2"][0]
    assert ",1,1>" in vd and ",1,0>" in vp, (vd, vp)
    assert res["deferred"][1] == res["phase2"][1] and res["deferred"][2] == res["phase2"][2]
    for c in range(len(chips)):
        assert np.array_equal(res["deferred"][3][c], res["phase2"][3][c]), c
        assert np.array_equal(res["deferred"][4][c], res["phase2"][4][c]), c
