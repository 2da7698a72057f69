"""Small runs of every kernel instantiation, for compute-sanitizer
(memcheck / racecheck / synccheck). Each case is capped to a few iterations so
the instrumented run stays short; the sanitizer reports hazards, not results.

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_23221_b200 as bk  # noqa: E402

ctx = bk.Context(0)
dev = torch.device("cuda", 0)
IT = int(os.environ.get("BK_SAN_ITERS", "12"))


def cfg(tol=1e-12, it=IT):
    return bk.SolverConfig(tol, it, "jacobi")


def dchips(cases):
    from types import SimpleNamespace
    out = []
    for c in cases:
        ch = bk.synth_chip(*c)
        out.append(SimpleNamespace(grid=ch.grid, bc=ch.bc, k=torch.from_numpy(ch.k).to(dev),
                                   q_basis=torch.from_numpy(ch.q_basis).to(dev),
                                   coef=torch.from_numpy(ch.coef).to(dev)))
    return out


def batch(cases, streams, **opts):
    ch = dchips(cases)
    n, N = ch[0].grid.cell_count(), int(ch[0].coef.shape[1])
    T = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in ch]
    Q = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in ch]
    R = [torch.empty(N, dtype=torch.float64, device=dev) for _ in ch]
    with ctx.options(**opts):
        bk.generate_batch(ch, cfg(), T, Q, R, streams=streams, ctx=ctx, check_converged=False)
        torch.cuda.synchronize()
        print("batch", ctx.last_solver_variant, flush=True)


def single(case, tol=1e-12, **opts):
    ch = bk.synth_chip(*case)
    with ctx.options(**opts):
        T, Q, R, rep, _ = bk.generate_chip(ch.grid, ch.k, ch.bc, ch.q_basis, ch.coef, cfg(tol),
                                           ctx=ctx, check_converged=False)
        print("single", ctx.last_solver_variant, rep.iterations, flush=True)


single((1, 48, 40, 1, 8, 6))                                  # <8,1,0,0>
single((2, 64, 48, 1, 16, 6), no_resident=1)                  # <16,0,0,1> ring
single((3, 16, 16, 8, 32, 6))                                 # <32,0,0,1>
batch([(2, 48, 40, 1, 16, 6, 1, c) for c in range(4)], 4)     # <16,1,1,0>
batch([(2, 64, 48, 1, 16, 6, 1, c) for c in range(2)], 2, no_resident=1)  # <16,0,1,1> ring
batch([(3, 16, 16, 8, 32, 6, 1, c) for c in range(2)], 2)     # <32,0,1,1>
batch([(4, 24, 20, 4, 16, 6, 1, c) for c in range(4)], 4, no_resident=1)  # <16,0,1,0>
single((5, 16, 16, 16, 64, 6), tol=1e-10)                     # block_cg_large<64> tma
single((3, 16, 16, 8, 32, 6), force_large=1)                  # block_cg_large<32>
ch = bk.synth_chip(1, 32, 32, 1, 8, 40)
bk.generate_stream([ch, ch], cfg(), sink=None, chunk=16, ctx=ctx, check_converged=False)
print("stream ok", flush=True)
bk.generate_blockoa(bk.GenerationConfig.default_run_config(), ctx=ctx)
print("generate_blockoa ok", flush=True)
torch.cuda.synchronize()
print("SANITIZE CASES DONE")
