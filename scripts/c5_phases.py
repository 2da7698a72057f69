"""Per-sweep device times of the C5 multi-kernel solve (capped iterations),
A/B over kernel-variant options:  python scripts/c5_phases.py [iters] [opt=v ...]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_23221_b200 as bk  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 20
opts = dict(a.split("=") for a in sys.argv[2:])
ctx = bk.Context(0)
dev = torch.device("cuda", 0)
inp = bk.synth_chip(5, 512, 512, 16, 64, 16)
op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
q = torch.from_numpy(inp.q_basis).to(dev)
B = torch.empty_like(q)
bk.rhs_from_power(op, q, out=B)
X = torch.empty_like(q)
ctx.set_option("phase_timing", 1)
ref = None
for variant in ({}, opts) if opts else ({},):
    with ctx.options(**{k: int(v) for k, v in variant.items()}):
        for rep in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = bk.block_cg(op, B, bk.SolverConfig(1e-10, it, "jacobi"), out=X)
            e1.record()
            torch.cuda.synchronize()
        ph = ctx.last_solve_phases()
        Xh = X.cpu().numpy()
        diff = None if ref is None else float(np.linalg.norm(Xh - ref) / np.linalg.norm(ref))
        if ref is None:
            ref = Xh
        print(f"{variant or 'default'} {ctx.last_solver_variant}: {e0.elapsed_time(e1) / it:.3f} ms/iter",
              {k: round(v["ms"] / max(v["launches"], 1), 3) for k, v in ph.items()},
              "matvecs", r.report.matvec_count, "rel diff vs first", diff,
              "sha", hashlib.sha256(Xh.tobytes()).hexdigest()[:16], flush=True)
