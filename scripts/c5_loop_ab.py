"""C5 multi-kernel solve: device-driven graph loop vs host-driven iterations.
Full solve at the bench tolerance (or capped: argv[1] = max_iter), bitwise X
comparison and ms per iteration:  python scripts/c5_loop_ab.py [max_iter] [opt=v ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_23221_b200 as bk  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
opts = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
ctx = bk.Context(0)
dev = torch.device("cuda", 0)
inp = bk.synth_chip(5, 512, 512, 16, 64, 16)
op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
q = torch.from_numpy(inp.q_basis).to(dev)
B = torch.empty_like(q)
bk.rhs_from_power(op, q, out=B)
X = torch.empty_like(q)
cfg = bk.SolverConfig(1e-10, it, "jacobi")
res = {}
for name, o in (("host", {}), ("graph", {"graph_loop": 1}), ("host+opts", opts)):
    if name == "host+opts" and not opts:
        continue
    with ctx.options(**o):
        for rep in range(2 if it < 100 else 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            r = bk.block_cg(op, B, cfg, out=X).report
            e1.record()
            torch.cuda.synchronize()
    res[name] = X.cpu().numpy()
    ms = e0.elapsed_time(e1)
    print(f"{name}: {ctx.last_solver_variant}: iters {r.iterations} matvecs {r.matvec_count} "
          f"{ms:.1f} ms = {ms / max(r.iterations, 1):.3f} ms/iter, bitwise vs host "
          f"{np.array_equal(res[name], res['host'])}, launches {ctx.launch_count}", flush=True)
