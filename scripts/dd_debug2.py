import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_23221_b200 as bk
from paper_2510_23221_b200 import dd
ctx = bk.Context(0)
inp = bk.synth_chip(5, 48, 40, 16, 64, 2)
op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
dev = torch.device("cuda", 0)
q = torch.from_numpy(inp.q_basis).to(dev)
B = torch.empty_like(q); bk.rhs_from_power(op, q, out=B); torch.cuda.synchronize()
Bh = B.cpu().numpy()
for mi in (1, 2, 5, 20, 60, 200):
    cfg = bk.SolverConfig(1e-12, mi, "jacobi")
    r = bk.block_cg(op, Bh, cfg)
    X, rep = dd.solve_decomposed(bk, ctx, op, B, cfg, dd.partition_rows(40, 1))
    torch.cuda.synchronize()
    ctx.set_stream(None)
    Xh = X.cpu().numpy()
    print(mi, "single it", r.report.iterations, "res", r.report.final_rel_residual.max(), "| dd it", rep.iterations, "res", rep.final_rel_residual.max(), "| diff", np.abs(Xh - r.x).max(), flush=True)
