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
cfg = bk.SolverConfig(1e-12, 20, "jacobi")
xs = [bk.block_cg(op, Bh, cfg).x for _ in range(3)]
print("single repeat diffs", np.abs(xs[0]-xs[1]).max(), np.abs(xs[0]-xs[2]).max())
ds = []
for _ in range(3):
    X, rep = dd.solve_decomposed(bk, ctx, op, B, cfg, dd.partition_rows(40, 1)); torch.cuda.synchronize(); ds.append(X.cpu().numpy()); ctx.set_stream(None)
print("dd repeat diffs", np.abs(ds[0]-ds[1]).max(), np.abs(ds[0]-ds[2]).max(), "dd vs single", np.abs(ds[0]-xs[0]).max())
for mi in range(5, 21):
    cfg = bk.SolverConfig(1e-12, mi, "jacobi")
    a = bk.block_cg(op, Bh, cfg).x
    X, rep = dd.solve_decomposed(bk, ctx, op, B, cfg, dd.partition_rows(40, 1)); torch.cuda.synchronize(); ctx.set_stream(None)
    print(mi, np.abs(X.cpu().numpy() - a).max(), flush=True)
