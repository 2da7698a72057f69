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
print("B norm", B.norm().item())
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
slabs = dd.make_slabs(bk, ctx, op, 64, dd.partition_rows(40, 1))
sl = slabs[0]
sl.load_rhs(B); torch.cuda.synchronize()
print("local B norm", sl.B.norm().item(), sl.B.shape, "nb", sl.nb, "part", sl.part.numel(), "ctl", sl.ctl.numel())
cfg = bk.SolverConfig(1e-12, 100000, "jacobi"); cc = cfg._c()
sl.step(dd.INIT_SWEEP, cc); torch.cuda.synchronize()
print("after init: red[:3]", sl.red[:3].tolist(), "bn2", sl.red[64*64:64*64+3].tolist(), "R norm", sl.R.norm().item(), "P norm", sl.P.norm().item())
sl.step(dd.CTL_INIT, cc); print("read", sl.step(dd.READ, cc))
for m in range(1, 4):
    sl.step(dd.SPMM, cc); torch.cuda.synchronize(); print(m, "G diag", sl.red[0].item(), "W norm", sl.W.norm().item())
    sl.step(dd.CTL_ALPHA, cc)
    sl.step(dd.UPDATE, cc); torch.cuda.synchronize(); print(m, "rr", sl.red[64*64].item(), "X norm", sl.X.norm().item(), "R", sl.R.norm().item())
    sl.step(dd.CTL_UPDATE, cc, m); print(m, "read", sl.step(dd.READ, cc))
    sl.step(dd.PUPDATE, cc); torch.cuda.synchronize(); print(m, "P norm", sl.P.norm().item())
