import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_23221_b200 as bk
ctx = bk.Context(0)
dev = torch.device("cuda", 0)
inp = bk.synth_chip(5, 512, 512, 16, 64, 16)
op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
qd = torch.from_numpy(inp.q_basis).to(dev)
B = torch.empty_like(qd); bk.rhs_from_power(op, qd, out=B)
X = torch.empty_like(qd)
mi = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for it in range(2):
    torch.cuda.synchronize(); t = time.time()
    r = bk.block_cg(op, B, bk.SolverConfig(1e-12, mi, "jacobi"), out=X)
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"C5 block_cg max_iter={mi}: {dt:.3f} s ({dt/max(r.report.iterations,1)*1e3:.2f} ms/iter) iters {r.report.iterations} res max {r.report.final_rel_residual.max():.2e} conv {r.report.converged.sum()}", flush=True)
