import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_23221_b200 as bk
ctx = bk.Context(0)
dev = torch.device("cuda", 0)
for (nx, nz, s) in [(512, 16, 64)]:
    inp = bk.synth_chip(5, nx, nx, nz, s, 4)
    op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
    qd = torch.from_numpy(inp.q_basis).to(dev)
    B = torch.empty_like(qd); bk.rhs_from_power(op, qd, out=B)
    X = torch.empty_like(qd)
    for mi in (600, 1200, 2400):
        t = time.time()
        r = bk.block_cg(op, B, bk.SolverConfig(1e-12, mi, "jacobi"), out=X)
        torch.cuda.synchronize(); dt = time.time() - t
        fr = r.report.final_rel_residual
        print(f"{nx}x{nx}x{nz} s={s} max_iter={mi}: iters {r.report.iterations} matvecs {r.report.matvec_count} conv {r.report.converged.sum()}/{s} res min {fr.min():.2e} med {np.median(fr):.2e} max {fr.max():.2e} ({dt:.1f}s)", flush=True)
        if r.report.all_converged(): break
