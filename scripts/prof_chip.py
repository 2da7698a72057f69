"""Run the per-chip pipeline a few times on device buffers (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_23221_b200 as bk
cfgid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = bk.CONFIGS[cfgid]
inp = bk.synth_chip(*c)
n, N = inp.grid.cell_count(), c[5]
dev = torch.device("cuda", 0)
ctx = bk.Context(0)
Td = torch.empty((N, n), dtype=torch.float64, device=dev); Qd = torch.empty_like(Td)
Rd = torch.empty(N, dtype=torch.float64, device=dev)
k, q, cc = (torch.from_numpy(a).to(dev) for a in (inp.k, inp.q_basis, inp.coef))
cfg = bk.SolverConfig(1e-12, 100000, "jacobi")
for _ in range(reps):
    T, Q, R, rep, tim = bk.generate_chip(inp.grid, k, inp.bc, q, cc, cfg, t_out=Td, q_out=Qd, resid_out=Rd, ctx=ctx)
    print(rep.iterations, tim)
