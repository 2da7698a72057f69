"""Per-phase timing (BK_CG_PROFILE) of a batched solve capped at a few
iterations: python scripts/phase_probe.py CONFIG K MAXIT (A/B of experimental
library builds via BK_LIBRARY)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("BK_CG_PROFILE", "1")
import torch

import paper_2510_23221_b200 as bk

cfgid, K, maxit = (int(v) for v in sys.argv[1:4])
_, nx, ny, nz, s, N = bk.CONFIGS[cfgid]
ctx = bk.Context(0)
dev = torch.device("cuda", 0)
chips = []
for c in range(K):
    inp = bk.synth_chip(cfgid, nx, ny, nz, s, 16, chip_id=c)
    inp.k, inp.q_basis, inp.coef = (torch.from_numpy(a).to(dev) for a in (inp.k, inp.q_basis, inp.coef))
    chips.append(inp)
n = nx * ny * nz
T = [torch.empty((16, n), dtype=torch.float64, device=dev) for _ in range(K)]
Q = [torch.empty_like(t) for t in T]
R = [torch.empty(16, dtype=torch.float64, device=dev) for _ in range(K)]
cfg = bk.SolverConfig(1e-12, maxit, "jacobi")
for _ in range(2):
    _, _, _, reps, tim = bk.generate_batch(chips, cfg, t_out=T, q_out=Q, resid_out=R, streams=K,
                                           ctx=ctx, check_converged=False)
print(f"solve {tim.basis_solve_s * 1e3:.2f} ms for {maxit} iterations x {K} chips")
