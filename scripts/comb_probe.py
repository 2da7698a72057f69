"""Time the fused combine + action alone on a config's operator with a random
basis: python scripts/comb_probe.py CONFIG [N] (device buffers)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_23221_b200 as bk

cfgid = int(sys.argv[1])
_, nx, ny, nz, s, N0 = bk.CONFIGS[cfgid]
N = int(sys.argv[2]) if len(sys.argv) > 2 else N0
inp = bk.synth_chip(cfgid, nx, ny, nz, s, N)
ctx = bk.Context(0)
dev = torch.device("cuda", 0)
op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
n = nx * ny * nz
X = torch.from_numpy(np.random.default_rng(1).uniform(0, 50, (n, s))).to(dev)
C = torch.from_numpy(inp.coef).to(dev)
T = torch.empty((N, n), dtype=torch.float64, device=dev)
Q = torch.empty_like(T)
R = torch.empty(N, dtype=torch.float64, device=dev)
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    bk.combine_action(op, X, C, t_out=T, q_out=Q, resid_out=R)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"config {cfgid}: combine+action {N} samples {dt * 1e3:.2f} ms "
      f"({16 * n * N / dt / 1e9:.0f} GB/s written)")
