"""Where does the e2e time of a 3-chip C2 generate_batch go? device vs host outputs."""
import os
import sys
import time
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_23221_b200 as bk

ctx = bk.Context(0)
dev = torch.device("cuda", 0)
inp = bk.synth_chip(2, 256, 256, 1, 16, 2048)
n, N = inp.grid.cell_count(), 2048
cfg = bk.SolverConfig(1e-12, 100000, "jacobi")
K = 3
pin = lambda t: t.pin_memory()  # noqa: E731
k_h, q_h, c_h = (pin(torch.from_numpy(a)) for a in (inp.k, inp.q_basis, inp.coef))
chips = [SimpleNamespace(grid=inp.grid, bc=inp.bc, k=k_h, q_basis=q_h, coef=c_h) for _ in range(K)]
Th = [pin(torch.empty((N, n), dtype=torch.float64)) for _ in range(K)]
Qh = [pin(torch.empty((N, n), dtype=torch.float64)) for _ in range(K)]
Rh = [pin(torch.empty(N, dtype=torch.float64)) for _ in range(K)]
Td = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in range(K)]
Qd = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in range(K)]
Rd = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(K)]
for name, T, Q, R in (("device", Td, Qd, Rd), ("host", Th, Qh, Rh), ("device", Td, Qd, Rd),
                      ("host", Th, Qh, Rh)):
    torch.cuda.synchronize()
    t = time.perf_counter()
    _, _, _, reps, tim = bk.generate_batch(chips, cfg, t_out=T, q_out=Q, resid_out=R, streams=1,
                                           ctx=ctx)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"batch x{K} {name}: {dt * 1e3:.1f} ms ({dt / K * 1e3:.1f} ms/chip) solve "
          f"{tim.basis_solve_s * 1e3 / K:.1f} combine {tim.combine_action_s * 1e3 / K:.1f} "
          f"d2h-tail {tim.d2h_s * 1e3 / K:.1f} ms/chip")
for name in ("single-chip host", "single-chip host"):
    torch.cuda.synchronize()
    t = time.perf_counter()
    bk.generate_chip(inp.grid, k_h, inp.bc, q_h, c_h, cfg, t_out=Th[0], q_out=Qh[0],
                     resid_out=Rh[0], ctx=ctx)
    print(f"{name}: {(time.perf_counter() - t) * 1e3:.1f} ms")
torch.cuda.synchronize()
t = time.perf_counter()
for i in range(K):
    Th[i].copy_(Td[i], non_blocking=True)
    Qh[i].copy_(Qd[i], non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"pure D2H of {K} chips: {dt * 1e3:.1f} ms ({2 * K * N * n * 8 / dt / 1e9:.1f} GB/s)")
