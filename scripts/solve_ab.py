"""A/B of a batched solve + combine step (bk_generate_batch, K chips in one
launch) under context options: python scripts/solve_ab.py CONFIG K [opt=v ...].
Prints per-variant step time (CUDA events, best of 3), the solve phase time,
and whether checksums of T / q equal the default variant's."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_23221_b200 as bk  # noqa: E402

cfgid, K = int(sys.argv[1]), int(sys.argv[2])
opts = {k: int(v) for k, v in (x.split("=") for x in sys.argv[3:])}
_, nx, ny, nz, s, N = bk.CONFIGS[cfgid]
if cfgid == 4:
    N = 8
ctx = bk.Context(0)
dev = torch.device("cuda", 0)
chips = []
for c in range(K):
    inp = bk.synth_chip(cfgid, nx, ny, nz, s, N, chip_id=c)
    inp.k = torch.from_numpy(inp.k).to(dev)
    inp.q_basis = torch.from_numpy(inp.q_basis).to(dev)
    inp.coef = torch.from_numpy(inp.coef).to(dev)
    chips.append(inp)
n = nx * ny * nz
T = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in range(K)]
Q = [torch.empty((N, n), dtype=torch.float64, device=dev) for _ in range(K)]
R = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(K)]
cfg = bk.SolverConfig(1e-12 if cfgid < 4 else 1e-10, 5000 if cfgid == 4 else 100000, "jacobi")
ref = None
for name, o in (("default", {}), ("opts " + str(opts), opts)):
    if not o and name != "default":
        continue
    best = 1e9
    with ctx.options(**o):
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, _, _, reps, tim = bk.generate_batch(chips, cfg, t_out=T, q_out=Q, resid_out=R,
                                                   streams=K, ctx=ctx, check_converged=False)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        var = ctx.last_solver_variant
    # checksums of every chip's outputs (a full copy would not fit beside them)
    cur = (torch.stack([t.double().sum() for t in T]), torch.stack([q[:, ::97].sum() for q in Q]))
    same = None if ref is None else (torch.equal(cur[0], ref[0]), torch.equal(cur[1], ref[1]))
    ref = ref or cur
    print(f"config {cfgid} x{K} {name} [{var}]: {best:.1f} ms ({K * N / best * 1e3:.0f} samples/s), "
          f"iterations {[r.iterations for r in reps][:4]}..., bitwise T,q vs default {same}", flush=True)
