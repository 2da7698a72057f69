"""Throughput of K independent chips through bk_generate_batch on 1/2/4 streams
(device buffers): does running chips concurrently on SM shares pay off?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_23221_b200 as bk

cfgid = int(sys.argv[1]) if len(sys.argv) > 1 else 2
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
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
reps_n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
only = int(os.environ.get('PROBE_STREAMS', '4'))
for streams in ((only,) if reps_n > 2 else tuple(x for x in (1, 2, 4, 8) if x <= K)):
    for rep in range(reps_n):
        torch.cuda.synchronize()
        t = time.perf_counter()
        _, _, _, reps, tim = bk.generate_batch(chips, cfg, t_out=T, q_out=Q, resid_out=R,
                                               streams=streams, ctx=ctx, check_converged=False)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    its = [r.iterations for r in reps]
    print(f"config {cfgid}: {K} chips, streams={streams}: {dt * 1e3:.1f} ms "
          f"({K * N / dt:.0f} samples/s), iterations {its}")
