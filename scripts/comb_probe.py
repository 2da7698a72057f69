"""Time the fused combine + action alone on a config's operator with a random
basis: python scripts/comb_probe.py CONFIG [N] [option=value ...] (device
buffers; CUDA events, best of 5); with options, also checks the outputs are
bitwise those of the default kernel."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_23221_b200 as bk

cfgid = int(sys.argv[1])
_, nx, ny, nz, s, N0 = bk.CONFIGS[cfgid]
N = int(sys.argv[2]) if len(sys.argv) > 2 and "=" not in sys.argv[2] else N0
opts = {k: int(v) for k, v in (x.split("=") for x in sys.argv[2:] if "=" in x)}
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
def run(o):
    best = 1e9
    with ctx.options(**o):
        for it in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            bk.combine_action(op, X, C, t_out=T, q_out=Q, resid_out=R)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
    return best, T.clone(), Q.clone(), R.clone()


variants = [("default", {})] + ([("opts " + str(opts), opts)] if opts else [])
ref = None
for name, o in variants:
    dt, Tv, Qv, Rv = run(o)
    same = None if ref is None else (torch.equal(Tv, ref[0]) and torch.equal(Qv, ref[1]),
                                     float((Rv - ref[2]).abs().max()))
    ref = ref or (Tv, Qv, Rv)
    sha = hashlib.sha256(Tv.cpu().numpy().tobytes() + Qv.cpu().numpy().tobytes()
                         + Rv.cpu().numpy().tobytes()).hexdigest()[:16] if N * n <= 1 << 28 else "-"
    print(f"config {cfgid} {name}: sha {sha} combine+action {N} samples {dt * 1e3:.3f} ms "
          f"({16 * n * N / dt / 1e9:.0f} GB/s written) bitwise T,q / max resid diff vs default: {same}",
          flush=True)
