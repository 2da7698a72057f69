"""C5 streaming pipeline (bk_generate_stream, every sample drained to pinned host
memory): ms per chip over K chips, and the drain rate implied by
total = first solve + K x drain:  python scripts/c5_stream_probe.py [K]"""
import os
import sys
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_23221_b200 as bk  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = bk.Context(0)
inp = bk.synth_chip(5, 512, 512, 16, 64, 5000)
n, N = inp.grid.cell_count(), 5000
cfg = bk.SolverConfig(1e-10, 100000, "jacobi")
chip = SimpleNamespace(grid=inp.grid, bc=inp.bc, k=torch.from_numpy(inp.k).pin_memory(),
                       q_basis=torch.from_numpy(inp.q_basis).pin_memory(),
                       coef=torch.from_numpy(inp.coef).pin_memory())
bk.generate_stream([chip], cfg, sink=None, ctx=ctx)
for k in (1, K):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps, tim = bk.generate_stream([chip] * k, cfg, sink=None, ctx=ctx)
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3
    gb = (2 * n * N + N) * 8 * k / 1e9
    print(f"{k} chips: {s:.2f} s = {s / k:.2f} s/chip, {gb / s:.1f} GB/s overall, "
          f"{N * k / s:.0f} samples/s", flush=True)
