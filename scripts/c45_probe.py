"""Probe configs 4 and 5 on the GPU: batch throughput vs streams; C5 solve."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_23221_b200 as bk
ctx = bk.Context(0)
cfg = bk.SolverConfig(1e-12, 2000, "jacobi")
chips = [bk.synth_chip(4, 128, 128, 4, 16, 8, chip_id=c) for c in range(32)]
dev = torch.device("cuda", 0)
class Ch: pass
dchips = []
for ch in chips:
    d = Ch(); d.grid = ch.grid; d.bc = ch.bc
    d.k = torch.from_numpy(ch.k).to(dev); d.q_basis = torch.from_numpy(ch.q_basis).to(dev); d.coef = torch.from_numpy(ch.coef).to(dev)
    dchips.append(d)
n = 128 * 128 * 4
T = [torch.empty((8, n), dtype=torch.float64, device=dev) for _ in chips]
Q = [torch.empty((8, n), dtype=torch.float64, device=dev) for _ in chips]
R = [torch.empty(8, dtype=torch.float64, device=dev) for _ in chips]
for streams in (1, 2, 4, 8, 16):
    bk.generate_batch(dchips[:streams], cfg, T[:streams], Q[:streams], R[:streams], streams=streams, ctx=ctx, check_converged=False)
    torch.cuda.synchronize(); t = time.time()
    _, _, _, reps, tim = bk.generate_batch(dchips, cfg, T, Q, R, streams=streams, ctx=ctx, check_converged=False)
    torch.cuda.synchronize(); dt = time.time() - t
    its = [r.iterations for r in reps]; nconv = sum(r.all_converged() for r in reps)
    print(f"C4 32 chips streams={streams}: {dt*1e3:.1f} ms -> {32*8/dt:.0f} samples/s; iters mean {np.mean(its):.0f} max {max(its)} converged {nconv}/32; solve sum {tim.basis_solve_s*1e3:.0f} ms", flush=True)
# C5 solve (generic S=64 path)
inp = bk.synth_chip(5, 512, 512, 16, 64, 16)
op = bk.assemble(inp.k, inp.grid, inp.bc, ctx)
qd = torch.from_numpy(inp.q_basis).to(dev)
B = torch.empty_like(qd); bk.rhs_from_power(op, qd, out=B)
X = torch.empty_like(qd)
for mi in (5, 50):
    torch.cuda.synchronize(); t = time.time()
    r = bk.block_cg(op, B, bk.SolverConfig(1e-12, mi, "jacobi"), out=X)
    torch.cuda.synchronize(); dt = time.time() - t
    print(f"C5 block_cg max_iter={mi}: {dt:.2f} s ({dt/mi*1e3:.1f} ms/iter) res {r.report.final_rel_residual.max():.2e}", flush=True)
