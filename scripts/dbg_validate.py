import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2510_23221_b200 as bk
ctx = bk.Context(0)
ins = bk.synth_chip(1, 64, 64, 1, 8, 64, master_seed=1, chip_id=0)
print("grid", ins.grid, "bc", ins.bc)
cfg = bk.SolverConfig(1e-12, 100000, "jacobi")
n, N = ins.grid.cell_count(), 64
T = torch.empty((N, n), dtype=torch.float64, device="cuda"); Q = torch.empty_like(T)
R = torch.empty(N, dtype=torch.float64, device="cuda")
bk.generate_chip(ins.grid, ins.k, ins.bc, ins.q_basis, ins.coef, cfg, T, Q, R, ctx=ctx)
print("pipeline resid", R[:4].tolist())
op_a = bk.assemble(ins.k, ins.grid, ins.bc, ctx)
faces = [bk.Robin(1e-300, 0.0) if isinstance(f, bk.Adiabatic) else f for f in ins.bc.faces]
op_r = bk.assemble(ins.k, ins.grid, bk.BoundarySpec(faces), ctx)
print("rr adiabatic op", bk.relative_residual(op_a, T, Q)[:4])
print("rr robin op", bk.relative_residual(op_r, T, Q)[:4])
ca, cr = op_a.csr(), op_r.csr()
for name, a, b in zip(("row_ptr", "col", "val", "g", "vol"), ca, cr):
    a, b = np.asarray(a), np.asarray(b)
    print(name, a.shape, b.shape, "equal" if a.shape == b.shape and np.array_equal(a, b) else "DIFF")
Th, Qh = T.cpu().numpy(), Q.cpu().numpy()
print("host path", bk.relative_residual(op_a, Th, Qh)[:4])
# numpy check
rp, col, val, g, vol = ca
Au = np.zeros(n)
u = Th[0]
for i in range(n):
    Au[i] = np.dot(val[rp[i]:rp[i+1]], u[col[rp[i]:rp[i+1]]])
b = vol * Qh[0] + g
print("numpy", np.linalg.norm(b - Au) / np.linalg.norm(b))
