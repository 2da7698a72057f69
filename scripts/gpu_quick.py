import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2510_23221_b200 as bk
from oracle.oracle import Oracle
import __graft_entry__ as ge
ge.smoke()
orc = Oracle()
ctx = bk.Context(0)
# stencil bitwise
for cfgid, shp in [(1,(32,32,1,8,16)),(3,(16,16,8,32,16)),(4,(16,16,4,16,8))]:
    inp = bk.synth_chip(cfgid, *shp)
    g = inp.grid
    op = bk.assemble(inp.k, g, inp.bc, ctx)
    o = orc.assemble((g.nx,g.ny,g.nz,g.lx,g.ly,g.lz), inp.k, inp.bc.as_tuples(), dz=g.dz)
    a, b = op.csr(), orc.csr(o)
    print('csr', cfgid, [np.array_equal(x,y) for x,y in zip(a,b)])
    X = np.random.default_rng(0).standard_normal((g.cell_count(), 7))
    print('apply', np.array_equal(op.apply_block(X), orc.apply_block(o, X)))
# timing C2 full
inp = bk.synth_chip(*bk.CONFIGS[2])
cfg = bk.SolverConfig(1e-12, 100000, 'jacobi')
for it in range(3):
    t=time.time()
    T,Q,R,rep,tim = bk.generate_chip(inp.grid, inp.k, inp.bc, inp.q_basis, inp.coef, cfg, ctx=ctx)
    print('C2', time.time()-t, rep.iterations, rep.matvec_count, tim, R.max())
import torch
Td = torch.empty((2048, 65536), dtype=torch.float64, device='cuda'); Qd = torch.empty_like(Td); Rd = torch.empty(2048, dtype=torch.float64, device='cuda')
kd = torch.from_numpy(inp.k).cuda(); qd = torch.from_numpy(inp.q_basis).cuda(); cd = torch.from_numpy(inp.coef).cuda()
for it in range(3):
    torch.cuda.synchronize(); t=time.time()
    T2,Q2,R2,rep,tim = bk.generate_chip(inp.grid, kd, inp.bc, qd, cd, cfg, t_out=Td, q_out=Qd, resid_out=Rd, ctx=ctx)
    torch.cuda.synchronize(); print('C2 dev', time.time()-t, rep.iterations, tim)
print('dev==host', torch.equal(Td.cpu(), torch.from_numpy(T)), torch.equal(Qd.cpu(), torch.from_numpy(Q)))
