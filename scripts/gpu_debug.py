import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2510_23221_b200 as bk
from oracle.oracle import Oracle
orc = Oracle()
ctx = bk.Context(0)
def gt(g): return (g.nx,g.ny,g.nz,g.lx,g.ly,g.lz)
for cfgid, shp in [(1,(32,32,1,8,16)),(3,(16,16,8,32,16)),(4,(16,16,4,16,8))]:
    inp = bk.synth_chip(cfgid, *shp)
    g = inp.grid
    op = bk.assemble(inp.k, g, inp.bc, ctx)
    o = orc.assemble(gt(g), inp.k, inp.bc.as_tuples(), dz=g.dz)
    a, b = op.csr(), orc.csr(o)
    print('csr', cfgid, [np.array_equal(x,y) for x,y in zip(a,b)], flush=True)
    X = np.random.default_rng(0).standard_normal((g.cell_count(), 7))
    print('apply', np.array_equal(op.apply_block(X), orc.apply_block(o, X)), flush=True)
    B = bk.rhs_from_power(op, inp.q_basis)
    Bo = orc.rhs_from_power(o, inp.q_basis)
    print('rhs', np.array_equal(B, Bo), flush=True)
    cfg = bk.SolverConfig(1e-12, 3000, 'jacobi')
    for mi in [1, 2, 3, 5, 3000]:
        cfg.max_iter = mi
        r = bk.block_cg(op, Bo, cfg)
        Xo, ro = orc.block_cg(o, Bo, 1e-12, mi, 1)
        err = np.linalg.norm(r.x - Xo) / np.linalg.norm(Xo)
        print(' bcg maxit', mi, r.report.iterations, ro['iterations'], r.report.matvec_count, ro['matvec_count'], 'relerr %.3e' % err, 'res', r.report.final_rel_residual.max(), ro['final_rel_residual'].max(), np.isnan(r.x).sum(), flush=True)
    T, Q, R = bk.combine_action(op, Xo, inp.coef)
    To, Qo, Ro = orc.combine_action(o, Xo, inp.coef)
    print(' combine T eq', np.array_equal(T, To), 'Q eq', np.array_equal(Q, Qo), np.abs(Q-Qo).max()/np.abs(Qo).max(), 'R', R[:3], Ro[:3], flush=True)
