import ctypes as C, sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_23221_b200 as bk
lib = C.CDLL(bk.library_path())
for s in (8, 16, 32):
    cyc = C.c_longlong(); rank = C.c_int(); coef = np.zeros(s * s)
    err = lib.bk_debug_small_solve_cycles(s, 200, C.byref(cyc), C.byref(rank), coef.ctypes.data_as(C.c_void_p))
    i, j = np.meshgrid(np.arange(s), np.arange(s), indexing='ij')
    M = np.where(i == j, 1.0, 0.01 / (1 + i + j)) * np.exp(-0.5 * (i + j))
    R = np.where(i == j, 2.0, 0.1) * np.exp(-0.25 * (i + j))
    ref = np.linalg.solve(M, R)
    print(f"S={s} err={err} cycles/solve={cyc.value} rank={rank.value} relerr={np.linalg.norm(coef.reshape(s,s)-ref)/np.linalg.norm(ref):.2e}")
