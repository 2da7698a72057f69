"""Cycles of the S = 64 control solve (alpha / beta, Gauss-Jordan with the
reference's diagonal pivoting) by warps in the pivot loop."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_23221_b200 as bk  # noqa: E402

lib = C.CDLL(bk.library_path())
cyc = (C.c_longlong * 10)()
coef = np.zeros(2 * 64 * 64)
only_reg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
err = lib.bk_debug_ctl_solve_cycles(50, cyc, coef.ctypes.data_as(C.c_void_p), only_reg)
i, j = np.meshgrid(np.arange(64), np.arange(64), indexing="ij")
M = np.where(i == j, 1.0, 0.01 / (1 + i + j)) * np.exp(-0.05 * (i + j))
R = np.where(i == j, 2.0, 0.1) * np.exp(-0.025 * (i + j))
ref = np.linalg.solve(M, R)
a, b = coef[:4096].reshape(64, 64), coef[4096:].reshape(64, 64)
print(f"err={err} rank={cyc[5]} cycles: small_solve_t 16 warps {cyc[0]}, 8 {cyc[1]}, 4 {cyc[2]}, "
      f"2 {cyc[3]}; small_solve_reg {cyc[4]}; relerr {np.linalg.norm(a - ref) / np.linalg.norm(ref):.2e}, "
      f"reg bitwise {np.array_equal(a, b)}; reg variants: no-update {cyc[6]}, 8 warps (256 thr) {cyc[7]}, "
      f"4 warps (128 thr) {cyc[8]}, no-barrier {cyc[9]}")
