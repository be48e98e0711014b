"""Conditioning of the Schur split's top-separator block S~_RR (SchurSplit) on
one interior patch, and the accuracy of applying S~_RR^{-1} as an explicit
symmetric inverse vs the Cholesky triangular solves (numpy, float64).
Usage: python tools/cond_top.py CONFIG [PATCH]"""
import sys
import time

import numpy as np
import scipy.linalg as sl

sys.path.insert(0, "/root/repo")
import paper_2107_14758_b200 as F

cfg = int(sys.argv[1])
prob = F.Problem(cfg)
sol = F.Solver(prob)
L = sol.layout()
j = int(sys.argv[2]) if len(sys.argv) > 2 else prob.npatches // 2
m, nR = L["n_interface"], L["n_top"]
nF = m - nR
t = time.time()
S = sol.patch_schur(j)
S = np.tril(S) + np.tril(S, -1).T
SFF, SRF, SRR = S[:nF, :nF], S[nF:, :nF], S[nF:, nF:]
cF = sl.cho_factor(SFF, lower=True)
St = SRR - SRF @ sl.cho_solve(cF, SRF.T)
ev = np.linalg.eigvalsh(St)
evF = np.linalg.eigvalsh(SFF)
evG = np.linalg.eigvalsh(S)
print(f"config {cfg} patch {j}: m {m} nF {nF} nR {nR}  ({time.time() - t:.1f} s)")
print(f"cond S_G {evG[-1] / evG[0]:.3e}  cond S_FF {evF[-1] / evF[0]:.3e}  cond S~_RR {ev[-1] / ev[0]:.3e}")
Lr = np.linalg.cholesky(St)
Winv = sl.solve_triangular(Lr, np.eye(nR), lower=True)
Ainv = Winv.T @ Winv
rng = np.random.default_rng(0)
for trial in range(3):
    b = rng.standard_normal(nR)
    x_chol = sl.solve_triangular(Lr.T, sl.solve_triangular(Lr, b, lower=True), lower=False)
    x_inv = Ainv @ b
    # reference by one step of iterative refinement in extended precision of the residual
    r = b - (St.astype(np.longdouble) @ x_chol.astype(np.longdouble)).astype(np.float64)
    x_ref = x_chol + sl.solve_triangular(Lr.T, sl.solve_triangular(Lr, r, lower=True), lower=False)
    e = lambda x: np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref)
    print(f"trial {trial}: rel err cholesky {e(x_chol):.2e}  explicit inverse {e(x_inv):.2e}")
