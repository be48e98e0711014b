"""Small end-to-end driver for compute-sanitizer runs (one tool per gpurun call):
scalar (2, 2, 3) and (1, 2, 3) factor / operators / PCG, elasticity in 2D Q3 and 3D Q15."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2107_14758_b200 as F

for prob in (F.Problem(2, 2, 3), F.Problem(1, 2, 3), F.Problem.elasticity(2, 3, 3, 1.0, 2.0),
             F.Problem.elasticity(3, 2, 15, 1.0, 1.0)):
    sol = F.Solver(prob)
    sol.factor()
    r = prob.rhs()
    for fn in (sol.apply_St, sol.apply_S, sol.apply_A, sol.smooth):
        y = fn(r)
        assert np.isfinite(y).all()
    sol.calibrate_damping()
    x, rep = sol.pcg(torch.from_numpy(r).cuda(), maxit=300)
    torch.cuda.synchronize()
    print(prob.ndof, rep["iterations"], rep["converged"], flush=True)
print("sanitize driver ok")
