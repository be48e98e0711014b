"""Development sweep: elasticity GPU vs oracle over (dim, n, p, lambda) variants."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2107_14758_b200 as F
from oracle import oracle as O


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


bad = 0
for arg in sys.argv[1:]:
    dim, n, p, lam = (float(v) for v in arg.split(","))
    dim, n, p = int(dim), int(n), int(p)
    t0 = time.time()
    try:
        prob = F.Problem.elasticity(dim, n, p, 1.0, lam)
        sol = F.Solver(prob)
        sol.factor()
        ref = O.ElasticProblem(dim, n, p, 1.0, lam, threads=16)
        ref.build()
        r = ref.random_free(5)
        errs = {"A": rel(sol.apply_A(r), ref.apply_A(r)), "smooth": rel(sol.smooth(r), ref.op("smooth", r))}
        w = sol.calibrate_damping()["omega"]
        wr = ref.twolevel_info()["omega"]
        b = prob.rhs()
        _, rep = sol.pcg(torch.from_numpy(b).cuda(), maxit=600)
        _, rr = ref.pcg(b, maxit=600)
        ok = max(errs.values()) < 1e-11 and rep["iterations"] == rr["iterations"] and abs(w - wr) <= 1e-10 * wr
        bad += not ok
        print(f"{'ok ' if ok else 'BAD'} {(dim, n, p, lam)}: {errs} omega {w:.6f}/{wr:.6f} pcg {rep['iterations']}/"
              f"{rr['iterations']} {time.time() - t0:.1f}s", flush=True)
    except Exception as e:
        bad += 1
        print(f"ERR {(dim, n, p, lam)}: {e}", flush=True)
print("sweep bad cases:", bad)
