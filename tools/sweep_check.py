"""Development sweep: GPU vs oracle on many (config, n, p) variants, incl. the generic
(non-specialised) kernel paths; prints one line per case with the worst rel-l2 and PCG counts."""
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
    cfg = tuple(int(v) for v in arg.split(","))
    t0 = time.time()
    try:
        prob = F.Problem(*cfg)
        sol = F.Solver(prob)
        sol.factor()
        ref = O.Problem(*cfg, build_global=True, threads=16)
        ref.factor()
        r = prob.rhs()
        errs = {n: rel(g(r), o(r)) for n, g, o in [("St", sol.apply_St, ref.apply_St), ("S", sol.apply_S, ref.apply_S),
                                                   ("A", sol.apply_A, ref.apply_A), ("smooth", sol.smooth, ref.smooth)]}
        sol.calibrate_damping()
        ref.build_twolevel()
        _, rep = sol.pcg(torch.from_numpy(r).cuda(), maxit=300)
        _, rr = ref.pcg(r, maxit=300)
        worst = max(errs.values())
        ok = worst < 1e-11 and rep["iterations"] == rr["iterations"]
        bad += not ok
        print(f"{'ok ' if ok else 'BAD'} {cfg}: worst {worst:.1e} {errs} pcg {rep['iterations']}/{rr['iterations']} "
              f"{time.time() - t0:.1f}s", flush=True)
    except Exception as e:
        bad += 1
        print(f"ERR {cfg}: {e}", flush=True)
print("sweep bad cases:", bad)
