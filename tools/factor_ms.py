"""Factorisation time (CUDA events, best of 3) for configs: python tools/factor_ms.py 3 5 ..."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2107_14758_b200 as F

for a in sys.argv[1:]:
    sol = F.Solver(F.Problem(int(a)))
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        sol.factor()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"C{a} factor {min(ts):.2f} ms", flush=True)
