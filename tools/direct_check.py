"""Scratch: direct top block (default) vs the full tile factorisation (FDMGPU_DIRECT=0):
relaxation agreement on small cases and full configs, factor times."""
import gc, os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
import paper_2107_14758_b200 as F


def solver(prob, direct, schur="1"):
    os.environ["FDMGPU_DIRECT"] = "1" if direct else "0"
    os.environ["FDMGPU_SCHUR"] = schur
    sol = F.Solver(prob)
    sol.set_stream(torch.cuda.current_stream())
    t = []
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter(); sol.factor(); torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    return sol, min(t)


cases = [(2, 3, 3, True), (2, 3, 3, False), (4, 4, 5, True), (3, 3, 5, False), (3, 2, 15, True), (4, 3, 15, True), (3, 0, 0, True)]
if len(sys.argv) > 1 and sys.argv[1] == "5":
    cases = [(5, 0, 0, True)]
for cfg, n, p, skip in cases:
    prob = F.Problem(cfg, n, p, skip_boundary_patches=skip) if n else F.Problem(cfg)
    r = torch.from_numpy(prob.rhs()).cuda()
    out, tm = {}, {}
    for direct in (True, False):
        sol, tm[direct] = solver(prob, direct)
        L = sol.layout()
        assert L["top_direct"] == (1 if direct else 0), L
        out[direct] = sol.smooth(r).cpu().numpy()
        del sol; gc.collect(); torch.cuda.synchronize()
    err = np.linalg.norm(out[True] - out[False]) / np.linalg.norm(out[False])
    print(f"case {cfg},{n},{p},{skip}: rel {err:.2e}  factor direct {tm[True]*1e3:.2f} ms  full {tm[False]*1e3:.2f} ms", flush=True)
