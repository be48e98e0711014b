"""Development: PCG wall time (device-resident graph loop) per config."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
for a in sys.argv[1:]:
    cfg = tuple(int(v) for v in a.split(","))
    prob = F.Problem(*cfg); sol = F.Solver(prob); sol.factor()
    t = time.perf_counter(); w = sol.calibrate_damping(); tc = time.perf_counter() - t
    b = torch.from_numpy(prob.rhs()).cuda()
    x, rep = sol.pcg(b); x, rep = sol.pcg(b)
    print(cfg, "calibrate %.1f ms" % (tc * 1e3), "pcg it", rep["iterations"], "kappa %.4f" % rep["kappa"], "time %.2f ms" % (rep["wall_time"] * 1e3), "omega", w["omega"], flush=True)
