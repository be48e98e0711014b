"""Factorisation time (CUDA events, mean of 3 after one warm-up) per config."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
for cfg in sys.argv[1:] or ["3"]:
    c = tuple(int(v) for v in cfg.split(","))
    prob = F.Problem(*c); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream())
    sol.factor(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3): sol.factor()
    e1.record(); torch.cuda.synchronize()
    r = prob.rhs(); z = sol.smooth(r)
    print(cfg, "factor ms", e0.elapsed_time(e1) / 3, "smooth norm", float((z * z).sum()) ** 0.5, flush=True)
