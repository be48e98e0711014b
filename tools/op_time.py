"""Per-operator device time (CUDA events, mean of 50 after warm-up): apply_St, apply_S, apply_A, smooth."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
for cfg in sys.argv[1:] or ["3"]:
    c = tuple(int(v) for v in cfg.split(","))
    prob = F.Problem(*c); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream()); sol.factor()
    r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
    out = {}
    for name, fn in (("St", sol.apply_St), ("S", sol.apply_S), ("A", sol.apply_A), ("smooth", sol.smooth)):
        for _ in range(5): fn(r, z)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50): fn(r, z)
        b.record(); torch.cuda.synchronize()
        out[name] = round(a.elapsed_time(b) / 50 * 1e3, 2)
    print(cfg, "us", out, flush=True)
