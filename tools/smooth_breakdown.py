"""Scratch: warm per-class kernel times (CUDA events) over 20 relaxation applies."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
cfg = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (3, 0, 0)
prob = F.Problem(*cfg); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream()); sol.factor()
r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
for _ in range(3): sol.smooth(r, z)
torch.cuda.synchronize()
sol.kernel_timing(True)
for _ in range(20): sol.smooth(r, z)
torch.cuda.synchronize()
for k in ("patch_solve", "transform"):
    t, n = sol.kernel_time(k); print(f"{k:12s} {t / 20 * 1e3:8.1f} us per apply ({n // 20} launches)")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
sol.kernel_timing(False)
e0.record()
for _ in range(20): sol.smooth(r, z)
e1.record(); torch.cuda.synchronize()
print(f"apply total {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us")
