"""Scratch: factor once, then smooth x2 and apply_A x2 (ncu launch-list target)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
cfg = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (3, 0, 0)
only_a = len(sys.argv) > 2 and sys.argv[2] == "A"
prob = F.Problem(*cfg); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream())
if not only_a: sol.factor()
r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("ops")
for _ in range(0 if only_a else 2): sol.smooth(r, z)
for _ in range(2): sol.apply_A(r, z)
torch.cuda.synchronize()
print("ok")
