"""Scratch: factor + calibrate once, then 2 V-cycles (ncu launch-list target)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
cfg = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (3, 0, 0)
prob = F.Problem(*cfg); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream()); sol.factor()
sol.omega = 0.22
r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
torch.cuda.synchronize()
for _ in range(2): sol.vcycle(r, z)
torch.cuda.synchronize()
print("ok")
