"""Scratch: one factorisation + 3 patch solves at C3 (ncu target for k_patch_solve)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
prob = F.Problem(3); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream()); sol.factor()
r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
for _ in range(3): sol.patch_apply(r, z)
torch.cuda.synchronize()
print("ok")
