"""Scratch: one factorisation at the given config (ncu target for the factor kernels)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
cfg = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (3, 0, 0)
prob = F.Problem(*cfg); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream()); sol.factor()
torch.cuda.synchronize()
print("ok")
