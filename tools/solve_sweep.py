"""Scratch: time the patch solve kernel alone (patch_apply, CUDA events via kernel_timing)."""
import os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
prob = F.Problem(3); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream()); sol.factor()
r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
sol.kernel_timing(True)
for _ in range(3): sol.patch_apply(r, z)
torch.cuda.synchronize()
sol.kernel_timing(True)
for _ in range(10): sol.patch_apply(r, z)
torch.cuda.synchronize()
t, n = sol.kernel_time("patch_solve"); print(os.environ.get("FDMGPU_DBG_NP"), os.environ.get("FDMGPU_DBG_ST"), "solve ms", t / n, flush=True)
