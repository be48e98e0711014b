"""Scratch: one operator (St | S | A | smooth) repeated on C3-like configs (ncu target)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
op = sys.argv[1] if len(sys.argv) > 1 else "St"
cfg = tuple(int(v) for v in sys.argv[2].split(",")) if len(sys.argv) > 2 else (3, 0, 0)
prob = F.Problem(*cfg); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream())
if op == "smooth": sol.factor()
r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
fn = {"St": sol.apply_St, "S": sol.apply_S, "A": sol.apply_A, "smooth": sol.smooth}[op]
for _ in range(5): fn(r, z)
torch.cuda.synchronize()
print("ok")
