"""Scratch: C5 residual apply (trilinear quadrature path) timing per FDMGPU_QUAD_STRIP mode; output hash for equality."""
import hashlib, os, sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
cfg = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (5, 0, 0)
prob = F.Problem(*cfg); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream())
r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
for _ in range(5): sol.apply_A(r, z)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
ev[0].record()
for i in range(20):
    sol.apply_A(r, z); ev[i + 1].record()
torch.cuda.synchronize()
t = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(20))
print(f"QUAD_STRIP={os.environ.get('FDMGPU_QUAD_STRIP', 'default')} apply_A median {t[10]:.4f} ms min {t[0]:.4f} ms hash {hashlib.sha1(z.cpu().numpy().tobytes()).hexdigest()[:16]}", flush=True)
