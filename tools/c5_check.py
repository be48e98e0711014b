"""Scratch: p=31 slab transforms vs the CPU oracle (S, S^T, A) and vs the staged
path (smooth / patch apply, via FDMGPU_FORCE_STAGED=1 in a second process)."""
import os, subprocess, sys
sys.path.insert(0, "/root/repo")
import numpy as np
cfg = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (5, 2, 31)
mode = sys.argv[2] if len(sys.argv) > 2 else "main"
import paper_2107_14758_b200 as F
import torch
prob = F.Problem(*cfg); sol = F.Solver(prob); sol.factor()
r = prob.rhs()
out = {"St": sol.apply_St(r), "S": sol.apply_S(r), "smooth": sol.smooth(r), "patch": sol.patch_apply(sol.apply_St(r))}
if mode == "staged":
    np.savez("/tmp/c5_staged.npz", **out); sys.exit(0)
env = dict(os.environ, FDMGPU_FORCE_STAGED="1")
subprocess.run([sys.executable, __file__, sys.argv[1] if len(sys.argv) > 1 else "5,2,31", "staged"], env=env, check=True)
st = np.load("/tmp/c5_staged.npz")
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for k in out: print(f"{k:7s} new-vs-staged rel {rel(out[k], st[k]):.3e}", flush=True)
from oracle import oracle as O
ref = O.Problem(*cfg, build_global=True, threads=os.cpu_count())
print("St vs oracle", rel(out["St"], ref.apply_St(r)), "S vs oracle", rel(out["S"], ref.apply_S(r)), flush=True)
