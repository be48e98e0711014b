"""Scratch GPU timing (development): per-operator CUDA-event timings on one config."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F

cfg = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (3, 0, 0)
t = time.time(); prob = F.Problem(*cfg); print(f"host setup {time.time()-t:.2f}s ndof {prob.ndof} nfree {prob.nfree}", flush=True)
t = time.time(); sol = F.Solver(prob); print(f"attach {time.time()-t:.2f}s layout {sol.layout()}", flush=True)
s = torch.cuda.current_stream(); sol.set_stream(s)
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
ms = timeit(sol.factor, 2); print(f"factor {ms:.2f} ms", flush=True)
L = sol.layout()
r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r); z2 = torch.empty_like(r)
for name, fn in [("St", lambda: sol.apply_St(r, z)), ("S", lambda: sol.apply_S(r, z)), ("A", lambda: sol.apply_A(r, z)),
                 ("patch", lambda: sol.patch_apply(r, z)), ("smooth", lambda: sol.smooth(r, z))]:
    ms = timeit(fn, 10)
    extra = ""
    if name == "smooth":
        nnz = L["nnz_L"] * L["npatch"]; P = prob.sum_nj
        by = 8 * (2 * nnz + 2 * P + 4 * prob.ndof)
        extra = f" GDOF/s {prob.nfree/ms/1e6:.3f}  algorithmic {by/1e9:.2f} GB -> {by/ms/1e6:.0f} GB/s"
    print(f"{name:7s} {ms:8.3f} ms{extra}", flush=True)
w = sol.calibrate_damping(); print("omega", w, flush=True)
x, rep = sol.pcg(r); print("pcg", rep["iterations"], rep["kappa"], rep["wall_time"], flush=True)
