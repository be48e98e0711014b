"""Scratch GPU parity check (development): product vs oracle on small configs."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import torch
import paper_2107_14758_b200 as F
from oracle import oracle as O

def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)

cases = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(2, 3, 3), (1, 0, 0), (2, 0, 0)]
for cfg in cases:
    t0 = time.time()
    prob = F.Problem(*cfg)
    sol = F.Solver(prob)
    L = sol.layout()
    ref = O.Problem(*cfg, build_global=True, threads=16)
    print(f"cfg {cfg}: ndof {prob.ndof} patches {prob.npatches} layout {L}", flush=True)
    t = time.time(); sol.factor(); torch.cuda.synchronize(); print(f"  gpu factor {time.time()-t:.3f}s", flush=True)
    t = time.time(); ref.factor(); print(f"  cpu factor {time.time()-t:.3f}s", flush=True)
    r = prob.rhs()
    for name, g, o in [("St", sol.apply_St, ref.apply_St), ("S", sol.apply_S, ref.apply_S), ("A", sol.apply_A, ref.apply_A),
                       ("patch", sol.patch_apply, ref.patch_apply), ("smooth", sol.smooth, ref.smooth)]:
        x = r if name != "patch" else ref.apply_St(r)
        print(f"  {name:7s} rel-l2 {rel(g(x), o(x)):.3e}", flush=True)
    w = sol.calibrate_damping()
    ref.build_twolevel()
    wr = ref.twolevel_info()
    print(f"  omega gpu {w} ref {wr}", flush=True)
    sol.omega = wr["omega"]
    print(f"  vcycle rel-l2 {rel(sol.vcycle(r), ref.vcycle(r)):.3e}")
    sol.omega = w["omega"]
    b = torch.from_numpy(r).cuda()
    x, rep = sol.pcg(b)
    xr, repr_ = ref.pcg(r)
    print(f"  pcg gpu it {rep['iterations']} kappa {rep['kappa']:.4f} | ref it {repr_['iterations']} kappa {repr_['kappa']:.4f}; x rel {rel(x.cpu().numpy(), xr):.2e}; {time.time()-t0:.1f}s", flush=True)
