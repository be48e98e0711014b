"""Cluster-split patch solve (FDMGPU_SOLVE_CS): parity against the single-CTA
solve and the solve / smooth times per cluster size.  Usage: python tools/solve_cs.py CONFIG"""
import os, subprocess, sys, json

if len(sys.argv) > 2:  # child: one cluster size
    sys.path.insert(0, "/root/repo")
    import numpy as np, torch
    import paper_2107_14758_b200 as F
    cfg = [int(v) for v in sys.argv[1].split(",")]
    prob = F.Problem(*cfg); sol = F.Solver(prob); sol.set_stream(torch.cuda.current_stream()); sol.factor()
    r = torch.from_numpy(prob.rhs()).cuda(); z = torch.empty_like(r)
    rt = sol.apply_St(prob.rhs())
    zp = sol.patch_apply(rt)
    np.save(sys.argv[2], zp)
    sol.kernel_timing(True)
    for _ in range(3): sol.patch_apply(r, z)
    torch.cuda.synchronize()
    sol.kernel_timing(True)
    for _ in range(20): sol.patch_apply(r, z)
    torch.cuda.synchronize()
    t, n = sol.kernel_time("patch_solve")
    sol.kernel_timing(False)
    for _ in range(3): sol.smooth(r, z)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(50): sol.smooth(r, z)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"solve_ms": t / n, "smooth_ms": e0.elapsed_time(e1) / 50}), flush=True)
    sys.exit(0)

import numpy as np
cfg = sys.argv[1] if len(sys.argv) > 1 else "3"
os.makedirs("/tmp/cs", exist_ok=True)
res = {}
# (cluster size of the split solve: 0 = auto, 1 = none; split only the tail)
VARIANTS = [(1, 1), (0, 1), (2, 1), (3, 1), (4, 1), (2, 0)]
for vi, (cs, tail) in enumerate(VARIANTS):
    env = dict(os.environ, FDMGPU_SOLVE_CS=str(cs), FDMGPU_SOLVE_TAIL=str(tail))
    try:
        out = subprocess.run([sys.executable, __file__, cfg, f"/tmp/cs/z{vi}.npy"], env=env, capture_output=True,
                             text=True, timeout=120)
    except subprocess.TimeoutExpired:
        print(cs, tail, "TIMEOUT (hang)", flush=True)
        continue
    if out.returncode != 0:
        print(cs, "FAILED", out.stderr[-2000:], flush=True)
        continue
    d = json.loads(out.stdout.strip().splitlines()[-1])
    z1 = np.load("/tmp/cs/z0.npy"); zc = np.load(f"/tmp/cs/z{vi}.npy")
    d["rel_vs_cs1"] = float(np.linalg.norm(zc - z1) / np.linalg.norm(z1))
    print("config", cfg, "cs", cs, "tail", tail, json.dumps(d), flush=True)
