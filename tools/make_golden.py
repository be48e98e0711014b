"""Generates tests/golden/*.json from the CPU oracle (the restated reference).

Each fixture pins, for one configuration: sizes, hashes of the bit-exact index
maps, the Appendix-A factor structure of patch 0, the calibrated damping and
the PCG iteration count at rtol 1e-8, and size-independent summaries of the
relaxation output on the config's RHS (norm, dot with a seeded probe vector,
the values at 8 spread-out free DOFs, 64 slice norms).  Run: python tools/make_golden.py [config[,n,p]] ...
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:24]


NBLOCK = 64


def summarize(v, probe, free_idx):
    """Size-independent summary: norm, probe dot, the values at 8 spread-out free
    DOFs, and the norms of NBLOCK contiguous slices of the vector."""
    blocks = np.array_split(v, NBLOCK)
    return {"norm": float(np.linalg.norm(v)), "probe_dot": float(v @ probe),
            "free_head": [float(v[i]) for i in free_idx], "block_norms": [float(np.linalg.norm(b)) for b in blocks]}


def free_sample(constrained):
    free = np.flatnonzero(constrained == 0)
    return [int(free[k]) for k in np.linspace(0, len(free) - 1, 8).round().astype(int)]


def make(cfg, n=0, p=0, threads=os.cpu_count()):
    t0 = time.time()
    pb = O.Problem(cfg, n, p, build_global=False, threads=threads)
    m, pt = pb.maps(), pb.patches()
    r = pb.rhs()
    probe = np.random.default_rng(12345).standard_normal(pb.ndof)
    fidx = free_sample(m["constrained"])
    pb.factor(threads=threads)
    fi = pb.factor_info(0)
    out = {
        "config": cfg, "n": n, "p": pb.p, "dim": pb.dim, "ndof": pb.ndof, "nfree": pb.nfree,
        "npatches": pb.npatches, "sum_nj": pb.sum_nj,
        "hash": {"cell_dofs": sha(m["cell_dofs"]), "constrained": sha(m["constrained"]),
                 "labels": sha(np.stack([m["label_cls"], m["label_entity"]])), "patch_dofs": sha(pt["dofs"]),
                 "patch_perm": sha(pt["perm"]), "rhs": sha(r)},
        "free_idx": fidx,
        "patch0": {"n": fi["n"], "nnz_L": fi["nnz"], "flops": fi["flops"]},
        "apply_St": summarize(pb.apply_St(r), probe, fidx),
        "apply_A": summarize(pb.apply_A(r), probe, fidx),
        "smooth": summarize(pb.smooth(r), probe, fidx),
    }
    pb.build_twolevel(calibrate=True)
    tl = pb.twolevel_info()
    out["damping"] = {"omega": tl["omega"], "lambda_min": tl["lambda_min"], "lambda_max": tl["lambda_max"]}
    out["vcycle"] = summarize(pb.vcycle(r), probe, fidx)
    x, rep = pb.pcg(r, rtol=1e-8, maxit=200)
    out["pcg"] = {"iterations": rep["iterations"], "kappa": rep["kappa"], "converged": rep["converged"],
                  "final_residual": float(rep["residuals"][-1])}
    out["solution"] = summarize(x, probe, fidx)
    out["seconds"] = time.time() - t0
    return out


if __name__ == "__main__":
    specs = sys.argv[1:] or ["1", "2", "2,3,3", "4,4,5", "5,3,4", "5,0,3", "3", "4"]
    for s in specs:
        args = [int(v) for v in s.split(",")]
        res = make(*args)
        name = "c" + "_".join(str(a) for a in args) + ".json"
        with open(os.path.join(ROOT, "tests", "golden", name), "w") as f:
            json.dump(res, f, indent=1)
        print(name, res["pcg"], f"{res['seconds']:.1f}s", flush=True)
