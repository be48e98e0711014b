"""CPU baseline matrix of BASELINE.md §4 (a reported baseline, not the target).

The reference itself cannot be compiled (Eigen3 absent), so the CPU side is
the oracle (oracle/, plain-C++ restatement of the reference path, test
infrastructure).  Run on the GPU box's host cores:

    python tools/cpu_baseline.py [--configs 1,2,3,5] [--reps 5] [--out profiles/cpu_baseline_r2.json]

Per configuration and thread count (SolverConfig::threads = 1 and = nproc,
parallel_for over patches as src/schwarz.cpp:16-29), median / min / max of
--reps repetitions after one warm-up (std::chrono-equivalent perf_counter,
SPEC.md:682 methodology) of the units
  apply_St, apply_S, apply_A  -- serial in the reference at any thread count,
  smooth                      -- S (PatchSolver::apply (S^T r)), patch stage threaded,
  factorisation               -- cholesky() of sampled patches (k = threads), scaled,
  pcg                         -- full PCG at the golden omega (C1-C3), with its count.
C5 (p = 31) runs only the transforms, the operator and a sampled patch stage:
one reference factorisation is 8.66e10 multiply-adds (~143 s), so `threads`
patches are factored once in parallel and timed; the full CPU C5 path needs
~160 GB of factors.
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

import bench  # noqa: E402  (host_info)


def timed(fn, reps):
    fn()  # warm-up
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return {"median_s": statistics.median(ts), "min_s": min(ts), "max_s": max(ts), "reps": reps}


def run_config(cfg, threads_list, reps, log):
    out = {"config": cfg, "workload": bench.WORKLOADS[cfg], "units": {}}
    g = None
    gpath = os.path.join(ROOT, "tests", "golden", f"c{cfg}.json")
    if os.path.exists(gpath):
        g = json.load(open(gpath))
    nproc = max(threads_list)
    ref = O.Problem(cfg, build_global=False, threads=nproc)
    out.update(ndof=ref.ndof, nfree=ref.nfree, npatches=ref.npatches, p=ref.p)
    r = ref.rhs()
    u = out["units"]
    for name, fn in (("apply_St", ref.apply_St), ("apply_S", ref.apply_S), ("apply_A", ref.apply_A)):
        u[name] = timed(lambda: fn(r), reps if ref.p < 31 else 3)
        u[name]["note"] = "serial in the reference at any thread count"
        log(f"C{cfg} {name}: {u[name]['median_s']:.4f} s")
    npatch = ref.npatches
    for th in threads_list:
        key = f"threads_{th}"
        k = min(th, npatch)
        idx = np.linspace(0, npatch - 1, k).round().astype(np.int32)
        pb = O.Problem(cfg, build_global=False, threads=th)
        t = time.perf_counter()
        pb.factor(idx, threads=th)
        tf = time.perf_counter() - t
        fi = pb.factor_info(int(idx[0]))
        u[f"factor_{key}"] = {"sampled_patches": k, "wall_s": tf, "scaled_all_patches_s": tf * npatch / k,
                              "flops_per_patch_madds": fi["flops"],
                              "gflops_per_s": 2.0 * fi["flops"] * k / tf / 1e9,
                              "note": f"cholesky() of {k} patches on {th} threads (one rep), scaled by {npatch}/{k}"}
        log(f"C{cfg} factor {key}: {tf:.2f} s for {k} patches")
        rt = pb.apply_St(r)
        sm = timed(lambda: pb.patch_apply(rt), reps)
        t_st, t_s = u["apply_St"]["median_s"], u["apply_S"]["median_s"]
        t_smooth = t_st + t_s + sm["median_s"] * npatch / k
        u[f"smooth_{key}"] = {"patch_stage_sampled": sm, "sampled_patches": k,
                              "smooth_s": t_smooth, "gdof_per_s": ref.nfree / t_smooth / 1e9,
                              "note": f"apply_St + apply_S (medians) + PatchSolver::apply on {k} patches x "
                                      f"{npatch}/{k}"}
        log(f"C{cfg} smooth {key}: {t_smooth:.4f} s = {ref.nfree / t_smooth / 1e9:.5f} GDOF/s")
        del pb
        if g is not None and ref.p < 31 and (th == nproc or npatch <= 64):
            full = O.Problem(cfg, build_global=False, threads=th)
            t = time.perf_counter()
            full.factor(threads=th)
            tfull = time.perf_counter() - t
            full.build_twolevel(calibrate=False)
            full.set_omega(g["damping"]["omega"])
            t = time.perf_counter()
            _, rep = full.pcg(r, rtol=1e-8, maxit=200)
            tp = time.perf_counter() - t
            u[f"pcg_{key}"] = {"iterations": rep["iterations"], "solve_s": tp, "factor_all_s": tfull,
                               "omega": g["damping"]["omega"],
                               "note": "pcg from zero to rtol 1e-8 with the V(1,1) preconditioner at the golden omega"}
            log(f"C{cfg} pcg {key}: {rep['iterations']} it, {tp:.2f} s (factor all {tfull:.2f} s)")
            del full
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "cpu_baseline_r2.json"))
    args = ap.parse_args()
    nproc = os.cpu_count() or 1
    res = {"host": bench.host_info(), "threads": [1, nproc], "kind": "port (oracle/, the reference needs Eigen3)",
           "method": f"median of {args.reps} after 1 warm-up (C5 transforms: 3)", "configs": []}

    def log(msg):
        print(msg, flush=True)

    for c in (int(v) for v in args.configs.split(",")):
        res["configs"].append(run_config(c, [1, nproc], args.reps, log))
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)
    print(json.dumps(res["host"]))


if __name__ == "__main__":
    main()
