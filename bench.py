#!/usr/bin/env python3
"""Benchmark of the B200 vertex-star FDM Schwarz relaxation (BASELINE.json metric).

Workload (config.workload): BASELINE.json config C5, the largest configuration
and the one that fits one GPU (83.9 GB of patch factors in 180 GB HBM) -- 3D
Poisson on the unit cube, 8x8x8 hexes with interior vertices perturbed by
+-0.1h (seed 4), Q31 on GLL nodes, 343 interior vertex-star patches of
226,981 DOFs, 15.07 M free DOFs.  One step = one relaxation apply
TwoLevel::smooth (src/schwarz.cpp:121-123): S^T transform, 343 patch solves,
S transform.  `value` = free DOFs relaxed per second over the whole job
(GDOF/s), inputs resident in HBM; `e2e` = the same through the C-ABI
host-buffer call (fdmgpu_apply_async) with the H2D copy of r and the D2H copy
of z of every step inside the timed region.  The patch factorisation time
(the metric's second half) and a PCG solve are reported beside it, and C3
(8^3 Cartesian, Q15) as a sub-result.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl reference]

--impl reference times the CPU restatement of the reference (oracle/, the
reference itself cannot be compiled here: Eigen3 is absent) on the host
cores: S^T and S over all cells plus PatchSolver::apply on a bounded sample of
patches (one per core), scaled to all patches (see cpu_baseline.sample).
Multi-GPU (torchrun): one independent replica per rank ("replicas only",
weak scaling, no collective); value = sum of all ranks' DOFs / max time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Schwarz relaxation apply GDOF/s (FP64) + % HBM roofline; patch factorization time"
# measured: tools/probe/fp64_peak.cu on this pool, DMMA 37.09 / DFMA 36.54 TFLOP/s at 1965 MHz
# (profiles/r2a_fp64_peak.txt, with the clocks sampled during the run); MEASURED_PEAKS.json has no FP64 entry
FP64_PEAK_TFLOPS = 37.0
READ_PEAK_GBPS = 7399.3  # pure-read HBM stream on this pool's B200 (tools/probe/read_bw.cu, profiles/r3_read_bw.txt)
WORKLOADS = {
    1: "C1: 2D Poisson 8x8 quads, Q7 GLL, 49 vertex-star patches",
    2: "C2: 3D Poisson 4^3 hexes, Q7 GLL, 27 vertex-star patches",
    3: "C3: 3D Poisson 8^3 hexes, Q15 GLL, 343 vertex-star patches, RHS N(0,1) seed 2",
    4: "C4: 3D anisotropic tensor grid 8^3, kappa_K lognormal, Q15 GLL, 343 patches",
    5: "C5: 3D perturbed 8^3 hexes, Q31 GLL, 343 patches (surrogate patch solver)",
}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks / throttle reasons sampled every 50 ms during the timed region.
    Uses NVML in-process (no fork stalls the launching thread); falls back to
    nvidia-smi when NVML is unavailable."""

    def __init__(self, device):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(device))
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml:
            nv, h = self._nvml
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            names = [name for bit, name in ((nv.nvmlClocksEventReasonHwSlowdown, "hw_slowdown"),
                                            (nv.nvmlClocksEventReasonHwThermalSlowdown, "hw_thermal_slowdown"),
                                            (nv.nvmlClocksEventReasonSwThermalSlowdown, "sw_thermal_slowdown"),
                                            (nv.nvmlClocksEventReasonSwPowerCap, "sw_power_cap")) if r & bit]
            return (nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM),
                    names)
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5)
        p = [x.strip() for x in out.stdout.strip().split(",")]
        names = [n for n, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], p[2:])
                 if v.lower() == "active"]
        return float(p[0]), float(p[1]), names

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.1)  # first sample (and any setup) happens before the timed region
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted({n for s in self.samples for n in s[2]}), "samples": len(self.samples),
                "source": "nvml" if self._nvml else "nvidia-smi"}


def host_info():
    """CPU model, logical cores and RAM of the box."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 1024 ** 2, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "ram_gib": ram}


P31_FACTORED = 4  # C5: patches factored on the CPU (143 s each); the other timed patches solve with copies


def cpu_sample(config, steps, warmup, threads, sample_patches):
    """CPU restatement of the reference (oracle/) on the host cores, one bounded
    sample of the relaxation apply TwoLevel::smooth per step: apply_St and apply_S
    over all cells (serial, as src/assembly.cpp:308-342) plus PatchSolver::apply
    (src/schwarz.cpp:41-54, parallel_for over `threads`) on k of the npatch
    patches, its time scaled by npatch / k.  Both bench arms call this with the
    same arguments."""
    import numpy as np
    from oracle import oracle as O

    t0 = time.perf_counter()
    ref = O.Problem(config, build_global=False, threads=threads)
    npatch = ref.npatches
    k = min(sample_patches, npatch)
    idx = np.linspace(0, npatch - 1, k).round().astype(np.int32)
    copies = ""
    if ref.p >= 31 and k > P31_FACTORED:
        # p = 31: one factorisation is 8.66e10 multiply-adds (~143 s on one core);
        # factor P31_FACTORED of the sampled patches, the others solve with copies
        # of those factors (same structure and bytes streamed per solve)
        ref.factor(idx[:P31_FACTORED], threads=P31_FACTORED)
        for i in range(P31_FACTORED, k):
            ref.copy_factor(int(idx[i % P31_FACTORED]), int(idx[i]))
        copies = (f"; {P31_FACTORED} of them factored on the CPU, the other {k - P31_FACTORED} solve with copies "
                  f"of those factors (identical structure, same bytes per solve)")
    else:
        ref.factor(idx, threads=threads)
    setup_s = time.perf_counter() - t0
    r = ref.rhs()
    times = []
    for it in range(warmup + steps):
        t = time.perf_counter()
        rt = ref.apply_St(r)
        t_st = time.perf_counter() - t
        t = time.perf_counter()
        ref.patch_apply(rt)
        t_patch = time.perf_counter() - t
        t = time.perf_counter()
        ref.apply_S(rt)
        t_s = time.perf_counter() - t
        if it >= warmup:
            times.append(t_st + t_s + t_patch * npatch / k)
    t_step = statistics.median(times)
    return {
        "value": ref.nfree / t_step / 1e9,
        "unit": "GDOF/s",
        "cores": threads,
        "kind": "port",
        "sample": (f"oracle (plain-C++ restatement; the reference needs Eigen3, absent) on config C{config}: apply_St "
                   f"+ apply_S over all {ref.ncells} cells and PatchSolver::apply on {k} of {npatch} patches "
                   f"(parallel_for, {threads} threads{copies}), patch time scaled by {npatch}/{k}; median of "
                   f"{steps} steps after {warmup} warm-up"),
        "ms_per_step": t_step * 1e3,
        "ms_min": min(times) * 1e3,
        "ms_max": max(times) * 1e3,
        "setup_s": setup_s,
        "host": host_info(),
    }


def config_dict(config):
    """The `config` object both arms print (identical, so the driver's same_config holds)."""
    l2 = ("L2 flushed before every step (512 MB write outside the per-step events)" if config in (1, 2) else
          "inputs larger than L2: the packed patch factor streamed per step is GBs (>> 126 MB L2)")
    return {"workload": WORKLOADS[config], "config": config, "l2": l2}


def run_reference(args):
    from paper_2107_14758_b200.replicas import dist_env

    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    cb = cpu_sample(args.config, args.steps, args.warmup, threads, args.cpu_sample_patches or threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "GDOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cb["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config),
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "cpu_spread_ms": {"min": cb["ms_min"], "median": cb["ms_per_step"], "max": cb["ms_max"]},
        "host": cb["host"], "setup_s": cb["setup_s"],
        "e2e": {"value": cb["value"], "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def residual_roofline(prob, ms, hbm_peak):
    """one apply_A; roofline = max(Bytes/BW, Flops/FP64 peak), compute-bound for p >= 7 in 3D."""
    d, n1, nc = prob.dim, prob.p + 1, prob.ncells
    if prob.all_cartesian:
        flops = 2.0 * d * d * n1 ** (d + 1) * nc
        fdef = "2 d^2 (p+1)^(d+1) cells (the reference kron_apply count)"
    else:
        q = prob.p + 2
        flops = 18 * 2.0 * q ** d * n1 * nc
        fdef = "trilinear true form: 18 sum-factorised contractions at q = p+2, 2 q^3 (p+1) flop each, per cell"
    byts = 16.0 * prob.ndof
    t_floor = max(byts / (hbm_peak * 1e9), flops / (FP64_PEAK_TFLOPS * 1e12))
    return {"ms": ms, "bound": "fp64" if flops / FP64_PEAK_TFLOPS / 1e12 > byts / hbm_peak / 1e9 else "hbm",
            "flops": flops, "bytes": byts, "achieved_TFLOPs": flops / (ms * 1e-3) / 1e12,
            "frac": t_floor / (ms * 1e-3), "flops_def": fdef, "bytes_def": "16 ndof (read x, write y)"}


def transform_roofline(prob, ms, hbm_peak):
    """one S or S^T: 2 d (p+1)^(d+1) cells flop, 16 ndof bytes."""
    d, n1, nc = prob.dim, prob.p + 1, prob.ncells
    flops, byts = 2.0 * d * n1 ** (d + 1) * nc, 16.0 * prob.ndof
    t_floor = max(byts / (hbm_peak * 1e9), flops / (FP64_PEAK_TFLOPS * 1e12))
    return {"ms": ms, "flops": flops, "bytes": byts, "achieved_TFLOPs": flops / (ms * 1e-3) / 1e12,
            "achieved_GBps": byts / (ms * 1e-3) / 1e9, "frac": t_floor / (ms * 1e-3), "op": "apply_St"}


CPU_STEPS = 5  # CPU-leg samples in the GPU arm (median of 5 after 1 warm-up)


def solve_kernel_bytes(L, prob):
    """Algorithmic bytes of one separator solve (every launch of the patch solve):
    8 B x the matrix values the solve reads per patch (fdmgpu_layout.solve_values: Schur split
    = S~_RR^{-1} lower triangle once (or L_RR twice) + 2 x the S_FF components + S_RF + S_FR;
    full stream = 2 x separator nnz(L_j)) + 20 B x m per patch (RHS gather, solution write,
    gather map)."""
    return 8.0 * L["solve_values"] * L["npatch"] + 20.0 * L["npatch"] * L["n_interface"]


def top_kernel_bytes(L):
    """Algorithmic bytes of the top-block stage (k_schur_symv): the lower triangle of
    S~_RR^{-1} once (FDMGPU_TOP=chol: L_RR twice) + t_R read / x_R write, per patch."""
    nr = L["n_top"]
    passes = 1 if L["schur_split"] == 2 else 2
    return (8.0 * passes * nr * (nr + 1) / 2 + 16.0 * nr) * L["npatch"]


def inverse_issued_flops(L):
    """FP64 tensor-pipe flops k_schur_uinv / k_schur_ainv issue per factorisation (dense 64x64
    tile GEMMs: column J of U takes sum_{I>J} (I - J + 1), tile (I, J) of A takes nT - I)."""
    if L["schur_split"] != 2:
        return 0.0
    nt = -(-L["n_top"] // 64)
    gemms = sum(I - J + 1 for J in range(nt) for I in range(J + 1, nt)) + sum(nt - I for I in range(nt)
                                                                             for J in range(I + 1))
    return 2.0 * 64 ** 3 * gemms * L["npatch"]


def inverse_flops(L):
    """Flops of the top-block inverse per factorisation: W = L_RR^{-1} (n^3/6 multiply-adds)
    and S~_RR^{-1} = W^T W (n^3/6), n = |R|, all patches (0 for FDMGPU_TOP=chol or no split)."""
    if L["schur_split"] != 2:
        return 0.0
    return 2.0 * (L["n_top"] ** 3 / 3.0) * L["npatch"]


def factor_flops(L):
    """In-use flops of one fdmgpu_factor over all patches.  Full tile factorisation: 2 x
    CholFactor::flops of the factor in use + the top-block inverse.  Direct top block
    (fdmgpu_layout.top_direct): the full factor is never formed -- the dense Cholesky of S~_RR
    (n^3 / 3) + the inverse (2 n^3 / 3), n = |R|; the sparse assembly of S~_RR (k_schur_form) and
    the 64 x 64 component factorisations are not counted, so the fraction is a lower bound."""
    if L.get("top_direct"):
        return float(L["n_top"]) ** 3 * L["npatch"]
    return 2.0 * L["flops_ref"] * L["npatch"] + inverse_flops(L)


def factor_issued_flops(L):
    """FP64 tensor-pipe flops the factorisation issues (dense 64 x 64 tile GEMMs), all patches."""
    if L.get("top_direct"):
        nt = -(-L["n_top"] // 64)
        upd = sum(K * (nt - K) for K in range(nt))  # tile (I, K), I >= K, takes K rank-64 updates
        trsm = nt * (nt - 1) // 2                   # off-diagonal tiles times L_KK^{-1}
        return 2.0 * 64 ** 3 * (upd + trsm) * L["npatch"] + inverse_issued_flops(L)
    return L["dmma_flops"] * L["npatch"] + inverse_issued_flops(L)


def sub_measure(config, steps, warmup, stream, device):
    """Secondary configuration beside the headline (same timing rules, device-resident
    vectors, inputs larger than L2): relaxation rate, separator-solve roofline,
    factorisation time and a PCG solve."""
    import torch

    import paper_2107_14758_b200 as pkg

    prob = pkg.Problem(config)
    sol = pkg.Solver(prob, device=device, stream=stream)
    L = sol.layout()
    fac = []
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        sol.factor()
        b.record(stream)
        torch.cuda.synchronize()
        fac.append(a.elapsed_time(b))
    r = torch.from_numpy(prob.rhs()).to(torch.device("cuda", device))
    z = torch.empty_like(r)
    for _ in range(max(warmup, 3)):
        sol.smooth(r, z)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        sol.smooth(r, z)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    sol.kernel_timing(True)
    n = min(steps, 20)
    for _ in range(n):
        sol.smooth(r, z)
    torch.cuda.synchronize()
    solve_ms = sol.kernel_time("patch_solve")[0] / n
    top_ms = sol.kernel_time("top_block")[0] / n
    sol.kernel_timing(False)
    hbm_peak, _ = measured_peaks()
    kb = solve_kernel_bytes(L, prob)
    tb = top_kernel_bytes(L)
    cal = sol.calibrate_damping()
    _, rep = sol.pcg(r, rtol=1e-8, maxit=200)
    fac_flops = factor_flops(L)
    return {"workload": WORKLOADS[config], "value": prob.nfree / (ms * 1e-3) / 1e9, "unit": "GDOF/s",
            "ms_per_step": ms, "steps": steps,
            "roofline": {"kernel": "k_schur_symv (S~_RR^{-1} product)" if L["schur_split"] == 2 else
                         "k_patch_solve on L_RR" if L["schur_split"] else
                         "k_patch_solve (+ split tail)",
                         "achieved": (tb if L["schur_split"] else kb) / ((top_ms if L["schur_split"] else solve_ms)
                                                                          * 1e-3) / 1e9,
                         "peak": hbm_peak, "unit": "GB/s",
                         "frac": (tb if L["schur_split"] else kb) / ((top_ms if L["schur_split"] else solve_ms)
                                                                     * 1e-3) / 1e9 / hbm_peak,
                         "kernel_ms": top_ms if L["schur_split"] else solve_ms,
                         "algorithmic_bytes": tb if L["schur_split"] else kb},
            "solve_roofline": {"ms": solve_ms, "algorithmic_bytes": kb, "achieved": kb / (solve_ms * 1e-3) / 1e9,
                               "frac": kb / (solve_ms * 1e-3) / 1e9 / hbm_peak},
            "factor_ms": min(fac),
            "factor_fp64_frac": fac_flops / (min(fac) * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
            "factor_issued_frac": factor_issued_flops(L) / (min(fac) * 1e-3) / 1e12
            / FP64_PEAK_TFLOPS,
            "pcg": {"iterations": rep["iterations"], "converged": rep["converged"], "omega": cal["omega"],
                    "solve_s": rep["wall_time"]}}


def run_ours(args):
    import numpy as np
    import torch

    import paper_2107_14758_b200 as pkg
    from paper_2107_14758_b200 import replicas

    rank, world, local = replicas.dist_env()
    torch.cuda.set_device(local)
    replicas.init("nccl")
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    t0 = time.perf_counter()
    prob = pkg.Problem(args.config)
    sol = pkg.Solver(prob, device=local, stream=stream)
    setup_s = time.perf_counter() - t0
    L = sol.layout()

    # ---- patch factorisation (the metric's second half) ----
    fac_ms = []
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        sol.factor()
        e1.record(stream)
        torch.cuda.synchronize()
        fac_ms.append(e0.elapsed_time(e1))
    factor_ms = min(fac_ms)

    r = torch.from_numpy(prob.rhs()).to(dev)
    z = torch.empty_like(r)
    for _ in range(args.warmup):
        sol.smooth(r, z)
    torch.cuda.synchronize()

    # ---- timed region: K relaxation applies, device-resident vectors ----
    # Working sets that fit in L2 (C1/C2) are flushed before every step (a
    # 512 MB write outside the per-step events); C3-C5 stream more than L2.
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    working_set = 2 * L["stream_bytes"] + 4 * 8 * prob.ndof
    flush = working_set < 2 * l2_bytes
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush else None
    replicas.barrier()
    torch.cuda.synchronize()
    launches0 = sol.launch_count()
    with ClockSampler(local) as clk:
        if flush:
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
            for a, b in ev:
                flush_buf.zero_()
                a.record(stream)
                sol.smooth(r, z)
                b.record(stream)
            torch.cuda.synchronize()
            ms = sum(a.elapsed_time(b) for a, b in ev)
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                sol.smooth(r, z)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
    gpu_launches = sol.launch_count() - launches0
    l2_note = (f"L2 flushed before every step (512 MB write outside the per-step events): working set "
               f"{working_set / 1e6:.1f} MB < 2 x L2" if flush else
               f"inputs larger than L2: 2 x {L['stream_bytes'] / 1e9:.2f} GB packed patch factor streamed per step")

    # ---- residual evaluation (apply_A) and basis transform (apply_St), device vectors ----
    def timed(fn, n):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n
    n_op = max(5, min(args.steps, 50))
    a_ms = timed(lambda: sol.apply_A(r, z), n_op)
    st_ms = timed(lambda: sol.apply_St(r, z), n_op)
    # per-kernel durations for the roofline: a second pass with CUDA events around
    # every library launch on the library's stream (kept out of the timed region
    # above, whose kernels chain with programmatic dependent launch)
    sol.kernel_timing(True)
    n_timed = min(args.steps, 20)
    for _ in range(n_timed):
        sol.smooth(r, z)
    torch.cuda.synchronize()
    solve_ms, solve_n = sol.kernel_time("patch_solve")
    top_ms, top_n = sol.kernel_time("top_block")
    tr_ms, tr_n = sol.kernel_time("transform")
    sol.kernel_timing(False)
    ms = replicas.max_over_ranks(ms, dev)
    ms_per_step = ms / args.steps
    value = replicas.whole_job_rate(prob.nfree, world, ms_per_step * 1e-3) / 1e9

    # ---- e2e through the C ABI with host buffers (H2D + D2H inside) ----
    h_in = torch.from_numpy(prob.rhs()).pin_memory().numpy()
    h_out = torch.empty(prob.ndof, dtype=torch.float64).pin_memory().numpy()
    sol.apply(pkg.OP_SMOOTH, h_in, h_out)
    torch.cuda.synchronize()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ee0.record(stream)
    for _ in range(args.steps):
        sol.apply(pkg.OP_SMOOTH, h_in, h_out)
    ee1.record(stream)
    torch.cuda.synchronize()
    e2e_sync_ms = ee0.elapsed_time(ee1) / args.steps
    # e2e: the stream form of the same host-buffer call (fdmgpu_apply_async): every
    # step still copies its r in and its z out (pinned), on copy streams that overlap
    # the neighbouring steps' compute
    h_outs = [torch.empty(prob.ndof, dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
    for k in range(2):
        sol.apply_async(pkg.OP_SMOOTH, h_in, h_outs[k])
    sol.synchronize()
    ee0.record(stream)
    for k in range(args.steps):
        sol.apply_async(pkg.OP_SMOOTH, h_in, h_outs[k & 1])
    sol.async_join()
    ee1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = ee0.elapsed_time(ee1) / args.steps
    e2e_ms = replicas.max_over_ranks(e2e_ms, dev)
    e2e_sync_ms = replicas.max_over_ranks(e2e_sync_ms, dev)

    # ---- PCG solve (for context: iteration count, time) ----
    pcg = None
    if not args.no_pcg:
        t = time.perf_counter()
        cal = sol.calibrate_damping()
        cal_s = time.perf_counter() - t
        x, rep = sol.pcg(r, rtol=1e-8, maxit=200)
        pcg = {"iterations": rep["iterations"], "converged": rep["converged"], "kappa": rep["kappa"],
               "solve_s": rep["wall_time"], "calibrate_s": cal_s, "omega": cal["omega"]}

    hbm_peak, peak_src = measured_peaks()
    traffic = None  # ncu dram bytes per launch (profiles/ncu_traffic.json, committed from a --set full capture)
    try:
        tr = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")))
        ent = tr.get(str(args.config))
        want = "k_schur_symv" if L["schur_split"] == 2 else "k_patch_solve"
        if ent and str(ent.get("kernel", "")).startswith(want):
            traffic = float(ent["dram_bytes_read"] + ent["dram_bytes_write"])
    except (OSError, ValueError, KeyError):
        traffic = None
    nnz_total = L["nnz_L_reference"] * L["npatch"]  # reference patch_ordering factor (SURVEY.md Bytes_relax)
    # separator columns of the factor the kernel streams (order in use; interior columns are never stored)
    solve_bytes = solve_kernel_bytes(L, prob)
    solve_kms = solve_ms / n_timed  # every launch of the separator solve (one timed interval)
    inv_top = L["schur_split"] == 2
    if L["schur_split"]:
        # dominant kernel: the top-block stage of the Schur split
        kern_bytes = top_kernel_bytes(L)
        kern_ms = top_ms / n_timed
        solve_kernels = ("k_schur_symv (S~_RR^{-1} symmetric product, chunk-parallel)" if inv_top else
                         "k_patch_solve (+ split tail) on L_RR")
        bytes_def = ("8 B x |R|(|R|+1)/2 (lower triangle of S~_RR^{-1}, streamed once) + t_R read / x_R write, "
                     "per patch, all patches" if inv_top else
                     "16 B x nnz(L_RR) (fwd + bwd) + t_R read / x_R write, per patch, all patches")
    else:
        kern_bytes, kern_ms = solve_bytes, solve_kms
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        split = L["tile_cols"] >= 16 and L["npatch"] % nsm != 0 and os.environ.get("FDMGPU_SOLVE_CS") != "1"
        solve_kernels = "k_patch_solve + k_patch_solve_cl (split tail, overlapped)" if split else "k_patch_solve"
        bytes_def = ("16 B x separator nnz(L_j) of the factor in use (fwd + bwd; plane-by-plane separator order) "
                     "+ separator RHS gather / solution write, per launch, all patches")
    achieved = kern_bytes / (kern_ms * 1e-3) / 1e9
    relax_bytes = 8.0 * (2 * nnz_total + 2 * prob.sum_nj + 4 * prob.ndof)  # SURVEY.md §8(d) Bytes_relax
    fac_flops = factor_flops(L)  # factor in use (+ top-block inverse), or the direct top block's dense work
    fac_flops_refeq = 2.0 * L["flops_reference"] * L["npatch"]  # reference patch_ordering factor
    result = {
        "metric": METRIC, "value": value, "unit": "GDOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config),
        "sizes": {"ndof": prob.ndof, "nfree": prob.nfree, "patches": L["npatch"], "patch_dofs": L["n"],
                  "separator_dofs": L["n_interface"], "parallelism": "replicas" if world > 1 else "single",
                  "l2": l2_note},
        "roofline": {"kernel": solve_kernels, "bound": "hbm", "achieved": achieved, "peak": hbm_peak,
                     "unit": "GB/s", "frac": achieved / hbm_peak, "frac_nominal_8TBps": achieved / 8000.0,
                     "read_peak": READ_PEAK_GBPS, "frac_of_read_peak": achieved / READ_PEAK_GBPS,
                     "read_peak_source": "tools/probe/read_bw.cu: 16 GiB read by 32 KB cp.async.bulk chunks, "
                                         "6-stage ring, one CTA per SM (profiles/r3_read_bw.txt); `peak` is "
                                         "MEASURED_PEAKS' copy (read + write)",
                     "traffic": traffic,
                     "peak_source": peak_src, "kernel_ms": kern_ms, "algorithmic_bytes": kern_bytes,
                     "share_of_step": kern_ms / ms_per_step if ms_per_step > 0 else None,
                     "bytes_def": bytes_def,
                     "stored_bytes_per_pass": L["stream_bytes"]},
        "solve_roofline": {
            "kernels": "every launch of the separator solve (Schur split: S_FF components, S_RF / S_FR products, "
                       "top block, partial sums)" if L["schur_split"] else solve_kernels,
            "ms": solve_kms, "algorithmic_bytes": solve_bytes, "achieved": solve_bytes / (solve_kms * 1e-3) / 1e9,
            "peak": hbm_peak, "unit": "GB/s", "frac": solve_bytes / (solve_kms * 1e-3) / 1e9 / hbm_peak,
            "share_of_step": solve_kms / ms_per_step if ms_per_step > 0 else None,
            "bytes_def": "8 B x fdmgpu_layout.solve_values x patches + 20 B x m x patches"},
        "relaxation_reference_equivalent": {
            "bytes": relax_bytes, "rate_GBps": relax_bytes / (ms_per_step * 1e-3) / 1e9,
            "note": "not a roofline fraction: SURVEY.md 8(d) Bytes_relax = 8*(2*NNZ + 2*sum n_j + 4*ndof) with NNZ of "
                    "the reference patch_ordering factor, divided by this path's step, which streams a smaller "
                    "factor (plane-by-plane separator order, interior columns eliminated in the cell kernels)"},
        "residual_roofline": residual_roofline(prob, a_ms, hbm_peak),
        "transform_roofline": transform_roofline(prob, st_ms, hbm_peak),
        "factor_ms": factor_ms,
        "factor_roofline": {"bound": "fp64", "achieved": fac_flops / (factor_ms * 1e-3) / 1e12,
                            "issued_TFLOPs": factor_issued_flops(L) / (factor_ms * 1e-3) / 1e12,
                            "issued_frac": factor_issued_flops(L) / (factor_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                            "issued_def": "FP64 tensor-pipe flops the tile kernels issue (dense 64x64 tile GEMMs "
                                          "minus skipped zero 16-wide panels; fdmgpu_layout.dmma_flops), not "
                                          "counting the diagonal-tile POTRF/inverse",
                            "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                            "frac": fac_flops / (factor_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                            "flops_def": ("direct top block: dense Cholesky of S~_RR (|R|^3 / 3) + its inverse "
                                          "(2 |R|^3 / 3) per patch; the sparse assembly of S~_RR and the component "
                                          "factorisations are not counted (lower bound)") if L.get("top_direct") else
                                         ("2 x CholFactor::flops (src/cholesky.cpp:74) of the factor in use, summed "
                                          "over patches, + the top-block inverse (W = L_RR^{-1}, W^T W: 2 |R|^3 / 3 "
                                          "per patch; 0 with FDMGPU_TOP=chol)"),
                            "top_direct": int(L.get("top_direct", 0)),
                            "inverse_flops": inverse_flops(L),
                            "reference_equivalent_TFLOPs": fac_flops_refeq / (factor_ms * 1e-3) / 1e12},
        "e2e": {"value": world * prob.nfree / (e2e_ms * 1e-3) / 1e9, "unit": "GDOF/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 8 * prob.ndof, "d2h_bytes_per_step": 8 * prob.ndof,
                "api": "fdmgpu_apply_async(OP_SMOOTH, pinned host r, pinned host z) per step, copies on copy "
                       "streams overlapping neighbouring steps",
                "sync_value": world * prob.nfree / (e2e_sync_ms * 1e-3) / 1e9, "sync_ms_per_step": e2e_sync_ms,
                "sync_api": "fdmgpu_apply(OP_SMOOTH, host=1): the LinOp drop-in, copy in / compute / copy out serialised"},
        "gpu_launches": gpu_launches,
        "clocks": clk.summary(),
        "setup_s": setup_s,
        "pcg": pcg,
    }
    if rank == 0 and world == 1 and args.config == 5 and not args.no_sub:
        # C3 (8^3 Cartesian, Q15) kept beside the C5 headline
        try:
            del sol
            torch.cuda.empty_cache()
            result["sub_results"] = {"C3": sub_measure(3, min(args.steps, 50), args.warmup, stream, local)}
        except Exception as ex:  # reported, not fatal for the headline line
            result["sub_results"] = {"C3": {"failed": str(ex)}}
    if rank == 0 and world == 1 and not args.no_elastic:
        # the widened row, reported beside the headline: 3D elasticity,
        # 8^3 cells, vector Q15 (bench.py --elastic 3,8,15,1 gives the full line)
        try:
            sol = None
            torch.cuda.empty_cache()
            e = elastic_measure("3,8,15,1", min(args.steps, 20), args.warmup, True)
            result["elasticity"] = {
                "workload": e["config"]["workload"], "value": e["value"], "unit": e["unit"],
                "ms_per_step": e["ms_per_step"], "apply_A_kernel_ms": e["residual_roofline"]["kernel_ms"],
                "apply_A_fp64_frac": e["residual_roofline"]["frac"], "factor_ms": e["factor_ms"],
                "pcg_iterations": e["pcg"]["iterations"], "e2e": e["e2e"]["value"]}
        except Exception as ex:  # reported, not fatal for the headline line
            result["elasticity"] = {"failed": str(ex)}
        # the DG half of SURVEY.md 8(f)3: SIPG two-level solver, 3D 4^3 cells, DG Q5
        try:
            result["sipg"] = sipg_measure("3,4,5", min(args.steps, 20), args.warmup)
        except Exception as ex:
            result["sipg"] = {"failed": str(ex)}
    # the CPU leg last (its host threads and memory do not disturb the GPU sub-lines' host
    # copies), on rank 0 of single-GPU runs only
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            cb = cpu_sample(args.config, CPU_STEPS, 1, threads, args.cpu_sample_patches or threads)
            result["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            result["cpu_spread_ms"] = {"min": cb["ms_min"], "median": cb["ms_per_step"], "max": cb["ms_max"]}
            result["host"] = cb["host"]
        except Exception as e:  # reported, not fatal for the GPU line
            result["cpu_baseline"] = {"value": None, "unit": "GDOF/s", "cores": os.cpu_count(), "kind": "port",
                                      "sample": f"failed: {e}"}
    replicas.barrier()
    replicas.finalize()
    if rank == 0:
        print(json.dumps(result), flush=True)
    return 0


def elastic_flops(prob):
    """kron_apply count of elasticity_primal_operator (src/elasticity.cpp:83-119): per cell d^2 diagonal-block
    terms + 2 d (d-1) cross-block terms, each d contractions of 2 (p+1)^(d+1) flop."""
    d, n1 = prob.dim, prob.p + 1
    return 2.0 * n1 ** (d + 1) * d * (d * d + 2 * d * (d - 1)) * prob.ncells


def run_elastic(args):
    """Linear-elasticity workload: the SDC/FDM relaxation of build_elasticity_twolevel on the
    reference's Table-2 problem in 3D (--elastic DIM,N,P,LAMBDA).  Same timing rules as the main line."""
    print(json.dumps(elastic_measure(args.elastic, args.steps, args.warmup, args.no_cpu)), flush=True)
    return 0


def elastic_measure(spec, steps, warmup, no_cpu):
    import numpy as np
    import torch

    import paper_2107_14758_b200 as pkg

    class _A:
        pass

    args = _A()
    args.steps, args.warmup, args.no_cpu = steps, max(warmup, 3), no_cpu
    dim, n, p, lam = (float(v) for v in spec.split(","))
    dim, n, p = int(dim), int(n), int(p)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    t0 = time.perf_counter()
    prob = pkg.Problem.elasticity(dim, n, p, 1.0, lam)
    sol = pkg.Solver(prob, device=0, stream=stream)
    setup_s = time.perf_counter() - t0
    L = sol.layout()

    def ev_time(fn, reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    factor_ms = min(ev_time(sol.factor, 1) for _ in range(2))
    r = torch.from_numpy(prob.rhs()).to(dev)
    z = torch.empty_like(r)
    for _ in range(args.warmup):
        sol.smooth(r, z)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    working_set = 2 * L["stream_bytes"] + 4 * 8 * prob.ndof
    flush = working_set < 2 * l2_bytes
    flush_buf = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if flush else None
    launches0 = sol.launch_count()
    with ClockSampler(0) as clk:
        if flush:
            ms = 0.0
            for _ in range(args.steps):
                flush_buf.zero_()
                ms += ev_time(lambda: sol.smooth(r, z), 1)
        else:
            ms = ev_time(lambda: sol.smooth(r, z), args.steps) * args.steps
    gpu_launches = sol.launch_count() - launches0
    ms_per_step = ms / args.steps
    n_op = max(5, min(args.steps, 50))
    for _ in range(3):
        sol.apply_A(r, z)
    a_ms = ev_time(lambda: sol.apply_A(r, z), n_op)
    sol.kernel_timing(True)
    for _ in range(n_op):
        sol.apply_A(r, z)
    torch.cuda.synchronize()
    ak_ms, ak_n = sol.kernel_time("stiffness")
    sol.kernel_timing(False)
    h_in = torch.from_numpy(prob.rhs()).pin_memory().numpy()
    h_out = torch.empty(prob.ndof, dtype=torch.float64).pin_memory().numpy()
    sol.apply(pkg.OP_SMOOTH, h_in, h_out)
    e2e_sync_ms = ev_time(lambda: sol.apply(pkg.OP_SMOOTH, h_in, h_out), args.steps)
    h_outs = [h_out, torch.empty(prob.ndof, dtype=torch.float64).pin_memory().numpy()]
    sol.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for k in range(args.steps):
        sol.apply_async(pkg.OP_SMOOTH, h_in, h_outs[k & 1])
    sol.async_join()
    a1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a0.elapsed_time(a1) / args.steps
    t = time.perf_counter()
    cal = sol.calibrate_damping()
    cal_s = time.perf_counter() - t
    x, rep = sol.pcg(r, rtol=1e-8, maxit=600)
    flops = elastic_flops(prob)
    hbm_peak, peak_src = measured_peaks()
    result = {
        "metric": "Elasticity SDC relaxation apply GDOF/s (FP64)", "value": prob.nfree / (ms_per_step * 1e-3) / 1e9,
        "unit": "GDOF/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"elasticity (Table-2 problem, tests/test_elasticity.cpp:157-185) dim {dim}, {n}^{dim} "
                               f"cells, vector Q{p}, mu 1, lambda {lam:g}, boundary stars included",
                   "ndof": prob.ndof, "nfree": prob.nfree, "patches": L["npatch"], "components": prob.ncomp,
                   "l2": "L2 flushed before every step" if flush else
                         f"inputs larger than L2: 2 x {L['stream_bytes'] / 1e9:.2f} GB packed factors per step"},
        "residual_roofline": {"kernel": "k_cells_elastic (+ per-component k_gather)", "bound": "fp64",
                              "op_ms": a_ms, "kernel_ms": ak_ms / max(ak_n, 1), "flops": flops,
                              "achieved_TFLOPs": flops / (ak_ms / max(ak_n, 1) * 1e-3) / 1e12,
                              "peak": FP64_PEAK_TFLOPS,
                              "frac": flops / (ak_ms / max(ak_n, 1) * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                              "flops_def": "kron_apply count: d^2 + 2d(d-1) Kronecker terms x d contractions x "
                                           "2 (p+1)^(d+1) flop per cell"},
        "factor_ms": factor_ms,
        "e2e": {"value": prob.nfree / (e2e_ms * 1e-3) / 1e9, "unit": "GDOF/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": 8 * prob.ndof, "d2h_bytes_per_step": 8 * prob.ndof,
                "api": "fdmgpu_apply_async (copies overlapped across steps)",
                "sync_value": prob.nfree / (e2e_sync_ms * 1e-3) / 1e9, "sync_api": "fdmgpu_apply(host=1)"},
        "gpu_launches": gpu_launches, "clocks": clk.summary(), "setup_s": setup_s, "peak_source": peak_src,
        "pcg": {"iterations": rep["iterations"], "converged": rep["converged"], "kappa": rep["kappa"],
                "solve_s": rep["wall_time"], "calibrate_s": cal_s, "omega": cal["omega"]},
    }
    if not args.no_cpu:
        from oracle import oracle as O

        # bounded CPU sample: the oracle's elasticity path (global SDC assembly, vector patch
        # factors) on the 3D problem with 3^3 cells at the same p, timed smooth
        try:
            threads = os.cpu_count() or 1
            ref = O.ElasticProblem(dim, 3, p, 1.0, lam, threads=threads)
            ref.build(calibrate=False)
            rr = ref.rhs()
            ts = []
            for _ in range(3):
                t = time.perf_counter()
                ref.op("smooth", rr)
                ts.append(time.perf_counter() - t)
            result["cpu_baseline"] = {"value": ref.nfree / statistics.median(ts) / 1e9, "unit": "GDOF/s",
                                      "cores": threads, "kind": "port",
                                      "sample": f"oracle elasticity smooth on dim {dim}, 3^{dim} cells, Q{p} "
                                                f"(parallel_for over patches, {threads} threads), median of 3"}
        except Exception as e:
            result["cpu_baseline"] = {"value": None, "sample": f"failed: {e}"}
    return result


def sipg_measure(spec, steps, warmup):
    """SIPG-DG workload (src/sipg.cpp): the two-level DG solver of
    tests/test_sipg.cpp:184-197 on dq_space(unit DIM-cube, N^DIM cells, Q_P), weak
    Dirichlet, default penalty; one step = one relaxation apply (S, the DG vertex-star
    patch solves with (2P+2)^DIM DOFs each, S^T), device-resident vectors."""
    import torch

    import paper_2107_14758_b200 as pkg

    dim, n, p = (int(v) for v in spec.split(","))
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    prob = pkg.Problem.sipg(dim, n, p)
    sol = pkg.Solver(prob, device=0, stream=stream)
    L = sol.layout()

    def ev_time(fn, reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    factor_ms = min(ev_time(sol.factor, 1) for _ in range(2))
    r = torch.from_numpy(prob.rhs()).to(dev)
    z = torch.empty_like(r)
    for _ in range(max(warmup, 3)):
        sol.smooth(r, z)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    ms = 0.0
    for _ in range(steps):  # L2 flushed before every step (the DG factors of small meshes fit in L2)
        flush.zero_()
        ms += ev_time(lambda: sol.smooth(r, z), 1)
    ms /= steps
    a_ms = ev_time(lambda: sol.apply_A(r, z), max(5, min(steps, 50)))
    cal = sol.calibrate_damping()
    _, rep = sol.pcg(r, rtol=1e-8, maxit=200)
    return {"workload": f"SIPG DG (src/sipg.cpp) dim {dim}, {n}^{dim} cells, DG Q{p}, eta (p+1)(p+d), "
                        f"{prob.npatches} vertex stars of {L['n']} DOFs", "value": prob.nfree / (ms * 1e-3) / 1e9,
            "unit": "GDOF/s", "ms_per_step": ms, "l2": "flushed before every step", "apply_A_ms": a_ms,
            "factor_ms": factor_ms, "factor_nnz_per_patch": L["nnz_L"],
            "pcg": {"iterations": rep["iterations"], "converged": rep["converged"], "omega": cal["omega"]}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample-patches", type=int, default=0, help="patches in the CPU sample (0: one per core)")
    ap.add_argument("--no-sub", action="store_true", help="skip the C3 sub-result of the default C5 run")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--elastic", default=None, help="DIM,N,P,LAMBDA: linear-elasticity workload (SURVEY.md 8(f)3)")
    ap.add_argument("--no-elastic", action="store_true", help="skip the elasticity and SIPG sub-lines of the default run")
    ap.add_argument("--sipg", default=None, help="DIM,N,P: SIPG-DG workload (SURVEY.md 8(f)3)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    if args.elastic:
        return run_elastic(args)
    if args.sipg:
        print(json.dumps(sipg_measure(args.sipg, args.steps, args.warmup)), flush=True)
        return 0
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
