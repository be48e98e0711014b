"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle on
the same seeded inputs, at sizes the oracle finishes in seconds, against the
golden fixtures at full size, plus size-independent properties.

Tolerances (BASELINE.json north star / SURVEY.md §7.4):
  patch solve, relaxation, V-cycle: rel-l2 <= 1e-11;  S, S^T, A: rel-l2 <= 1e-12;
  PCG: identical iteration counts at rtol 1e-8; omega rel <= 1e-10;
  index maps: bit-exact (tests/test_host_maps.py).
"""
import glob
import json
import os

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu
TOL_RELAX = 1e-11
TOL_TRANSFORM = 1e-12

CASES = [(1, 0, 0), (2, 0, 0), (2, 3, 3), (1, 4, 5), (4, 4, 5), (3, 3, 5), (4, 0, 3), (3, 2, 15), (4, 3, 15)]


@pytest.fixture(scope="module")
def torch():
    import torch as T

    assert T.cuda.is_available(), "GPU tests need a CUDA device"
    return T


@pytest.fixture(scope="module", params=CASES, ids=lambda c: "C%d_n%d_p%d" % c)
def pair(request, pkg, oracle, torch):
    cfg = request.param
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob)
    sol.factor()
    ref = oracle.Problem(*cfg, build_global=True, threads=os.cpu_count())
    ref.factor()
    return prob, sol, ref


def test_operators_match_oracle(pair, torch):
    prob, sol, ref = pair
    r = prob.rhs()
    assert rel(sol.apply_St(r), ref.apply_St(r)) <= TOL_TRANSFORM
    assert rel(sol.apply_S(r), ref.apply_S(r)) <= TOL_TRANSFORM
    assert rel(sol.apply_A(r), ref.apply_A(r)) <= TOL_TRANSFORM
    rt = ref.apply_St(r)
    assert rel(sol.patch_apply(rt), ref.patch_apply(rt)) <= TOL_RELAX
    assert rel(sol.smooth(r), ref.smooth(r)) <= TOL_RELAX
    # device path equals the host-buffer (LinOp drop-in) path bitwise
    d = torch.from_numpy(r).cuda()
    assert np.array_equal(sol.smooth(d).cpu().numpy(), sol.smooth(r))


def test_two_level_and_pcg_match_oracle(pair, torch):
    prob, sol, ref = pair
    w = sol.calibrate_damping()
    ref.build_twolevel()
    tl = ref.twolevel_info()
    assert abs(w["omega"] - tl["omega"]) <= 1e-10 * tl["omega"]
    assert abs(w["lambda_max"] - tl["lambda_max"]) <= 1e-10 * tl["lambda_max"]
    r = prob.rhs()
    sol.omega = tl["omega"]
    assert rel(sol.vcycle(r), ref.vcycle(r)) <= TOL_RELAX
    sol.omega = w["omega"]
    x, rep = sol.pcg(torch.from_numpy(r).cuda(), rtol=1e-8, maxit=200)
    xr, rr = ref.pcg(r, rtol=1e-8, maxit=200)
    assert rep["converged"] and rep["iterations"] == rr["iterations"]
    assert abs(rep["kappa"] - rr["kappa"]) <= 1e-8 * rr["kappa"]
    assert rel(x.cpu().numpy(), xr) <= 1e-9
    Ax = sol.apply_A(x.cpu().numpy())
    assert np.linalg.norm(Ax - r) / np.linalg.norm(r) <= 1e-8 * (1 + 1e-4)


def test_zero_in_zero_out(pair):
    prob, sol, _ = pair
    z = np.zeros(prob.ndof)
    assert np.linalg.norm(sol.smooth(z)) == 0.0 and np.linalg.norm(sol.patch_apply(z)) == 0.0


GOLDEN = {os.path.basename(p): p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.json"))}

# ---- full-size configurations against the in-process oracle (whole vectors) --------
FULL_ORACLE = [(3, 0, 0), (4, 0, 0), (5, 0, 3)]


@pytest.fixture(scope="module", params=FULL_ORACLE, ids=lambda c: "C%d_full_p%d" % (c[0], c[2]))
def full_pair(request, pkg, oracle, torch):
    cfg = request.param
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob)
    sol.factor()
    ref = oracle.Problem(*cfg, build_global=True, threads=os.cpu_count())
    ref.factor()  # C3/C4: 343 patches x 9.6e8 multiply-adds, in parallel on the host cores
    return prob, sol, ref


def test_full_size_vectors_match_oracle(full_pair, torch):
    """BASELINE.json configs C3, C4 and C5's mesh at p = 3, at full size: every
    operator, the patch solve, the relaxation and the V-cycle compared as whole
    vectors (rel-l2), and PCG to the iteration at the golden calibrated omega (the damping
    calibration itself is pinned by test_full_size_against_golden)."""
    prob, sol, ref = full_pair
    r = prob.rhs()
    rt = ref.apply_St(r)
    assert rel(sol.apply_St(r), rt) <= TOL_TRANSFORM
    assert rel(sol.apply_S(r), ref.apply_S(r)) <= TOL_TRANSFORM
    assert rel(sol.apply_A(r), ref.apply_A(r)) <= TOL_TRANSFORM
    assert rel(sol.patch_apply(rt), ref.patch_apply(rt)) <= TOL_RELAX
    assert rel(sol.smooth(r), ref.smooth(r)) <= TOL_RELAX
    ref.build_twolevel(calibrate=False)
    name = "c%d.json" % prob.config if prob.p == {3: 15, 4: 15, 5: 31}[prob.config] else "c%d_0_%d.json" % (
        prob.config, prob.p)
    w = json.load(open(GOLDEN[name]))["damping"]["omega"]  # the calibrated omega (pinned by the golden test)
    ref.set_omega(w)
    sol.omega = w
    assert rel(sol.vcycle(r), ref.vcycle(r)) <= TOL_RELAX
    x, rep = sol.pcg(torch.from_numpy(r).cuda(), rtol=1e-8, maxit=200)
    xr, rr = ref.pcg(r, rtol=1e-8, maxit=200)
    assert rep["converged"] and rep["iterations"] == rr["iterations"]
    assert abs(rep["kappa"] - rr["kappa"]) <= 1e-8 * rr["kappa"]
    assert rel(x.cpu().numpy(), xr) <= 1e-9


# ---- full-size configurations against the golden fixtures -------------------------
GOLDEN = {os.path.basename(p): p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.json"))}
FULL = [g for g in ("c3.json", "c4.json", "c1.json", "c2.json", "c5_0_3.json") if g in GOLDEN]


@pytest.mark.parametrize("name", FULL)
def test_full_size_against_golden(pkg, torch, name):
    g = json.load(open(GOLDEN[name]))
    prob = pkg.Problem(g["config"], g["n"], g["p"])
    sol = pkg.Solver(prob)
    sol.factor()
    L = sol.layout()
    assert L["nnz_L_reference"] == g["patch0"]["nnz_L"] and L["flops_reference"] == g["patch0"]["flops"]
    r = prob.rhs()
    probe = np.random.default_rng(12345).standard_normal(prob.ndof)
    for name_, v, tol in (("apply_St", sol.apply_St(r), TOL_TRANSFORM), ("apply_A", sol.apply_A(r), TOL_TRANSFORM),
                          ("smooth", sol.smooth(r), TOL_RELAX)):
        gg = g[name_]
        assert abs(np.linalg.norm(v) - gg["norm"]) <= tol * gg["norm"], name_
        assert abs(v @ probe - gg["probe_dot"]) <= 10 * tol * gg["norm"] * np.linalg.norm(probe), name_
        # values at 8 spread-out free DOFs and 64 slice norms (the first entries of
        # every config are constrained zeros, so a plain head would test nothing)
        assert np.allclose(v[g["free_idx"]], gg["free_head"], rtol=0, atol=10 * tol * gg["norm"]), name_
        blocks = np.array([np.linalg.norm(b) for b in np.array_split(v, len(gg["block_norms"]))])
        assert np.allclose(blocks, gg["block_norms"], rtol=0, atol=10 * tol * gg["norm"]), name_
    w = sol.calibrate_damping()
    assert abs(w["omega"] - g["damping"]["omega"]) <= 1e-10 * g["damping"]["omega"]
    x, rep = sol.pcg(torch.from_numpy(r).cuda(), rtol=1e-8, maxit=200)
    assert rep["iterations"] == g["pcg"]["iterations"]
    if "free_head" in g["vcycle"]:
        sol.omega = g["damping"]["omega"]
        for name_, v, tol in (("vcycle", sol.vcycle(r), TOL_RELAX), ("solution", x.cpu().numpy(), 1e-9)):
            gg = g[name_]
            assert abs(np.linalg.norm(v) - gg["norm"]) <= tol * gg["norm"], name_
            blocks = np.array([np.linalg.norm(b) for b in np.array_split(v, len(gg["block_norms"]))])
            assert np.allclose(blocks, gg["block_norms"], rtol=0, atol=10 * tol * gg["norm"]), name_


# ---- size-independent properties at full size (C3) ----------------------------------
@pytest.fixture(scope="module")
def c3(pkg, torch):
    prob = pkg.Problem(3)
    sol = pkg.Solver(prob)
    sol.factor()
    return prob, sol


def test_c3_layout_matches_appendix_a(c3):
    _, sol = c3
    L = sol.layout()
    assert (L["npatch"], L["n"], L["n_interior"], L["n_interface"]) == (343, 24389, 21952, 2437)
    # SURVEY.md Appendix A, reference patch_ordering
    assert L["nnz_L_reference"] == 1960925 and L["flops_reference"] == 956196192
    # plane-by-plane separator order (default): ~40 % fewer factor nonzeros
    assert L["separator_order"] == 0 and L["nnz_L"] == 1171423 and L["flops_ref"] == 388055724


@pytest.mark.parametrize("cfg", [(2, 0, 0), (4, 4, 5)])
def test_reference_separator_order(pkg, oracle, torch, cfg):
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob, separator_order="reference")
    sol.factor()
    L = sol.layout()
    assert L["separator_order"] == 1 and L["nnz_L"] == L["nnz_L_reference"]
    ref = oracle.Problem(*cfg, build_global=False, threads=os.cpu_count())
    ref.factor([0])
    assert L["nnz_L"] == ref.factor_info(0)["nnz"] and L["flops_ref"] == ref.factor_info(0)["flops"]
    ref.factor()
    r = prob.rhs()
    assert rel(sol.smooth(r), ref.smooth(r)) <= TOL_RELAX


def test_c3_relaxation_properties(c3, torch):
    prob, sol = c3
    rng = np.random.default_rng(7)
    con = prob.maps()["constrained"].astype(bool)
    x, y = rng.standard_normal(prob.ndof), rng.standard_normal(prob.ndof)
    x[con] = y[con] = 0
    Px, Py = sol.smooth(x), sol.smooth(y)
    assert abs(x @ Py - y @ Px) <= 1e-12 * abs(x @ Py)  # symmetric preconditioner
    assert x @ Px > 0 and y @ Py > 0  # positive definite
    a, b = 0.75, -1.5
    assert rel(sol.smooth(a * x + b * y), a * Px + b * Py) <= 1e-12  # linear
    assert np.array_equal(sol.smooth(x), Px)  # deterministic, bitwise
    A_x = sol.apply_A(x)
    assert abs(y @ A_x - x @ sol.apply_A(y)) <= 1e-12 * abs(y @ A_x)
    # S / S^T adjointness (tests/test_assembly.cpp:186-193): y^T S x = (S^T y)^T x
    Sx, Sty = sol.apply_S(x), sol.apply_St(y)
    assert abs(y @ Sx - Sty @ x) <= 1e-12 * np.linalg.norm(y) * np.linalg.norm(Sx)


def test_not_spd_reports_pivot(pkg, torch):
    prob = pkg.Problem(2, 3, 3)
    sol = pkg.Solver(prob)
    mu = prob.geometry()["mu"].copy()
    sol.set_cell_coeffs(-mu)
    with pytest.raises(pkg.NotSPDError, match="not SPD at pivot 0"):
        sol.factor()
    with pytest.raises(pkg.IndefiniteError, match="indefinite operator at iteration 1"):
        sol.pcg(torch.from_numpy(prob.rhs()).cuda(), precond=0)
    sol.set_cell_coeffs(mu)
    sol.factor()


def test_pcg_on_callers_default_stream(pkg, torch):
    # the handle runs on torch's (legacy default) stream; the PCG graph is
    # captured on a private stream and launched on the caller's
    prob = pkg.Problem(2, 3, 3)
    sol = pkg.Solver(prob, stream=torch.cuda.current_stream())
    sol.factor()
    sol.calibrate_damping()
    _, rep = sol.pcg(torch.from_numpy(prob.rhs()).cuda())
    assert rep["converged"] and rep["iterations"] == 13


def test_launch_evidence(pkg, torch):
    prob = pkg.Problem(2, 3, 3)
    sol = pkg.Solver(prob)
    sol.factor()
    n0 = sol.launch_count()
    sol.smooth(prob.rhs())
    # S^T cells, separator solve, patch gather, S cells (+ the Schur split's
    # F-block forward / R right-hand side / F-block backward launches)
    # split: + F-block forward, t_R, F-block backward, c_F launches; the inverse top block
    # (schur_split 2) adds its chunk-sum launch
    assert sol.launch_count() - n0 == 6 + {0: 0, 1: 3, 2: 5}[sol.layout()["schur_split"]]
    maps = open("/proc/self/maps").read()
    assert os.path.realpath(pkg.LIB_PATH) in maps or pkg.LIB_PATH in maps


def test_smoke(torch):
    import __graft_entry__

    __graft_entry__.smoke()


def test_p31_slab_path(pkg, oracle, torch):
    # p = 31 (C5 shape, one patch): the slab-blocked transforms (T1/T2/T3) and the
    # register-blocked quadrature operator against the oracle; the fused FDM
    # interior elimination/rebuild inside smooth against the staged per-axis path
    prob = pkg.Problem(5, 2, 31)
    sol = pkg.Solver(prob)
    sol.factor()
    r = prob.rhs()
    ref = oracle.Problem(5, 2, 31, build_global=True, threads=os.cpu_count())
    assert rel(sol.apply_St(r), ref.apply_St(r)) <= TOL_TRANSFORM
    assert rel(sol.apply_S(r), ref.apply_S(r)) <= TOL_TRANSFORM
    assert rel(sol.apply_A(r), ref.apply_A(r)) <= TOL_TRANSFORM
    z = sol.smooth(r)
    os.environ["FDMGPU_FORCE_STAGED"] = "1"
    try:
        staged = pkg.Solver(prob)
    finally:
        del os.environ["FDMGPU_FORCE_STAGED"]
    staged.factor()
    assert rel(z, staged.smooth(r)) <= TOL_RELAX


@pytest.mark.parametrize("cfg", [(5, 2, 5), (5, 2, 31)])
def test_quadrature_gemm_task_shapes_are_bitwise_equal(pkg, torch, cfg):
    # trilinear residual (k_quad_stage1..3): the 8 x 16 warp tasks (FDMGPU_QUAD_STRIP=0), the row
    # strips (1 / 2: k-loop unrolled by 2 / 4) and the variant that keeps stage 2 / 3 outputs over
    # their input (3) sum every output over k in the same order: identical bits
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob)
    r = prob.rhs()
    out = {}
    for mode in ("0", "1", "2", "3"):
        os.environ["FDMGPU_QUAD_STRIP"] = mode
        try:
            out[mode] = np.array(sol.apply_A(r), copy=True)
        finally:
            del os.environ["FDMGPU_QUAD_STRIP"]
    for mode in ("1", "2", "3"):
        assert np.array_equal(out["0"], out[mode]), mode


@pytest.mark.parametrize("cfg", [(2, 0, 0), (1, 0, 0), (5, 3, 4)])
def test_cellwise_transfer_matches_csr(pkg, torch, cfg):
    # the sum-factorised restriction / prolongation (fdmgpu_set_coarse_cells)
    # against the CSR of build_prolongation (src/schwarz.cpp:139-165)
    prob = pkg.Problem(*cfg)
    sols = []
    for mode in ("cells", "csr"):
        if mode == "csr":
            os.environ["FDMGPU_TRANSFER"] = "csr"
        try:
            s = pkg.Solver(prob)
        finally:
            os.environ.pop("FDMGPU_TRANSFER", None)
        s.factor()
        s.omega = 0.3
        sols.append(s)
    r = prob.rhs()
    assert rel(sols[0].vcycle(r), sols[1].vcycle(r)) <= 1e-13


# ---- external meshes with facet tags, boundary stars -------------
@pytest.mark.parametrize("skip", [True, False], ids=["interior_stars", "boundary_stars"])
@pytest.mark.parametrize("cfg,lfs", [((5, 3, 4), (0, 3)), ((1, 4, 5), (2,)), ((4, 3, 3), (1,)), ((5, 1, 3), (0,))])
def test_tagged_mesh_matches_oracle(pkg, oracle, torch, tmp_path, cfg, lfs, skip):
    """Neumann faces on a perturbed (or cartesian) mesh loaded from a JSON mesh
    file: every operator, the relaxation, the V-cycle and PCG against the oracle
    built from the same arrays.  skip=True (the configs' setting, SURVEY.md §8
    a7): the Neumann-face DOFs are reached only through the coarse space and
    PCG stalls exactly as the reference's does, so the first 20 iterations are
    compared.  skip=False (SolverConfig's default): boundary stars embedded in
    the patch template; PCG converges and must match to the iteration."""
    path = str(tmp_path / "m.json")
    pkg.Problem(*cfg).save_mesh(path)
    doc = json.load(open(path))
    for t in doc["facet_tags"]:
        if t["local_facet"] in lfs:
            t["tag"] = "neumann"
    json.dump(doc, open(path, "w"))
    p = cfg[2]
    prob = pkg.Problem.from_mesh_file(path, p, seed=3, skip_boundary_patches=skip)
    tags = [(t["cell"], t["local_facet"], t["tag"]) for t in doc["facet_tags"]]
    ref = oracle.Problem.from_mesh(doc["dim"], doc["vertices"], doc["cells"], p, facet_tags=tags, seed=3,
                                   build_global=True, threads=os.cpu_count(), skip_boundary_patches=skip)
    assert np.array_equal(prob.rhs(), ref.rhs()) and prob.npatches == ref.npatches and prob.sum_nj == ref.sum_nj
    sol = pkg.Solver(prob)
    sol.factor()
    ref.factor()
    r = prob.rhs()
    assert rel(sol.apply_St(r), ref.apply_St(r)) <= TOL_TRANSFORM
    assert rel(sol.apply_A(r), ref.apply_A(r)) <= TOL_TRANSFORM
    rt = ref.apply_St(r)
    assert rel(sol.patch_apply(rt), ref.patch_apply(rt)) <= TOL_RELAX
    assert rel(sol.smooth(r), ref.smooth(r)) <= TOL_RELAX
    w = sol.calibrate_damping()
    ref.build_twolevel()
    tl = ref.twolevel_info()
    assert abs(w["omega"] - tl["omega"]) <= 1e-10 * tl["omega"]
    assert rel(sol.vcycle(r), ref.vcycle(r)) <= TOL_RELAX
    maxit = 20 if skip else 200
    x, rep = sol.pcg(torch.from_numpy(r).cuda(), rtol=1e-8, maxit=maxit)
    xr, rr = ref.pcg(r, rtol=1e-8, maxit=maxit)
    assert rep["converged"] == rr["converged"] and rep["iterations"] == rr["iterations"]
    assert skip or rep["converged"]
    assert rel(x.cpu().numpy(), xr) <= 1e-9


def test_two_level_with_boundary_stars_reference_pins(pkg, oracle, torch):
    """tests/test_schwarz.cpp:93-129 (default SolverConfig: boundary stars on):
    2D 4x4, p = 3, 5, 7 -- symmetric preconditioner, contractive damped
    smoother, kappa <= 1.7, <= 11 iterations, spread <= 2; here on the device
    path, with the iteration counts matched against the oracle."""
    its = []
    for p in (3, 5, 7):
        prob = pkg.Problem(1, 4, p, skip_boundary_patches=False)
        sol = pkg.Solver(prob)
        sol.factor()
        sol.calibrate_damping()
        rng = np.random.default_rng(p)
        free = prob.maps()["constrained"] == 0
        x, y = rng.standard_normal(prob.ndof) * free, rng.standard_normal(prob.ndof) * free
        assert abs(x @ sol.vcycle(y) - y @ sol.vcycle(x)) <= 1e-10 * abs(x @ sol.vcycle(y))
        v = rng.standard_normal(prob.ndof) * free
        rho = 0.0
        for _ in range(30):
            Ev = v - sol.omega * sol.smooth(sol.apply_A(v))
            rho = np.sqrt((Ev @ sol.apply_A(Ev)) / (v @ sol.apply_A(v)))
            v = Ev / np.linalg.norm(Ev)
        assert rho < 1.0 - 1e-3
        r = prob.rhs()
        _, rep = sol.pcg(torch.from_numpy(r).cuda(), rtol=1e-8, maxit=100)
        ref = oracle.Problem(1, 4, p, threads=os.cpu_count(), skip_boundary_patches=False)
        ref.factor()
        ref.build_twolevel()
        _, rr = ref.pcg(r, rtol=1e-8, maxit=100)
        assert rep["converged"] and rep["kappa"] <= 1.7 and rep["iterations"] <= 11
        assert rep["iterations"] == rr["iterations"]
        its.append(rep["iterations"])
    assert max(its) - min(its) <= 2


@pytest.mark.parametrize("cs,tail", [("1", "1"), ("2", "0"), ("3", "0"), ("4", "0"), ("2", "1")])
def test_cluster_split_solve(pkg, oracle, torch, monkeypatch, cs, tail):
    """k_patch_solve_cl: one patch spread over a cluster of 2-4 CTAs (DSMEM
    exchange of y_K / x_K and the backward partials) against the oracle and the
    single-CTA solve; 8 patches with 39 separator tile columns (p = 15)."""
    monkeypatch.setenv("FDMGPU_SOLVE_CS", cs)
    monkeypatch.setenv("FDMGPU_SOLVE_TAIL", tail)
    prob = pkg.Problem(4, 3, 15)
    sol = pkg.Solver(prob)
    sol.factor()
    ref = oracle.Problem(4, 3, 15, build_global=False, threads=os.cpu_count())
    ref.factor()
    rt = ref.apply_St(prob.rhs())
    z = sol.patch_apply(rt)
    assert rel(z, ref.patch_apply(rt)) <= TOL_RELAX
    assert np.array_equal(z, sol.patch_apply(rt))  # deterministic


@pytest.mark.parametrize("cfg,skip", [((4, 3, 5), True), ((5, 2, 4), False), ((1, 3, 5), False)])
def test_patch_schur_matches_oracle(pkg, oracle, torch, tmp_path, cfg, skip):
    """fdmgpu_patch_schur (the matrix the batched factorisation factors) against
    the oracle's patch matrix (extract_submatrix of the assembled transformed
    matrix) with its interior block eliminated; absent positions of boundary
    stars are identity rows; the MatrixMarket dump reads back exactly."""
    import scipy.io

    prob = pkg.Problem(*cfg, skip_boundary_patches=skip)
    sol = pkg.Solver(prob)
    ref = oracle.Problem(*cfg, build_global=True, skip_boundary_patches=skip)
    L = sol.layout()
    el = sol.elimination_dofs()
    pt = ref.patches()
    for j in sorted({0, L["npatch"] // 2, L["npatch"] - 1}):
        S = sol.patch_schur(j)
        ptr, col, val = ref.patch_matrix(j)
        n = len(ptr) - 1
        A = np.zeros((n, n))
        for r in range(n):
            A[r, col[ptr[r]:ptr[r + 1]]] = val[ptr[r]:ptr[r + 1]]
        dofs = pt["dofs"][pt["ptr"][j]:pt["ptr"][j + 1]]
        pos = {int(g): i for i, g in enumerate(dofs)}
        sep = el[j, L["n_interior"]:]
        present = sep >= 0
        isep = np.array([pos[int(g)] for g in sep[present]], dtype=np.int64)
        iint = np.setdiff1d(np.arange(n), isep)
        Sref = A[np.ix_(isep, isep)] - A[np.ix_(isep, iint)] @ np.linalg.solve(A[np.ix_(iint, iint)], A[np.ix_(iint, isep)])
        assert rel(S[np.ix_(present, present)], Sref) <= 1e-12
        assert not S[np.ix_(~present, present)].any() and np.all(np.diag(S)[~present] == 1.0)
    path = str(tmp_path / "s.mtx")
    sol.export_patch_matrix(0, path)
    R = scipy.io.mmread(path)
    R = R.toarray() if hasattr(R, "toarray") else np.asarray(R)
    assert np.array_equal(R, sol.patch_schur(0))


@pytest.mark.parametrize("cfg", [(2, 3, 5), (3, 2, 15)])
def test_apply_async_matches_sync(pkg, torch, cfg):
    """fdmgpu_apply_async (copy streams, two staging slots) returns what the
    synchronous host-buffer call returns, bitwise, for a stream of distinct inputs."""
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob)
    sol.factor()
    rng = np.random.default_rng(7)
    ins = [torch.from_numpy(rng.standard_normal(prob.ndof)).pin_memory().numpy() for _ in range(5)]
    outs = [torch.empty(prob.ndof, dtype=torch.float64).pin_memory().numpy() for _ in range(5)]
    for op in (pkg.OP_SMOOTH, pkg.OP_A):
        for x, y in zip(ins, outs):
            sol.apply_async(op, x, y)
        sol.synchronize()
        for x, y in zip(ins, outs):
            assert np.array_equal(y, sol.apply(op, x)), op


def test_inplace_and_separate_packing_agree(pkg, torch, monkeypatch):
    """Solve records packed in place after the factorisation (FDMGPU_PACK=inplace) and
    packed per tile column into their own buffer during it give identical relaxations."""
    prob = pkg.Problem(2, 3, 7)
    r = prob.rhs()
    sol = pkg.Solver(prob)
    sol.factor()
    z_sep = sol.smooth(r)
    monkeypatch.setenv("FDMGPU_PACK", "inplace")
    sol2 = pkg.Solver(prob)
    sol2.factor()
    assert np.array_equal(sol2.smooth(r), z_sep)


@pytest.mark.parametrize("cfg", [(4, 3, 15), (2, 0, 0)])
def test_compact_solve_records_opt_in(pkg, oracle, torch, monkeypatch, cfg):
    """FDMGPU_COMPACT=1: sparse 8x8 sub-blocks of the solve records stored as one
    value per row (layout.cpp) give the same relaxation as the default records."""
    monkeypatch.setenv("FDMGPU_SCHUR", "0")  # the option belongs to the full-factor stream
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob)
    sol.factor()
    monkeypatch.setenv("FDMGPU_COMPACT", "1")
    comp = pkg.Solver(prob)
    comp.factor()
    assert comp.layout()["stream_bytes"] < sol.layout()["stream_bytes"]
    ref = oracle.Problem(*cfg, build_global=False, threads=os.cpu_count())
    ref.factor()
    rt = ref.apply_St(prob.rhs())
    z = comp.patch_apply(rt)
    assert rel(z, ref.patch_apply(rt)) <= TOL_RELAX
    assert rel(z, sol.patch_apply(rt)) <= 1e-13


@pytest.mark.parametrize("cfg", [(3, 3, 15), (2, 0, 0), (5, 2, 7)])
def test_fused_column_factorisation(pkg, torch, monkeypatch, cfg):
    """k_patch_column (update + diagonal factor + trsm of a tile column in one
    launch, flag-synchronised) gives the same factor, bit for bit, as the
    separate k_patch_update / k_patch_trsm launches (FDMGPU_FUSED=0)."""
    monkeypatch.setenv("FDMGPU_DIRECT", "0")  # the full separator factorisation (the direct top block skips it)
    prob = pkg.Problem(*cfg)
    r = prob.rhs()
    fused = pkg.Solver(prob)
    fused.factor()
    fused.factor()  # second factorisation: the flags' epoch advances, no reset needed
    monkeypatch.setenv("FDMGPU_FUSED", "0")
    split = pkg.Solver(prob)
    split.factor()
    assert np.array_equal(fused.smooth(r), split.smooth(r))


@pytest.mark.parametrize("cfg", [(2, 0, 0), (4, 3, 5), (5, 2, 7), (1, 4, 5)])
def test_patch_factor_residual(pkg, torch, monkeypatch, cfg):
    """K2: the device factor of sampled patches reproduces the
    matrix it factors, ||L L^T - S_G||_max / ||S_G||_max <= 1e-12 (S_G the
    separator Schur complement, fdmgpu_patch_schur), L lower triangular with a
    positive diagonal."""
    monkeypatch.setenv("FDMGPU_DIRECT", "0")  # keeps the full separator factor tiles
    prob = pkg.Problem(*cfg)
    sol = pkg.Solver(prob)
    sol.factor()
    npatch = sol.layout()["npatch"]
    for j in sorted({0, npatch // 2, npatch - 1}):
        S = sol.patch_schur(j)
        L = sol.patch_factor(j)
        assert np.array_equal(L, np.tril(L)) and (np.diag(L) > 0).all()
        assert np.abs(L @ L.T - S).max() <= 1e-12 * np.abs(S).max()
