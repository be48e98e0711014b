"""Linear elasticity with the SDC/FDM relaxation (src/elasticity.cpp).

CPU part: the oracle restatement pinned by the reference's own elasticity
known-answer tests (tests/test_elasticity.cpp): sdc coefficients, the
Cartesian Kronecker blocks against the quadrature cell matrix (1e-11), the
SDC/FDM relaxation against the dense per-patch SDC solve (1e-10), and the
Table-2 iteration counts (13, 14, 24, 70, 199 within [0.8x, 1.2x + 1],
monotone, lambda = 1000 at least 10x lambda = 0); plus the host mirror's
maps / star lists / load vector against the oracle (bit-exact maps).

GPU part (-m gpu): the sm_100a path through the C ABI against the oracle on
the same problems: true-form operator and S / S^T within 1e-12, patch solve,
relaxation and V-cycle within 1e-11, identical PCG iteration counts at rtol
1e-8, omega within 1e-10.
"""
import numpy as np
import pytest

from conftest import rel

TABLE2_LAMBDAS = [0.0, 1.0, 10.0, 100.0, 1000.0]
TABLE2_EXPECTED = [13, 14, 24, 70, 199]  # tests/test_elasticity.cpp:166


def test_sdc_coefficients(oracle):  # tests/test_elasticity.cpp:32-39
    assert np.allclose(oracle.sdc_axis_coefficients(0, 2, 1.0, 0.0), [2.0, 1.0])
    assert np.allclose(oracle.sdc_axis_coefficients(2, 3, 2.0, 5.0), [2.0, 2.0, 9.0])


@pytest.mark.parametrize("dim,n,p,mu,lam", [(2, 2, 3, 1.0, 2.5), (3, 1, 2, 1.3, 0.4)])
def test_kronecker_blocks_match_quadrature(oracle, dim, n, p, mu, lam):  # tests/test_elasticity.cpp:76-101
    e = oracle.ElasticProblem(dim, n, p, mu, lam)
    for c in range(e.ncells):
        kron, quad = e.cell_matrices(c)
        assert np.abs(kron - quad).max() < 1e-11 * np.abs(quad).max()


def test_sdc_relaxation_equals_dense_patch_solves(oracle):  # tests/test_elasticity.cpp:103-141
    e = oracle.ElasticProblem(2, 2, 3, 1.0, 0.9)
    e.build(calibrate=False)
    r = e.random_free(21)
    z = e.op("smooth", r)
    A = e.assemble_dense(sdc_only=True)
    P = e.patches()
    zo = np.zeros_like(r)
    for j in range(len(P["vertex"])):
        d = P["dofs"][P["ptr"][j]:P["ptr"][j + 1]]
        zo[d] += np.linalg.solve(A[np.ix_(d, d)], r[d])
    assert np.abs(z - zo).max() < 1e-10 * np.abs(zo).max()


def test_table2_iteration_counts(oracle):  # tests/test_elasticity.cpp:157-185
    its = []
    for lam in TABLE2_LAMBDAS:
        e = oracle.ElasticProblem(2, 8, 3, 1.0, lam)
        e.build()
        _, rep = e.pcg(e.rhs(), 1e-8, 600)
        assert rep["converged"]
        its.append(rep["iterations"])
    for k, (got, exp) in enumerate(zip(its, TABLE2_EXPECTED)):
        assert int(0.8 * exp) <= got <= int(1.2 * exp) + 1, (its, TABLE2_EXPECTED)
        if k:
            assert got >= its[k - 1]
    assert its[-1] >= 10 * its[0]


@pytest.mark.parametrize("dim,n,p,lam,skip", [(2, 8, 3, 10.0, False), (3, 3, 4, 1.0, False), (3, 2, 7, 5.0, True)])
def test_host_mirror_matches_oracle(pkg, oracle, dim, n, p, lam, skip):
    P = pkg.Problem.elasticity(dim, n, p, 1.0, lam, skip_boundary_patches=skip)
    E = oracle.ElasticProblem(dim, n, p, 1.0, lam, skip_boundary_patches=skip)
    assert P.ndof == E.ndof and P.ncomp == dim
    m, me = P.maps(), E.maps()
    for k in ("cell_dofs", "constrained", "multiplicity"):
        assert np.array_equal(m[k], me[k]), k
    assert rel(P.rhs(), E.rhs()) < 1e-14
    E.build(calibrate=False)
    pe, pp = E.patches(), P.patches()
    assert np.array_equal(pe["vertex"], pp["vertex"])
    assert np.array_equal(pe["ptr"], pp["ptr"])
    assert np.array_equal(pe["dofs"], pp["dofs"])
    assert P.ncoarse == E.twolevel_info()["ncoarse"]


# ---- GPU parity ---------------------------------------------------------------
# skip_boundary_patches=False throughout (the reference default): with Neumann
# faces, skipping the boundary stars leaves boundary DOFs outside every patch.
GPU_CASES = [(2, 8, 3, 10.0, False), (2, 4, 7, 1.0, False), (3, 3, 4, 1.0, False), (3, 2, 7, 5.0, False),
             (3, 2, 15, 2.0, False)]


@pytest.fixture(scope="module", params=GPU_CASES, ids=lambda c: "d%d_n%d_p%d_lam%g_skip%d" % c)
def epair(request, pkg, oracle):
    import os

    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    dim, n, p, lam, skip = request.param
    prob = pkg.Problem.elasticity(dim, n, p, 1.0, lam, skip_boundary_patches=skip)
    sol = pkg.Solver(prob)
    sol.factor()
    ref = oracle.ElasticProblem(dim, n, p, 1.0, lam, skip_boundary_patches=skip, threads=os.cpu_count())
    ref.build(calibrate=False)
    return prob, sol, ref


@pytest.mark.gpu
def test_elastic_operators_match_oracle(epair):
    prob, sol, ref = epair
    r = ref.random_free(21)
    assert rel(sol.apply_A(r), ref.apply_A(r)) <= 1e-12
    assert rel(sol.apply_St(r), ref.op("apply_St", r)) <= 1e-12
    assert rel(sol.apply_S(r), ref.op("apply_S", r)) <= 1e-12
    rt = ref.op("apply_St", r)
    assert rel(sol.patch_apply(rt), ref.op("patch", rt)) <= 1e-11
    assert rel(sol.smooth(r), ref.op("smooth", r)) <= 1e-11
    ref.set_omega(0.3)
    assert rel(sol.vcycle(r, omega=0.3), ref.op("vcycle", r)) <= 1e-11


@pytest.mark.gpu
def test_elastic_pcg_matches_oracle(epair):
    import torch

    prob, sol, ref = epair
    w = sol.calibrate_damping()
    ref.build(calibrate=True)
    wr = ref.twolevel_info()["omega"]
    assert abs(w["omega"] - wr) <= 1e-10 * abs(wr)
    b = prob.rhs()
    _, rep = sol.pcg(torch.from_numpy(b).cuda(), rtol=1e-8, maxit=600)
    _, rep_ref = ref.pcg(b, rtol=1e-8, maxit=600)
    assert rep["converged"] and rep["iterations"] == rep_ref["iterations"]


@pytest.mark.gpu
def test_elastic_table2_counts_on_gpu(pkg):
    import torch

    its = []
    for lam in TABLE2_LAMBDAS:
        prob = pkg.Problem.elasticity(2, 8, 3, 1.0, lam)
        sol = pkg.Solver(prob)
        sol.factor()
        sol.calibrate_damping()
        _, rep = sol.pcg(torch.from_numpy(prob.rhs()).cuda(), rtol=1e-8, maxit=600)
        assert rep["converged"]
        its.append(rep["iterations"])
    for got, exp in zip(its, TABLE2_EXPECTED):
        assert int(0.8 * exp) <= got <= int(1.2 * exp) + 1, its
    assert its == sorted(its) and its[-1] >= 10 * its[0]


@pytest.mark.gpu
def test_elastic_deterministic_and_async(pkg):
    """Two applies give bitwise-identical results (owner gathers, no atomics), and
    the asynchronous host-buffer path returns the synchronous results."""
    import torch

    prob = pkg.Problem.elasticity(3, 2, 7, 1.0, 3.0)
    sol = pkg.Solver(prob)
    sol.factor()
    r = prob.rhs() + np.random.default_rng(1).standard_normal(prob.ndof) * (prob.maps()["constrained"] == 0)
    for fn in (sol.smooth, sol.apply_A):
        assert np.array_equal(fn(r), fn(r))
    # symmetric operator and relaxation, adjoint transforms (full vector space)
    y = np.random.default_rng(2).standard_normal(prob.ndof) * (prob.maps()["constrained"] == 0)
    for fn in (sol.apply_A, sol.smooth):
        assert abs(y @ fn(r) - r @ fn(y)) <= 1e-12 * abs(y @ fn(r))
    assert abs(y @ sol.apply_S(r) - sol.apply_St(y) @ r) <= 1e-12 * np.linalg.norm(y) * np.linalg.norm(r)
    h_in = torch.from_numpy(r).pin_memory().numpy()
    outs = [torch.empty(prob.ndof, dtype=torch.float64).pin_memory().numpy() for _ in range(3)]
    for o in outs:
        sol.apply_async(pkg.OP_SMOOTH, h_in, o)
    sol.synchronize()
    ref = sol.smooth(r)
    for o in outs:
        assert np.array_equal(o, ref)


@pytest.mark.gpu
def test_elastic_handle_errors(pkg):
    """Vector handles reject what the device path does not cover, with status codes."""
    prob = pkg.Problem.elasticity(2, 3, 3, 1.0, 1.0)
    sol = pkg.Solver(prob)
    g = prob.geometry()
    with pytest.raises(pkg.FdmGpuError) as e:  # kappa is not part of the elasticity operator
        sol.set_cell_coeffs(g["mu"], kappa=np.full(prob.ncells, 2.0))
    assert e.value.status == 1
    with pytest.raises(pkg.FdmGpuError) as e:  # non-Cartesian cells need the dense quadrature form
        sol.set_cell_coeffs(g["mu"], kind=np.full(prob.ncells, 2, np.uint8))
    assert e.value.status == 6
    with pytest.raises(pkg.FdmGpuError) as e:  # scalar-only debug view
        sol.factor()
        sol.patch_schur(0)
    assert e.value.status == 6
