"""SIPG DG oracle (oracle/sipg.cpp, Cartesian facets) pinned by the Cartesian
subset of the reference's own known-answer tests (tests/test_sipg.cpp: penalty,
nodal facet traces, transformed-system exactness and stencils, patch rows, the
Cartesian two-level run).  Not restated: the flipped / pentagon two-level
variant, the Kronecker-vs-facet-quadrature check and the CG/DG energy check
(non-Cartesian meshes).  CPU only; the device path is checked against this
oracle in tests/test_gpu_sipg.py."""
import numpy as np
import pytest

from conftest import rel


def test_sipg_penalty_coefficient(oracle):  # tests/test_sipg.cpp:41-44
    assert oracle.sipg_default_eta(3, 2) == pytest.approx(20.0)
    assert oracle.sipg_default_eta(7, 3) == pytest.approx(80.0)


def test_sipg_facet_dirichlet_nodal_trace_structure(oracle):  # tests/test_sipg.cpp:46-60
    mu, eta = 1.7, 20.0
    E, _, _, td = oracle.sipg_facet_matrices(4, 0, mu, mu, eta, +1, -1)
    d = td[1]
    assert E[4, 4] == pytest.approx(mu * (eta - 2 * d[4]))
    for i in range(4):
        assert E[i, 4] == pytest.approx(-mu * d[i]) and E[4, i] == pytest.approx(-mu * d[i])
        assert np.all(E[i, :4] == 0.0)
    _, Ei, _, _ = oracle.sipg_facet_matrices(4, 0, 1.3, 1.3, eta, +1, -1)
    assert np.abs(Ei - Ei.T).max() < 1e-13


def test_dg_transformed_exactness_and_stencils(oracle):  # tests/test_sipg.cpp:122-148
    g = oracle.DGProblem(2, 2, 4)
    _, nnz, cls = g.dense(transformed=True)
    assert set(nnz[cls == 0].tolist()) == {7}  # 3d + 1 stored entries per interior row
    A, _, _ = g.dense()
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, g.ndof)
    assert rel(g.fdm_solve(b), np.linalg.solve(A, b)) < 1e-9  # A^{-1} = S At^{-1} S^T
    g0 = oracle.DGProblem(2, 2, 4, eta=0.0)  # not coercive
    with pytest.raises(oracle.OracleError, match="not SPD"):
        g0.fdm_solve(b)


def test_dg_vertex_star_patch(oracle):  # tests/test_sipg.cpp:150-167
    p = 4
    g = oracle.DGProblem(2, 4, p)
    info = g.patch()
    assert info["n"] == (2 * p + 2) ** 2 and info["nnz"] > 0


def test_dg_two_level_cartesian(oracle):  # tests/test_sipg.cpp:169-206 (Cartesian variant)
    g = oracle.DGProblem(2, 4, 4)
    g.build()
    _, rep = g.pcg(g.rhs(), 1e-8, 200)
    assert rep["converged"] and rep["iterations"] <= 16


def test_dg_operator_symmetric_and_transform_adjoint(oracle):
    g = oracle.DGProblem(3, 2, 3)
    rng = np.random.default_rng(5)
    x, y = rng.standard_normal(g.ndof), rng.standard_normal(g.ndof)
    assert abs(y @ g.apply("A", x) - x @ g.apply("A", y)) <= 1e-12 * abs(y @ g.apply("A", x))
    assert abs(y @ g.apply("S", x) - g.apply("St", y) @ x) <= 1e-12 * np.linalg.norm(x) * np.linalg.norm(y)
