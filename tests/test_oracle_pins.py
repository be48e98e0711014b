"""Pins the CPU oracle (oracle/, the plain-C++ restatement of the reference)
against the reference's own known-answer tests for the hot path
(/root/reference/proj/tests/*.cpp, cited per test) and SURVEY.md Appendix A.
The reference itself cannot be compiled here (Eigen3 absent), so these
in-process pins are what make the oracle trustworthy."""
import math

import numpy as np
import pytest
import scipy.linalg as sla

from conftest import rel


def moment(k):
    return 0.0 if k % 2 else 2.0 / (k + 1)


# ---- tests/test_refelem.cpp -----------------------------------------------------
def test_gll_nodes_analytic(oracle):  # test_refelem.cpp:23-47
    assert np.allclose(oracle.gll_nodes(1), [-1, 1])
    assert oracle.gll_nodes(2)[1] == 0.0
    n3 = oracle.gll_nodes(3)
    assert abs(n3[1] + 1 / math.sqrt(5)) < 1e-14 and abs(n3[2] - 1 / math.sqrt(5)) < 1e-14
    for p in (4, 9, 16, 33, 64):
        x = oracle.gll_nodes(p)
        assert x[0] == -1.0 and x[p] == 1.0
        assert np.all(np.diff(x) > 0)
        for i in range(1, p):
            assert abs(oracle.legendre(p, x[i])[1]) < 1e-10


def test_gauss_legendre_rules(oracle):  # test_refelem.cpp:49-78
    p1, w1 = oracle.gauss_legendre(1)
    assert p1[0] == 0.0 and abs(w1[0] - 2) < 1e-15
    p2, w2 = oracle.gauss_legendre(2)
    assert abs(p2[0] + 1 / math.sqrt(3)) < 1e-15 and np.allclose(w2, 1.0)
    p3, w3 = oracle.gauss_legendre(3)
    assert abs(w3[0] - 5 / 9) < 1e-14 and abs(w3[1] - 8 / 9) < 1e-14
    for n in (5, 12, 33, 64):
        p, w = oracle.gauss_legendre(n)
        assert w.min() > 0 and abs(w.sum() - 2) < 1e-14 and np.all(np.diff(p) > 0)
        for k in (2 * n - 2, 2 * n - 1):
            assert abs(np.sum(p ** k * w) - moment(k)) < 1e-12 * max(1, abs(moment(k)))


def test_reference_operators(oracle):  # test_refelem.cpp:80-140
    A, B, _, _ = oracle.reference_operators(1)
    assert np.allclose(A, [[0.5, -0.5], [-0.5, 0.5]]) and np.allclose(B, [[2 / 3, 1 / 3], [1 / 3, 2 / 3]])
    A3, _, _, _ = oracle.reference_operators(3, kind=1)  # Lobatto hierarchical
    assert abs(A3[1, 1] - 2 / 3) < 1e-14 and abs(A3[2, 2] - 2 / 5) < 1e-14 and abs(A3[1, 2]) < 1e-14
    A7, _, _, _ = oracle.reference_operators(7, kind=1)
    for i in range(1, 7):
        for j in range(1, 7):
            assert abs(A7[i, j] - (2 / (2 * i + 1) if i == j else 0)) < 1e-13
    A7n, B7n, _, _ = oracle.reference_operators(7)
    assert np.count_nonzero(np.abs(A7n) > 1e-12) == 64 and np.count_nonzero(np.abs(B7n) > 1e-12) == 64
    for p in (2, 5, 9):
        A, B, nodes, tv = oracle.reference_operators(p)
        assert np.allclose(tv[0], np.eye(p + 1)[0]) and np.allclose(tv[1], np.eye(p + 1)[p])
        for a in range(p + 1):
            for b in range(p + 1):
                if a + b <= 2 * p:
                    assert abs((nodes ** a) @ B @ (nodes ** b) - moment(a + b)) < 1e-12
    for kind in (0, 2):
        A, _, _, _ = oracle.reference_operators(6, kind)
        assert np.abs(A @ np.ones(7)).max() < 1e-13


def test_fdm_basis_eigenvalues(oracle):  # test_refelem.cpp:142-168
    assert abs(oracle.fdm_basis(2)["lam"][0] - 2.5) < 2.5e-13
    assert abs(oracle.fdm_basis(16)["lam"][0] - math.pi ** 2 / 4) < 1e-6
    prev = None
    for p in range(4, 21):
        lam = oracle.fdm_basis(p)["lam"]
        for j in range(3):
            assert lam[j] >= (j + 1) ** 2 * math.pi ** 2 / 4 - 1e-10
            if prev is not None:
                assert lam[j] <= prev[j] + 1e-10
        prev = lam


@pytest.mark.parametrize("p", [2, 3, 5, 8, 13, 21, 32])
def test_fdm_basis_identities(oracle, p):  # test_refelem.cpp:170-226
    A, B, _, _ = oracle.reference_operators(p)
    f = oracle.fdm_basis(p)
    S, ni = f["S"], p - 1
    At, Bt = S.T @ A @ S, S.T @ B @ S
    assert np.abs(At[1:p, 1:p] - np.diag(f["lam"])).max() < 1e-9
    assert np.abs(Bt[1:p, 1:p] - np.eye(ni)).max() < 1e-10
    assert max(np.abs(Bt[1:p, [0, p]]).max(), np.abs(Bt[[0, p], 1:p]).max()) < 1e-12
    SII = S[1:p, 1:p]
    BIG = B[1:p][:, [0, p]]
    Bgg = B[np.ix_([0, p], [0, p])]
    expect = Bgg - BIG.T @ SII @ SII.T @ BIG
    assert abs(Bt[0, 0] - expect[0, 0]) < 1e-12 and abs(Bt[0, p] - expect[0, 1]) < 1e-12
    assert np.count_nonzero(f["Btnz"]) == ni + 4 and np.count_nonzero(f["Atnz"]) == 5 * ni + 4
    for i, j in zip(*np.nonzero(f["Btnz"])):
        assert (0 < i < p) == (0 < j < p) and (not (0 < i < p) or i == j)
    assert np.abs(f["At"] - At).max() < 1e-9
    for j in range(1, p):
        imax = int(np.argmax(np.abs(S[:, j])))
        assert S[imax, j] > 0


def test_fdm_basis_needs_nodal(oracle):  # test_refelem.cpp:228-231
    with pytest.raises(oracle.OracleError):
        oracle.fdm_basis(4, kind=1)


# ---- tests/test_sparsela.cpp ----------------------------------------------------
def test_dense_sym_gen_eig(oracle):  # test_sparsela.cpp:140-186
    lam, _ = oracle.dense_sym_gen_eig(np.eye(4), np.eye(4))
    assert np.abs(lam - 1).max() < 1e-14
    lam, V = oracle.dense_sym_gen_eig(np.diag([1.0, 4.0]), np.eye(2))
    assert np.allclose(lam, [1, 4]) and abs(abs(V[0, 0]) - 1) < 1e-14
    lam, _ = oracle.dense_sym_gen_eig(np.array([[2.0, 1], [1, 3]]), np.array([[2.0, 0], [0, 1]]))
    d = math.sqrt(24.0)
    assert abs(lam[0] - (8 - d) / 4) < 1e-13 and abs(lam[1] - (8 + d) / 4) < 1e-13
    rng = np.random.default_rng(5)
    M, N = rng.uniform(-1, 1, (12, 12)), rng.uniform(-1, 1, (12, 12))
    A, B = M + M.T, N @ N.T + 12 * np.eye(12)
    lam, V = oracle.dense_sym_gen_eig(A, B)
    assert np.abs(A @ V - B @ V @ np.diag(lam)).max() < 1e-10 * np.abs(A).max()
    assert np.abs(V.T @ B @ V - np.eye(12)).max() < 1e-10
    assert np.abs(lam - sla.eigh(A, B, eigvals_only=True)).max() < 1e-10
    with pytest.raises(oracle.OracleError):
        oracle.dense_sym_gen_eig(A, -B)


def random_spd(n, band, seed):  # test_sparsela.cpp:28-48 (numpy RNG stand-in)
    rng = np.random.default_rng(seed)
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - band), i):
            if abs(rng.uniform(-1, 1)) < 0.4:
                continue
            v = rng.uniform(-1, 1)
            A[i, j] = A[j, i] = v
    A += np.diag(np.abs(A).sum(1) + 1.0)
    return A


def test_cholesky_known_answers(oracle):  # test_sparsela.cpp:188-234
    L, nnz, _, _ = oracle.cholesky_dense(np.diag([4.0, 9, 16, 25]))
    assert nnz == 4 and np.allclose(np.diag(L), [2, 3, 4, 5])
    A = random_spd(30, 6, 17)
    L, _, _, _ = oracle.cholesky_dense(A)
    assert np.abs(L @ L.T - A).max() < 1e-11 and np.all(np.diag(L) > 0)
    for n in (50, 600):
        A = random_spd(n, 8, 100 + n)
        b = np.random.default_rng(n).uniform(-1, 1, n)
        _, _, _, x = oracle.cholesky_dense(A, perm=np.arange(n)[::-1], b=b)
        assert np.linalg.norm(A @ x - b) / np.linalg.norm(b) < 1e-12
    with pytest.raises(oracle.OracleError, match="pivot 1"):
        oracle.cholesky_dense(np.diag([1.0, -1.0]))


def test_patch_ordering_groups(oracle):  # test_sparsela.cpp:236-256
    cls = [3] + [1] * 12 + [0] * 36
    ent = [0] + [f for f in range(4) for _ in range(3)] + [c for c in range(4) for _ in range(9)]
    perm, offs = oracle.patch_ordering(cls, ent)
    c = np.array(cls)[perm]
    assert np.all(c[:36] == 0) and np.all(c[36:48] == 1) and c[48] == 3
    assert list(offs) == [0, 36, 39, 42, 45, 48, 49]
    with pytest.raises(oracle.OracleError):
        oracle.patch_ordering([0], [-1])


# ---- tests/test_assembly.cpp ----------------------------------------------------
def test_q_space_counts(oracle):  # test_assembly.cpp:97-116
    pb = oracle.Problem(1, 2, 3)
    assert pb.ndof == 49 and pb.nfree == 25
    assert int(np.sum(pb.maps()["multiplicity"] == 4)) == 1
    pb3 = oracle.Problem(2, 2, 2)
    assert pb3.ndof == 125 and pb3.nfree == 27


def dense_of(op, n):
    return np.stack([op(np.eye(n)[i]) for i in range(n)], axis=1)


def test_transformed_system_identities(oracle):  # test_assembly.cpp:149-229
    pb = oracle.Problem(1, 2, 3)  # 2x2 unit square, p = 3
    rng = np.random.default_rng(1)
    con = pb.maps()["constrained"].astype(bool)
    x, y = rng.uniform(-1, 1, pb.ndof), rng.uniform(-1, 1, pb.ndof)
    x[con] = y[con] = 0
    assert abs(y @ pb.apply_S(x) - pb.apply_St(y) @ x) < 1e-12 * abs(y @ pb.apply_S(x))
    # A^{-1} = S At^{-1} S^T against a dense solve on the free block
    A = dense_of(pb.apply_A, pb.ndof)
    assert np.abs(A - A.T).max() < 1e-13
    b = rng.uniform(-1, 1, pb.ndof)
    b[con] = 0
    x_direct = np.linalg.solve(A, b)
    pb.factor()  # single interior patch = whole free space
    assert pb.npatches == 1
    x_fdm = pb.smooth(b)
    assert np.linalg.norm(x_fdm - x_direct) / np.linalg.norm(x_direct) < 1e-10


def test_patch_stencils(oracle):  # test_assembly.cpp:149-175
    pb = oracle.Problem(1, 2, 4)
    assert pb.npatches == 1 and pb.patches_n(0) == 7 * 7  # (2p-1)^2
    ptr, col, val = pb.patch_matrix(0)
    pt = pb.patches()
    lab = pb.maps()["label_cls"][pt["dofs"]]
    for k in range(len(lab)):
        if lab[k] == 0:
            assert ptr[k + 1] - ptr[k] == 3  # d+1 nonzeros on interior rows


# ---- tests/test_schwarz.cpp -----------------------------------------------------
def test_asm_dense_per_patch_oracle(oracle):  # test_schwarz.cpp:24-51
    pb = oracle.Problem(1, 2, 3, build_global=True)
    pb.factor()
    rng = np.random.default_rng(5)
    r = rng.uniform(-1, 1, pb.ndof)
    r[pb.maps()["constrained"].astype(bool)] = 0
    z = pb.patch_apply(r)
    pt = pb.patches()
    z_or = np.zeros(pb.ndof)
    for j in range(pb.npatches):
        dofs = pt["dofs"][pt["ptr"][j]:pt["ptr"][j + 1]]
        ptr, col, val = pb.patch_matrix(j)
        n = len(dofs)
        Aj = np.zeros((n, n))
        for i in range(n):
            Aj[i, col[ptr[i]:ptr[i + 1]]] = val[ptr[i]:ptr[i + 1]]
        z_or[dofs] += np.linalg.solve(Aj, r[dofs])
    assert np.abs(z - z_or).max() < 1e-11
    assert np.linalg.norm(pb.patch_apply(np.zeros(pb.ndof))) == 0.0


def test_single_patch_exact(oracle):  # test_schwarz.cpp:53-72
    pb = oracle.Problem(1, 2, 3)
    pb.factor()
    b = pb.rhs()
    _, rep = pb.pcg(b, rtol=1e-10, maxit=20, precond=1)
    assert rep["converged"] and rep["iterations"] == 1


def test_estimate_damping_known_spectra(oracle):  # test_schwarz.cpp:74-91
    A = 3.0 * np.eye(12)
    assert abs(oracle.estimate_damping_dense(A, np.eye(12) / 3.0)["omega"] - 1.0) < 1e-8
    d = np.ones(20)
    d[19] = 10
    est = oracle.estimate_damping_dense(np.diag(d), np.eye(20))
    assert abs(est["lambda_max"] - 10) < 1e-5 and abs(est["omega"] - 2 / 11) < 2e-6


def test_two_level_p_robust(oracle):  # test_schwarz.cpp:93-129 (2D 4x4, f = 1)
    its = []
    for p in (3, 5, 7):
        pb = oracle.Problem(1, 4, p)  # 4x4 unit square
        pb.factor()
        pb.build_twolevel()
        rng = np.random.default_rng(1)
        con = pb.maps()["constrained"].astype(bool)
        x, y = rng.uniform(-1, 1, pb.ndof), rng.uniform(-1, 1, pb.ndof)
        x[con] = y[con] = 0
        assert abs(x @ pb.vcycle(y) - y @ pb.vcycle(x)) < 1e-10 * abs(x @ pb.vcycle(y))
        f = pb.load_vector_one()
        u, rep = pb.pcg(f, rtol=1e-8, maxit=100)
        assert rep["converged"] and rep["kappa"] <= 1.7 and rep["iterations"] <= 11
        assert np.linalg.norm(pb.apply_A(u) - f) / np.linalg.norm(f) <= 1e-8 * 1.0001
        its.append(rep["iterations"])
    assert max(its) - min(its) <= 2


# ---- tests/test_krylov.cpp ------------------------------------------------------
def lap1d(n):
    return 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)


def test_pcg_known_answers(oracle):  # test_krylov.cpp:32-76
    b = np.arange(1.0, 9.0)
    x, rep = oracle.pcg_dense(np.eye(8), b, 1e-10, 10)
    assert rep["converged"] and rep["iterations"] == 1 and abs(rep["kappa"] - 1) < 1e-10
    T = lap1d(50)
    ev = np.linalg.eigvalsh(T)
    x, rep = oracle.pcg_dense(T, np.ones(50), 1e-10, 500)
    assert rep["converged"] and abs(rep["kappa"] - ev[-1] / ev[0]) / (ev[-1] / ev[0]) < 0.05
    T80 = lap1d(80)
    x, rep = oracle.pcg_dense(T80, np.ones(80), 1e-8, 2000)
    assert rep["iterations"] <= math.ceil(0.5 * math.sqrt(rep["kappa"]) * math.log(2 / 1e-8)) + 2
    x, rep = oracle.pcg_dense(lap1d(60), np.ones(60), 1e-12, 3)
    assert not rep["converged"] and rep["iterations"] == 3
    with pytest.raises(oracle.OracleError, match="indefinite"):
        oracle.pcg_dense(np.diag([1.0, -1.0]), np.array([0.0, 1.0]), 1e-8, 10)


# ---- structure of the patch factors -------------------------
@pytest.mark.parametrize("cfg,n,p,nj,nnz,madds", [
    (1, 0, 0, 169, 706, 2118),          # 2D p = 7
    (2, 0, 0, 2197, 78109, 6991136),    # 3D p = 7
])
def test_patch_factor_structure(oracle, cfg, n, p, nj, nnz, madds):
    pb = oracle.Problem(cfg, n, p, build_global=False)
    pb.factor([0])
    info = pb.factor_info(0)
    assert (info["n"], info["nnz"], info["flops"]) == (nj, nnz, madds)
    assert list(pb.group_offsets(0))[0] == 0


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6])
def test_sumfact_apply_pinned_to_dense_quadrature(oracle, p):
    """[ext] pin of the oracle's sum-factorised trilinear apply (used for C5,
    where the dense 8.6 GB/cell matrix is infeasible) against its restatement
    of the reference's dense cell_matrix_quadrature (src/assembly.cpp:198-228)
    on perturbed hexes, in the style of tests/test_assembly.cpp:54-95."""
    pb = oracle.Problem(5, 3, p, build_global=False)  # 3^3 cells, 8 perturbed interior vertices
    rng = np.random.default_rng(p)
    for cell in range(pb.ncells):
        A = pb.cell_matrix_quadrature(cell)
        u = rng.uniform(-1, 1, pb.npc)
        y = pb.cell_sumfact_apply(cell, u)
        assert np.linalg.norm(y - A @ u) <= 1e-12 * np.linalg.norm(A @ u), (cell, p)
