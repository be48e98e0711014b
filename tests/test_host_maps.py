"""Bit-exact index maps: the product's host setup (paper_2107_14758_b200/csrc/host,
the mirror of src/mesh.cpp, src/discretization.cpp, src/ordering.cpp,
src/schwarz.cpp:62-83) against the oracle, plus the colouring contract
(SURVEY.md §7.4).  CPU only: no compute calls on the device."""
import numpy as np
import pytest

CASES = [(1, 0, 0), (2, 0, 0), (1, 4, 5), (2, 3, 4), (3, 3, 3), (4, 4, 5), (5, 3, 4), (4, 0, 3), (5, 0, 3)]


@pytest.mark.parametrize("cfg", CASES)
def test_maps_bit_exact(pkg, oracle, cfg):
    a, b = pkg.Problem(*cfg), oracle.Problem(*cfg, build_global=False)
    assert (a.ndof, a.nfree, a.ncells, a.npatches, a.sum_nj) == (b.ndof, b.nfree, b.ncells, b.npatches, b.sum_nj)
    ma, mb = a.maps(), b.maps()
    for k in ("cell_dofs", "cell_modes", "constrained", "multiplicity", "label_cls", "label_entity"):
        assert np.array_equal(ma[k], mb[k]), k
    pa, pb_ = a.patches(), b.patches()
    for k in ("vertex", "ptr", "dofs", "perm"):
        assert np.array_equal(pa[k], pb_[k]), k
    assert np.array_equal(a.rhs(), b.rhs())
    ga, gb = a.geometry(), b.geometry()
    assert np.array_equal(ga["vertices"], gb["vertices"]) and np.array_equal(ga["kappa"], gb["kappa"])
    assert np.abs(ga["mu"] - gb["mu"]).max() <= 1e-15 * np.abs(gb["mu"]).max()
    ba, bb = a.basis(), b.basis()
    assert np.abs(ba["S"] - bb["S"]).max() < 1e-14
    assert np.array_equal(ba["Atnz"], bb["Atnz"]) and np.array_equal(ba["Btnz"], bb["Btnz"])


@pytest.mark.parametrize("cfg", [(1, 0, 0), (2, 0, 0), (3, 3, 3)])
def test_colouring(pkg, cfg):
    a = pkg.Problem(*cfg)
    pt = a.patches()
    col, cells = pt["colour"], pt["cells"]
    assert col.max() + 1 == 2 ** a.dim  # vertex-parity colouring on lattice meshes
    for c in range(col.max() + 1):
        members = cells[col == c].ravel()
        assert len(np.unique(members)) == len(members)  # same-colour stars share no cell
    # parity form: colour(v) determined by (i mod 2, j mod 2, k mod 2) up to relabelling
    n1 = a.n + 1
    v = pt["vertex"]
    par = (v % n1) % 2 + 2 * ((v // n1) % n1 % 2) + 4 * ((v // (n1 * n1)) % 2 if a.dim == 3 else 0)
    mapping = {}
    for pv, cv in zip(par, col):
        assert mapping.setdefault(int(pv), int(cv)) == int(cv)
    assert np.array_equal(col, pkg.Problem(*cfg).patches()["colour"])  # deterministic


def test_coarse_prolongation_matches_oracle(pkg, oracle):
    a = pkg.Problem(2, 3, 3)
    b = oracle.Problem(2, 3, 3, build_global=False)
    b.factor()
    b.build_twolevel(calibrate=False)
    ca = a.coarse()
    ptr, col, val = b.prolongation()
    assert np.array_equal(ca["P_ptr"], ptr) and np.array_equal(ca["P_col"], col)
    assert np.abs(ca["P_val"] - val).max() < 1e-15
