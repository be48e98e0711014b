"""MatrixMarket export (write_matrix_market, src/sparse.cpp:33-52; SURVEY.md
§8(f)4): the reference's exact text format, symmetric lower-triangle
filtering, column-major entry order, and a scipy round trip.  CPU only."""
import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

import paper_2107_14758_b200 as F


def test_format_matches_reference_writer(tmp_path):
    A = np.array([[4.0, 0.0, 1.0 / 3.0], [0.0, 2.5, 0.0], [1.0 / 3.0, 0.0, 1e-300]])
    path = tmp_path / "a.mtx"
    F.write_matrix_market(str(path), A, symmetric=True)
    lines = open(path).read().splitlines()
    # header, dims + lower-triangle count, then (row, col) 1-based in column-major order
    assert lines[0] == "%%MatrixMarket matrix coordinate real symmetric"
    assert lines[1] == "3 3 4"
    assert lines[2:] == ["1 1 4", "3 1 0.33333333333333331", "2 2 2.5", "3 3 1e-300"]
    F.write_matrix_market(str(path), A, symmetric=False)
    lines = open(path).read().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general" and lines[1] == "3 3 5"
    assert lines[2:4] == ["1 1 4", "3 1 " + format(1.0 / 3.0, ".17g")] and lines[4].startswith("2 2 ")


@pytest.mark.filterwarnings("ignore::DeprecationWarning")
def test_scipy_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    M = sp.random(40, 30, density=0.2, random_state=1, format="csr") * 7.0
    path = tmp_path / "m.mtx"
    F.write_matrix_market(str(path), M)
    R = scipy.io.mmread(str(path))
    assert (abs(R - M)).max() == 0.0  # 17 significant digits: exact
    S = M[:30, :30] + M[:30, :30].T
    F.write_matrix_market(str(path), S, symmetric=True)
    assert (abs(scipy.io.mmread(str(path)) - S)).max() == 0.0
    E = sp.csc_matrix((5, 4))
    F.write_matrix_market(str(path), E)
    assert open(path).read().splitlines()[1] == "5 4 0"


def test_cannot_open(tmp_path):
    with pytest.raises(F.FdmGpuError, match="cannot open"):
        F.write_matrix_market(str(tmp_path / "no" / "such" / "dir.mtx"), np.eye(2))
