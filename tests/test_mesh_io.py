"""External meshes in the reference's JSON format (load_mesh / save_mesh,
src/mesh.cpp:354-434): round trips, facet tags (Dirichlet /
Neumann) through the discretization maps against the oracle (bit-exact), and
the reference's error messages.  CPU only (host setup mirror + oracle)."""
import json
import os

import numpy as np
import pytest

import paper_2107_14758_b200 as F
from oracle import oracle as O


def _write(path, doc):
    with open(path, "w") as f:
        json.dump(doc, f)


def test_round_trip_is_exact(tmp_path):
    p = F.Problem(5, 2, 3)  # perturbed interior vertices (C5 generator)
    path = tmp_path / "m.json"
    p.save_mesh(str(path))
    doc = json.load(open(path))
    assert doc["dim"] == 3 and len(doc["cells"]) == p.ncells and len(doc["vertices"]) == p.nvertices
    assert all(t["tag"] == "dirichlet" for t in doc["facet_tags"]) and len(doc["facet_tags"]) == 6 * 4
    q = F.Problem.from_mesh_file(str(path), 3)
    a, b = p.maps(), q.maps()
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    ga, gb = p.geometry(), q.geometry()
    assert np.array_equal(ga["vertices"], gb["vertices"]) and np.array_equal(ga["mu"], gb["mu"])


@pytest.mark.parametrize("tagged", [("neumann", 0), ("neumann", 5), ("interior", 2)])
def test_facet_tags_match_oracle(tmp_path, tagged):
    kind, lf = tagged
    base = F.Problem(2, 3, 3)
    path = tmp_path / "m.json"
    base.save_mesh(str(path))
    doc = json.load(open(path))
    for t in doc["facet_tags"]:
        if t["local_facet"] == lf:
            t["tag"] = kind
    _write(path, doc)
    mine = F.Problem.from_mesh_file(str(path), 3, seed=7)
    tags = [(t["cell"], t["local_facet"], t["tag"]) for t in doc["facet_tags"]]
    ref = O.Problem.from_mesh(doc["dim"], doc["vertices"], doc["cells"], 3, facet_tags=tags, seed=7)
    assert (mine.ndof, mine.nfree) == (ref.ndof, ref.nfree)
    assert mine.nfree > base.nfree  # the relaxed face is free now
    a, r = mine.maps(), ref.maps()
    assert np.array_equal(a["cell_dofs"].ravel(), r["cell_dofs"].ravel())
    assert np.array_equal(a["constrained"], r["constrained"])
    assert np.array_equal(a["multiplicity"], r["multiplicity"])
    assert np.array_equal(mine.rhs(), ref.rhs())
    arr = F.Problem.from_mesh(doc["dim"], doc["vertices"], doc["cells"], 3, facet_tags=tags, seed=7)
    assert np.array_equal(arr.maps()["constrained"], a["constrained"])


def test_load_errors(tmp_path):
    with pytest.raises(F.FdmGpuError, match="load_mesh: cannot open"):
        F.Problem.from_mesh_file(str(tmp_path / "missing.json"), 2)
    base = F.Problem(2, 2, 2)
    path = tmp_path / "m.json"
    base.save_mesh(str(path))
    doc = json.load(open(path))
    bad = dict(doc, facet_tags=[{"cell": 0, "local_facet": 0, "tag": "robin"}])
    _write(path, bad)
    with pytest.raises(F.FdmGpuError, match="mesh file: unknown facet tag 'robin'"):
        F.Problem.from_mesh_file(str(path), 2)
    bad = dict(doc, facet_tags=[{"cell": 0, "local_facet": 6, "tag": "neumann"}])  # no such facet in 3D
    _write(path, bad)
    with pytest.raises(F.FdmGpuError, match="missing facet on cell 0"):
        F.Problem.from_mesh_file(str(path), 2)
    cells = [list(c) for c in doc["cells"]]
    cells[1][0], cells[1][1] = cells[1][1], cells[1][0]  # mirrored corner order
    _write(path, dict(doc, cells=cells, facet_tags=[]))
    with pytest.raises(F.FdmGpuError, match="non-positive Jacobian"):
        F.Problem.from_mesh_file(str(path), 2)
    with open(path, "w") as f:
        f.write('{"dim": 3, "vertices": [[0, 0, 0]')
    with pytest.raises(F.FdmGpuError, match="load_mesh: .*parse error"):
        F.Problem.from_mesh_file(str(path), 2)


@pytest.mark.parametrize("cfg", [(1, 4, 3), (5, 2, 3), (2, 1, 2)])
def test_boundary_star_lists_match_oracle(cfg):
    """skip_boundary_patches=False (SolverConfig's default, src/schwarz.cpp:71-81):
    the host adds the same boundary-vertex stars as the oracle."""
    mine = F.Problem(*cfg, skip_boundary_patches=False)
    ref = O.Problem(*cfg, build_global=False, skip_boundary_patches=False)
    base = F.Problem(*cfg)
    assert (mine.npatches, mine.sum_nj) == (ref.npatches, ref.sum_nj)
    assert mine.npatches == (cfg[1] + 1) ** mine.dim and base.npatches == (max(cfg[1] - 1, 0) ** mine.dim or mine.npatches)
