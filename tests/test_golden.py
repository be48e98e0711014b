"""The oracle reproduces the committed golden fixtures (tests/golden/, made by
tools/make_golden.py); the product host setup reproduces their map hashes."""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.json")))
SMALL = [g for g in GOLDEN if json.load(open(g))["ndof"] < 100000]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:24]


def load(path):
    return json.load(open(path))


def close(a, b, tol):
    return abs(a - b) <= tol * max(abs(b), 1e-300)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(g) for g in GOLDEN])
def test_product_map_hashes(pkg, path):
    g = load(path)
    pb = pkg.Problem(g["config"], g["n"], g["p"])
    m, pt = pb.maps(), pb.patches()
    assert (pb.ndof, pb.nfree, pb.npatches, pb.sum_nj) == (g["ndof"], g["nfree"], g["npatches"], g["sum_nj"])
    h = g["hash"]
    assert sha(m["cell_dofs"]) == h["cell_dofs"] and sha(m["constrained"]) == h["constrained"]
    assert sha(np.stack([m["label_cls"], m["label_entity"]])) == h["labels"]
    assert sha(pt["dofs"]) == h["patch_dofs"] and sha(pt["perm"]) == h["patch_perm"]
    assert sha(pb.rhs()) == h["rhs"]


@pytest.mark.parametrize("path", SMALL, ids=[os.path.basename(g) for g in SMALL])
def test_oracle_reproduces_golden(oracle, path):
    g = load(path)
    pb = oracle.Problem(g["config"], g["n"], g["p"], build_global=False, threads=4)
    r = pb.rhs()
    probe = np.random.default_rng(12345).standard_normal(pb.ndof)
    pb.factor()
    fi = pb.factor_info(0)
    assert (fi["n"], fi["nnz"], fi["flops"]) == (g["patch0"]["n"], g["patch0"]["nnz_L"], g["patch0"]["flops"])
    for name, v in (("apply_St", pb.apply_St(r)), ("apply_A", pb.apply_A(r)), ("smooth", pb.smooth(r))):
        assert close(float(np.linalg.norm(v)), g[name]["norm"], 1e-12), name
        assert close(float(v @ probe), g[name]["probe_dot"], 1e-10), name
    pb.build_twolevel()
    tl = pb.twolevel_info()
    assert close(tl["omega"], g["damping"]["omega"], 1e-10)
    _, rep = pb.pcg(r)
    assert rep["iterations"] == g["pcg"]["iterations"]


def test_elastic_table2_golden(oracle):
    import json
    import os

    import numpy as np

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "variants", "elastic_table2.json")))
    for lam, its, om in zip(g["lambdas"], g["iterations"], g["omega"]):
        e = oracle.ElasticProblem(2, 8, 3, 1.0, lam)
        e.build()
        _, rep = e.pcg(e.rhs(), 1e-8, 600)
        assert rep["iterations"] == its
        assert abs(e.twolevel_info()["omega"] - om) <= 1e-10 * om
    assert abs(np.linalg.norm(e.rhs()) - g["rhs_norm"]) <= 1e-14 * g["rhs_norm"]


def test_dg_two_level_golden(oracle):
    import json
    import os

    import numpy as np

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "variants", "dg_two_level.json")))
    d = oracle.DGProblem(2, 4, 4)
    d.build()
    x, rep = d.pcg(d.rhs(), 1e-8, 200)
    assert rep["iterations"] == g["iterations"] and rep["npatches"] == g["npatches"]
    assert abs(rep["omega"] - g["omega"]) <= 1e-10 * g["omega"]
    assert abs(np.linalg.norm(x) - g["x_norm"]) <= 1e-9 * g["x_norm"]
