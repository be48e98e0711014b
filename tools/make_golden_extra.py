"""Generates tests/golden/variants/elastic_table2.json and
tests/golden/variants/dg_two_level.json from the oracle.  These are oracle
regression snapshots (they freeze the oracle's elasticity / SIPG results; the
reference tests pin those only to +-20 % / upper bounds), not reference output."""
import json
import os
import sys

import numpy as np

ROOT = __file__.rsplit("/tools/", 1)[0]
sys.path.insert(0, ROOT)
from oracle import oracle as O

out = {"problem": "tests/test_elasticity.cpp:157-185 Table-2: 2D 8x8, vector Q3, mu 1", "lambdas": [], "iterations": [],
       "omega": [], "rhs_norm": None}
for lam in (0.0, 1.0, 10.0, 100.0, 1000.0):
    e = O.ElasticProblem(2, 8, 3, 1.0, lam)
    e.build()
    x, rep = e.pcg(e.rhs(), 1e-8, 600)
    out["lambdas"].append(lam)
    out["iterations"].append(rep["iterations"])
    out["omega"].append(e.twolevel_info()["omega"])
    out["rhs_norm"] = float(np.linalg.norm(e.rhs()))
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "variants", "elastic_table2.json"), "w"), indent=1)
g = O.DGProblem(2, 4, 4)
g.build()
x, rep = g.pcg(g.rhs(), 1e-8, 200)
json.dump({"problem": "tests/test_sipg.cpp:169-206 Cartesian: 2D 4x4, DG Q4, eta (p+1)(p+d)", "iterations": rep["iterations"],
           "omega": rep["omega"], "npatches": rep["npatches"], "x_norm": float(np.linalg.norm(x))},
          open(os.path.join(ROOT, "tests", "golden", "variants", "dg_two_level.json"), "w"), indent=1)
print("ok")
