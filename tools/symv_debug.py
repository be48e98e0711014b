"""Scratch: inverse-top vs Cholesky-top patch solve on one configuration, per chunk count."""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_2107_14758_b200 as F

cfg = tuple(int(v) for v in sys.argv[1].split(","))
prob = F.Problem(*cfg)
r = prob.rhs()


def run(top, chunks=None):
    os.environ["FDMGPU_TOP"] = top
    if chunks:
        os.environ["FDMGPU_SYMV_CHUNKS"] = str(chunks)
    else:
        os.environ.pop("FDMGPU_SYMV_CHUNKS", None)
    s = F.Solver(prob)
    s.factor()
    return s.patch_apply(r)


zc = run("chol")
for ch in (None, 1, 2, 3, 8):
    zi = run("inverse", ch)
    print("chunks", ch, "rel", np.linalg.norm(zi - zc) / np.linalg.norm(zc))
