"""Times the elasticity operators (apply_A, smooth) on the GPU: python tools/elastic_op_time.py DIM N P [LAMBDA]."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2107_14758_b200 as F

dim, n, p = (int(v) for v in sys.argv[1:4])
lam = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
prob = F.Problem.elasticity(dim, n, p, 1.0, lam)
sol = F.Solver(prob)
sol.factor()
r = torch.from_numpy(prob.rhs()).cuda()
z = torch.empty_like(r)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


ta = t(lambda: sol.apply_A(r, z))
sol.kernel_timing(True)
for _ in range(20):
    sol.apply_A(r, z)
torch.cuda.synchronize()
km, kn = sol.kernel_time("stiffness")
sol.kernel_timing(False)
d, n1 = dim, p + 1
flops = 2.0 * n1 ** (d + 1) * d * (d * d + 2 * d * (d - 1)) * prob.ncells
print(f"apply_A {ta * 1e3:.1f} us, kernel {km / kn * 1e3:.1f} us = {flops / (km / kn * 1e-3) / 1e12:.2f} TFLOP/s "
      f"(kron_apply count), smooth {t(lambda: sol.smooth(r, z)) * 1e3:.1f} us")
