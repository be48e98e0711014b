"""Development: build config (default C3) and run the batched factorisation twice."""
import sys
sys.path.insert(0, "/root/repo")
import paper_2107_14758_b200 as F
cfg = tuple(int(v) for v in sys.argv[1].split(",")) if len(sys.argv) > 1 else (3, 0, 0)
sol = F.Solver(F.Problem(*cfg))
sol.factor(); sol.factor(); sol.synchronize()
print("ok", sol.layout())
