"""Development: print the separator factor fill statistics (FDMGPU_DEBUG=1) for a config."""
import sys
sys.path.insert(0, "/root/repo")
import paper_2107_14758_b200 as F
for a in sys.argv[1:]:
    cfg = tuple(int(v) for v in a.split(","))
    sol = F.Solver(F.Problem(*cfg))
    L = sol.layout()
    print(cfg, "tiles", L["tiles"], "nnz_L", L["nnz_L"], "factor GB", L["factor_bytes"] / 1e9, "tile_gemms", L["tile_gemms"], flush=True)
