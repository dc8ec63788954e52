"""A/B: direct (one CTA per task) vs warp-kernel recompression by launch size (option 5)."""
import sys, torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver
from paper_1604_00617_b200.system import Tolerance
c = P.CONFIGS["cfg5"]
s = P.make_config("cfg5", nrhs=1)
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
sol.factor(bands)
opt = int(sys.argv[1]) if len(sys.argv) > 1 else 5
vals = [int(x) for x in sys.argv[2:]] or [-1, 0, 8, 32, 64, -1]
for v in vals:
    sol.lib.acr_plan_set_option(sol.plan, opt, v)
    ts = []
    for _ in range(3):
        sol.factor(bands)
        ts.append(sol.factor_ms)
    print("option", opt, v, [round(t, 1) for t in ts], flush=True)
