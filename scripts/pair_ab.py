"""A/B: force the CTA-pair recompression path for direct launches (option 3)."""
import sys, torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver
from paper_1604_00617_b200.system import Tolerance
c = P.CONFIGS["cfg5"]
s = P.make_config("cfg5", nrhs=1)
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
for force in (0, 1, 0, 1):
    sol.lib.acr_plan_set_option(sol.plan, 3, force)
    ts = []
    for _ in range(3):
        sol.factor(bands)
        ts.append(sol.factor_ms)
    print("force_pair", force, [round(t, 1) for t in ts], flush=True)
