"""Small factor + solve cases for compute-sanitizer runs (warp, block and
pair recompression paths, leaf kernels, hmat, LU, generators)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver, acr_solve
from paper_1604_00617_b200.system import Tolerance

s = P.random_system(8, 16, seed=3)
u, rep = acr_solve(s, Tolerance(1e-10), leaf_size=4)
print("random8x16 residual", rep.residual)
s = P.poisson_const(32, seed=1)
u, rep = acr_solve(s, Tolerance(1e-8), leaf_size=8, cutoff_blocks=2)
print("poisson32 residual", rep.residual)
c = P.CONFIGS["cfg1"]
for force in (0, 1):
    d = P.device_config("cfg1")
    sol = AcrSolver(d.n_blocks, d.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
    sol.lib.acr_plan_set_option(sol.plan, 3, force)
    sol.factor(d.bands)
    x = sol.solve(torch.stack([d.rhs, d.rhs], 1).contiguous())
    torch.cuda.synchronize()
    print("cfg1 force_pair", force, float(x.abs().max()))
