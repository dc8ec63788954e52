"""Small var-coef case whose m>32 recompressions take the warp path (racecheck / debug aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import acr_solve
from paper_1604_00617_b200.system import Tolerance
from oracle import acr_oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 16
s = P.varcoef_diffusion(n, seed=0)
tol = Tolerance(1e-6)
u, rep = acr_solve(s, tol, leaf_size=leaf)
print("gpu residual", rep.residual, [p.max_by_depth for p in rep.per_level_ranks])
if "--oracle" in sys.argv:
    uo, ro = O.acr_solve(s, tol, leaf_size=leaf)
    print("oracle residual", ro.residual, [p.max_by_depth for p in ro.per_level_ranks])
    print("rel diff", np.linalg.norm(u - uo) / np.linalg.norm(uo))
