"""Development aid: per-task trace of the direct (latency-bound) recompressions of one instrumented factor."""
import sys, os
import torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver
from paper_1604_00617_b200.system import Tolerance
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
c = P.CONFIGS[name]
s = P.make_config(name, nrhs=1)
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
sol.factor(bands)
sol.lib.acr_plan_set_option(sol.plan, 2, 1)
sol.factor(bands)
torch.cuda.synchronize()
