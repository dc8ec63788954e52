"""Run one factor of a config (for ncu launch lists / profiles)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver
from paper_1604_00617_b200.system import Tolerance
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
c = P.CONFIGS[name]
s = P.make_config(name, nrhs=1)
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
for _ in range(reps):
    sol.factor(bands)
torch.cuda.synchronize()
print(name, "factor_ms", sol.factor_ms, "launches", sol.kernel_launches)
