"""Factor cfg5 once, then one 16-RHS solve inside a profiler range."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver
from paper_1604_00617_b200.system import Tolerance
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
c = P.CONFIGS[name]
s = P.make_config(name)
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
f = torch.as_tensor(s.rhs, device="cuda")
sol.factor(bands)
sol.solve(f)
torch.cuda.synchronize()
torch.cuda.profiler.start()
u = sol.solve(f)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("solve_ms", sol.solve_ms)
