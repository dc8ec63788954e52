"""Cost of the fused forward sweep: factor() vs factor(rhs) vs factor()+solve(rhs)
on config 5 (device-resident inputs, CUDA events)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver
from paper_1604_00617_b200.system import Tolerance
c = P.CONFIGS["cfg5"]
s = P.make_config("cfg5")
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
f = torch.as_tensor(s.rhs, device="cuda")
def t(fn, reps=4):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
print("factor            %.2f ms" % t(lambda: sol.factor(bands)))
print("factor(rhs)       %.2f ms" % t(lambda: sol.factor(bands, rhs=f)))
def fs():
    sol.factor(bands, rhs=f); sol.solve()
print("factor(rhs)+back  %.2f ms" % t(fs))
def f2():
    sol.factor(bands); sol.solve(f)
print("factor+solve      %.2f ms" % t(f2))
