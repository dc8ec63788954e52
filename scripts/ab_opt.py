"""A/B of a plan option on config-5 factor time: python scripts/ab_opt.py OPT v1 v2 ...
(median of 5 factors after 2 warm-ups, same plan and bands; alternating)."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P                      # noqa: E402
from paper_1604_00617_b200.solver import AcrSolver                   # noqa: E402
from paper_1604_00617_b200.system import Tolerance                   # noqa: E402

opt = int(sys.argv[1])
vals = [int(v) for v in sys.argv[2:]]
name = "cfg5"
c = P.CONFIGS[name]
s = P.make_config(name, nrhs=1)
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
times = {v: [] for v in vals}
for v in vals:
    sol.lib.acr_plan_set_option(sol.plan, opt, v)
    sol.factor(bands)
    sol.factor(bands)
for rep in range(5):
    for v in vals:
        sol.lib.acr_plan_set_option(sol.plan, opt, v)
        sol.factor(bands)
        torch.cuda.synchronize()
        times[v].append(sol.factor_ms)
for v in vals:
    print(f"option {opt} = {v}: median {statistics.median(times[v]):.2f} ms  {['%.1f' % t for t in times[v]]}")
