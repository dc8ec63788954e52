"""GPU idle time inside one config-5 factor: kernel intervals from the
torch profiler (CUPTI activity records), their union against the span from
the first kernel start to the last kernel end, and the idle gaps by size."""
import sys, json
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
for _ in range(3):
    sol.factor(bands)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sol.factor(bands)
    torch.cuda.synchronize()
print("factor_ms", sol.factor_ms)
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
print("events", len(iv))
t0, t1 = iv[0][0], max(e for _, e, _ in iv)
busy, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
gaps, where = [], []
prev = iv[0][2]
for a, b, nm in iv[1:]:
    if a > cur_e:
        busy += cur_e - cur_s
        gaps.append(a - cur_e)
        where.append((prev[:40], nm[:40], round((a - t0) / 1e3, 2)))
        cur_s, cur_e = a, b
    else:
        cur_e = max(cur_e, b)
    if b >= cur_e:
        prev = nm
busy += cur_e - cur_s
span = t1 - t0
print(f"span_ms {span/1e3:.2f} busy_ms {busy/1e3:.2f} idle_ms {(span-busy)/1e3:.2f}")
import numpy as np
g = np.array(gaps)
for lo, hi in ((0, 2), (2, 5), (5, 10), (10, 50), (50, 1e9)):
    m = (g >= lo) & (g < hi)
    print(f"gaps [{lo},{hi}) us: n={m.sum()} total_ms={g[m].sum()/1e3:.2f}")
big = sorted(((gaps[i], i) for i in range(len(gaps))), reverse=True)[:10]
for x, i in big:
    print(f"gap {x:8.1f} us at {where[i][2]} ms: after {where[i][0]} before {where[i][1]}")
# kernel time by name (concurrent kernels both count)
from collections import defaultdict
tot, cnt = defaultdict(float), defaultdict(int)
for a, b, nm in iv:
    k = nm.split("(")[0][:48]
    tot[k] += b - a
    cnt[k] += 1
print("kernel totals:")
for k in sorted(tot, key=lambda x: -tot[x])[:24]:
    print(f"  {k:48s} n={cnt[k]:5d} ms={tot[k]/1e3:8.2f} avg_us={tot[k]/cnt[k]:8.1f}")
