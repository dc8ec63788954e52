"""Kernel timeline of the last reduction level of one config-5 factor (torch profiler)."""
import sys, json, collections
import torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver
from paper_1604_00617_b200.system import Tolerance
c = P.CONFIGS["cfg5"]
s = P.make_config("cfg5", nrhs=1)
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
for _ in range(3):
    sol.factor(bands)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    sol.factor(bands)
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/factor_trace.json")
tr = json.load(open("gpurun_out/factor_trace.json"))
ev = [e for e in tr["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]; t1 = max(e["ts"] + e["dur"] for e in ev)
print("span ms", (t1 - t0) / 1e3, "kernels", len(ev))
lo = t1 - 13500.0   # last level + LU
sel = [e for e in ev if e["ts"] >= lo]
by = collections.defaultdict(lambda: [0, 0.0])
for e in sel:
    k = e["name"].split("(")[0][:40]
    by[k][0] += 1; by[k][1] += e["dur"]
for k, v in sorted(by.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:42s} n={v[0]:4d} us={v[1]:9.1f}")
with open("gpurun_out/tail_events.txt", "w") as f:
    for e in sel:
        f.write(f"{e['ts']-lo:10.1f} {e['dur']:8.1f} s{e['args'].get('stream')} {e['name'].split('(')[0][:50]} grid={e['args'].get('grid')} block={e['args'].get('block')}\n")
