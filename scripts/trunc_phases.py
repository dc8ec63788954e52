"""Recompression phase breakdown of one instrumented config-5 factor (plan
option 2): clock64 cycles summed over tasks per phase, block and warp path,
and the block-path histogram by (R, rows) bucket."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P                      # noqa: E402
from paper_1604_00617_b200.solver import AcrSolver                   # noqa: E402
from paper_1604_00617_b200.system import Tolerance                   # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
c = P.CONFIGS[name]
s = P.make_config(name, nrhs=1)
sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
bands = sol.device_bands(s)
sol.factor(bands)
sol.lib.acr_plan_set_option(sol.plan, 2, 1)
sol.factor(bands)
torch.cuda.synchronize()
nl, ms = C.c_longlong(), C.c_double()
ctr = (C.c_ulonglong * 256)()
sol.lib.acr_kernel_stats(sol.plan, 100, C.byref(nl), C.byref(ms), ctr)
G = 1e9
print(f"block path: tasks {ctr[8]}, sweeps {ctr[10]}; Gcyc load {ctr[2]/G:.2f} qr {ctr[3]/G:.2f} "
      f"core {ctr[4]/G:.2f} jacobi {ctr[5]/G:.2f} select {ctr[6]/G:.2f} output {ctr[7]/G:.2f}")
print(f"warp path: tasks {ctr[9]}, sweeps {ctr[11]}; Gcyc load {ctr[12]/G:.2f} qr {ctr[13]/G:.2f} "
      f"core {ctr[14]/G:.2f} jacobi {ctr[15]/G:.2f} select {ctr[66]/G:.2f} output {ctr[67]/G:.2f} "
      f"slot-wait {ctr[68]/G:.2f}")
rl = ["R<=8", "R<=16", "R<=32", "R<=64", "R>64"]
ml = ["m<=128", "m<=256", "m<=512", "m<=1024", "m>1024"]
print("block-path histogram: count / Gcyc total / Gcyc jacobi")
for rb in range(5):
    row = []
    for mb in range(5):
        k = rb * 5 + mb
        if ctr[72 + k]:
            row.append(f"{ml[mb]}: {ctr[72+k]} / {ctr[97+k]/G:.2f} / {ctr[122+k]/G:.2f}")
    if row:
        print(f"  {rl[rb]}: " + "; ".join(row))
print("warp-path histogram [16..65]:", list(ctr[16:66]))
print(f"direct launches: tasks {ctr[160]}; Gcyc load {ctr[161]/G:.2f} qr {ctr[162]/G:.2f} core "
      f"{ctr[163]/G:.2f} jacobi {ctr[164]/G:.2f} select {ctr[165]/G:.2f} output {ctr[166]/G:.2f}")
print("direct histogram: count / Gcyc total / Gcyc QR")
for rb in range(5):
    row = []
    for mb in range(5):
        k = rb * 5 + mb
        if ctr[170 + k]:
            row.append(f"{ml[mb]}: {ctr[170+k]} / {ctr[195+k]/G:.3f} / {ctr[220+k]/G:.3f}")
    if row:
        print(f"  {rl[rb]}: " + "; ".join(row))
for cls, nm in enumerate(["trunc", "leafinv", "leafgemm", "hmat", "diag", "gp", "leaflr", "elem", "lu"]):
    c16 = (C.c_ulonglong * 16)()
    sol.lib.acr_kernel_stats(sol.plan, cls, C.byref(nl), C.byref(ms), c16)
    print(f"  {nm:8s} launches {nl.value:5d} ms {ms.value:8.2f}")
print("instrumented factor ms", sol.factor_ms)
