"""Quick timing of factor/solve per config on the GPU (development aid)."""
import sys, time, json
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1604_00617_b200 import problems as P
from paper_1604_00617_b200.solver import AcrSolver, relative_residual_gpu
from paper_1604_00617_b200.system import Tolerance

cfgs = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"]
for name in cfgs:
    c = P.CONFIGS[name]
    t0 = time.time()
    s = P.make_config(name)
    tg = time.time() - t0
    sol = AcrSolver(s.n_blocks, s.block_dim, Tolerance(c["eps"]), 1, c["leaf"])
    bands = sol.device_bands(s)
    f = torch.as_tensor(s.rhs, device="cuda")
    times = []
    for it in range(int(__import__("os").environ.get("REPS", "3"))):
        sol.factor(bands)
        times.append(sol.factor_ms)
    u = sol.solve(f)
    first_solve = sol.solve_ms
    u = sol.solve(f)
    res = relative_residual_gpu(bands, u, f, s.n_blocks, s.block_dim)
    prof = sol.rank_profiles()
    print(json.dumps(dict(cfg=name, gen_s=round(tg, 2), factor_ms=[round(x, 2) for x in times],
                          solve_ms=round(sol.solve_ms, 2), first_solve_ms=round(first_solve, 2), residual=res,
                          max_rank=max(p.max_rank for p in prof), launches=sol.kernel_launches,
                          storage=sol.storage_bytes(s.n_rhs),
                          unknowns_per_s=s.n_unknowns / (min(times) / 1e3))), flush=True)
    if __import__("os").environ.get("PROF"):
        import ctypes as C
        sol.lib.acr_plan_set_option(sol.plan, 2, 1)
        sol.factor(bands)
        sol.lib.acr_plan_set_option(sol.plan, 2, 0)
        st = {}
        for cls, nm in enumerate(["trunc", "leafinv", "leafgemm", "hmat", "leafgemm_diag"]):
            nl = C.c_longlong(); ms = C.c_double(); ctr = (C.c_ulonglong * 16)()
            sol.lib.acr_kernel_stats(sol.plan, cls, C.byref(nl), C.byref(ms), ctr)
            st[nm] = (nl.value, round(ms.value, 1))
            if cls == 0:
                st["trunc_ctr"] = list(ctr)
        print(json.dumps(dict(cfg=name, instrumented_factor_ms=round(sol.factor_ms, 1), classes=st)), flush=True)
        nl = C.c_longlong(); ms = C.c_double(); ctr = (C.c_ulonglong * 160)()
        sol.lib.acr_kernel_stats(sol.plan, 100, C.byref(nl), C.byref(ms), ctr)
        cnt = list(ctr)[16:41]; cyc = list(ctr)[41:66]
        tot = sum(cyc) or 1
        print("warp-path histogram (rows R<=4,8,16,32,>32; cols m<=32,64,128,256,>256): count / %cycles / kcyc-per-task")
        for rb in range(5):
            print("  ", " | ".join(f"{cnt[rb*5+mb]:8d} {100*cyc[rb*5+mb]/tot:5.1f}% {cyc[rb*5+mb]/max(cnt[rb*5+mb],1)/1e3:6.1f}" for mb in range(5)))
        print("warp phases G (load, qr, core, jacobi, select, output):", [round(ctr[i] / 1e9, 2) for i in (12, 13, 14, 15, 66, 67)])
        print("block phases G (load, qr, core, jacobi, select, output):", [round(ctr[i] / 1e9, 2) for i in range(2, 8)])
        bc = list(ctr)[72:97]; by = list(ctr)[97:122]; bj = list(ctr)[122:147]
        print("block-path histogram (R<=8,16,32,64,>64; m<=128,256,512,1024,>1024): count / kcyc-per-task / jacobi%")
        for rb in range(5):
            print("  ", " | ".join(f"{bc[rb*5+mb]:7d} {by[rb*5+mb]/max(bc[rb*5+mb],1)/1e3:7.1f} {100*bj[rb*5+mb]/max(by[rb*5+mb],1):4.0f}%" for mb in range(5)))
