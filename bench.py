"""Benchmark: ACR factor unknowns/s (fp64, 5-point 2D) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg5]

One step = one full factorisation (lift + every reduction level + cutoff
LU) of BASELINE.json config 5 (variable-coefficient diffusion 2048^2,
N = 4,194,304, leaf 64, eps 1e-6) with the bands resident in HBM.  The
bands (168 MB) and the HODLR working set (tens of GB) exceed the 126 MB L2,
so no explicit flush is needed between steps.  ``e2e`` is the same metric
through the public API with pinned host buffers: H2D of the bands and the
16-column RHS, factor, solve, D2H of u.

``--impl reference`` times the CPU restatement of the reference
(oracle/acr_oracle.py, the reference's own algorithm and LAPACK calls) on a
bounded sample of the same workload: the first 64 block rows of the config-5
system (same n, leaf, eps; 6 of the 11 levels), one BLAS thread (the
reference is single-threaded; all-core BLAS is reported beside it and is
slower on these block sizes), so every step stays within seconds.  The
reference package itself cannot travel to the GPU box; its own full-config
factor time measured in the build container is reported as context.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1604_00617_b200 import problems as P            # noqa: E402
from paper_1604_00617_b200.system import (BlockTridiagSystem,  # noqa: E402
                                          Tolerance)

METRIC = "ACR factor unknowns/s (fp64 5-pt 2D)"
UNIT = "unknowns/s"
SAMPLE_BLOCKS = 64          # 6 of config 5's 11 levels; ~5-10 s per step on one core


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx = [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        seen = set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    seen.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [],
                    "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx),
                "reasons": sorted(seen), "samples": len(sm)}


def sample_system(cfg: str, blocks: int = None) -> BlockTridiagSystem:
    """First ``blocks`` block rows of the config (same n, leaf, eps)."""
    s = P.make_config(cfg, nrhs=1)
    k = min(blocks or SAMPLE_BLOCKS, s.n_blocks)
    n = s.block_dim
    return BlockTridiagSystem(k, n, s.D_sub[:k], s.D_diag[:k], s.D_sup[:k],
                              s.E[:k - 1], s.F[:k - 1], s.rhs[:k * n],
                              name=f"{s.name}[:{k}]")


def cpu_reference_step(cfg: str, sub: BlockTridiagSystem, threads: int = 1):
    """One bounded sample of the reference algorithm on the host (oracle: the
    reference's algorithm with its LAPACK call sequence), BLAS limited to
    ``threads`` threads."""
    from threadpoolctl import threadpool_limits
    from oracle import acr_oracle as O
    c = P.CONFIGS[cfg]
    with threadpool_limits(threads):
        _, rep = O.acr_solve(sub, Tolerance(c["eps"]), leaf_size=c["leaf"])
    return sub.n_unknowns / (rep.reduce_ms / 1e3), rep


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_context(cfg: str) -> dict:
    """The real reference's own full-config factor time, measured in the
    build container on one core (tests/golden/<cfg>.npz reduce_ms, from
    make_golden.py running acrsolve.acr_solve unmodified)."""
    out = {}
    try:
        z = np.load(os.path.join(REPO, "tests", "golden", f"{cfg}.npz"))
        N = P.CONFIGS[cfg]["n"] ** 2
        ms = float(z["reduce_ms"])
        out = {"reference_full_config_reduce_ms": ms,
               "reference_full_config_unknowns_per_s": N / (ms / 1e3),
               "where": "build container, 1 core (8-core Intel Xeon), acrsolve unmodified"}
    except (OSError, KeyError):
        pass
    return out


def cpu_baseline_block(cfg: str, steps: int = 1):
    """1 BLAS thread (the reference is single-threaded) as the
    primary figure, plus one all-host-cores run; nproc and CPU model."""
    sub = sample_system(cfg)
    nproc = os.cpu_count() or 1
    vals, reds = [], []
    for _ in range(steps):
        v, rep = cpu_reference_step(cfg, sub, 1)
        vals.append(v)
        reds.append(rep.reduce_ms)
    v1 = sub.n_unknowns * steps / (sum(reds) / 1e3)
    va, rep_a = cpu_reference_step(cfg, sub, nproc)
    return sub, v1, {
        "value": v1, "unit": UNIT, "cores": 1, "kind": "port",
        "sample": (f"{cfg} first {sub.n_blocks} of {P.CONFIGS[cfg]['n']} block rows "
                   f"({sub.n_unknowns} unknowns, n={sub.block_dim}, "
                   f"{len(reds)} x reduce phase of oracle/acr_oracle.py = the reference's "
                   f"algorithm and LAPACK calls, {sum(reds) / 1e3:.1f} s)"),
        "all_cores": {"value": va, "cores": nproc, "reduce_ms": rep_a.reduce_ms},
        "nproc": nproc, "cpu_model": cpu_model(),
        "context": reference_context(cfg)}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    # warm-up: one config-1 solve per warm-up step
    w1 = P.make_config("cfg1")
    for _ in range(args.warmup):
        cpu_reference_step("cfg1", w1, 1)
    sub, value, cb = cpu_baseline_block(args.config, args.steps)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sub.n_unknowns / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator, BASELINE cfg5 formulas)",
        "impl": "reference",
        "config": {"workload": f"{args.config} bounded sample: {sub.n_blocks} of "
                   f"{P.CONFIGS[args.config]['n']} block rows",
                   "n": sub.block_dim, "leaf": P.CONFIGS[args.config]["leaf"],
                   "eps": P.CONFIGS[args.config]["eps"]},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if ws > torch.cuda.device_count():
        print(f"bench.py: {ws} ranks but {torch.cuda.device_count()} visible GPU(s)",
              file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1604_00617_b200.solver import AcrSolver, relative_residual_gpu

    cfg = args.config
    c = P.CONFIGS[cfg]
    sys_ = P.make_config(cfg)                      # nrhs from the config (16 for cfg5)
    m, n = sys_.n_blocks, sys_.block_dim
    N = sys_.n_unknowns
    k = sys_.n_rhs
    tol = Tolerance(c["eps"])
    if ws > 1:
        # sharded factor: contiguous block-row windows, NCCL neighbour halo,
        # top levels consolidated on rank 0 (paper_1604_00617_b200/dist.py)
        from paper_1604_00617_b200.dist import DistAcrSolver
        solver = DistAcrSolver(m, n, tol, 1, c["leaf"])
    else:
        solver = AcrSolver(m, n, tol, 1, c["leaf"])
    bands = [torch.as_tensor(np.ascontiguousarray(a), device="cuda") for a in
             (sys_.D_sub, sys_.D_diag, sys_.D_sup, sys_.E, sys_.F)]
    stream = torch.cuda.current_stream()

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        solver.factor(bands)
    launches_per_factor = solver.kernel_launches
    torch.cuda.synchronize()
    barrier()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            solver.factor(bands)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = N / (ms / 1e3)                          # one global system, all ranks

    # --- end to end through the public API with host buffers -------------
    host = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in
            (sys_.D_sub, sys_.D_diag, sys_.D_sup, sys_.E, sys_.F)]
    rhs_h = torch.from_numpy(np.ascontiguousarray(sys_.rhs)).pin_memory()
    u_h = torch.empty_like(rhs_h).pin_memory()
    dev = [torch.empty_like(h, device="cuda") for h in host]
    rhs_d = torch.empty_like(rhs_h, device="cuda")
    u_d = torch.zeros_like(rhs_d)
    h2d = sum(h.numel() * 8 for h in host) + rhs_h.numel() * 8
    d2h = u_h.numel() * 8
    e2e_steps = max(1, min(args.steps, 10))   # pipelined steady state: first upload / last download amortised

    copy_stream = torch.cuda.Stream()

    def e2e_step():
        for d, h in zip(dev, host):
            d.copy_(h, non_blocking=True)
        rhs_d.copy_(rhs_h, non_blocking=True)
        if ws == 1:          # forward sweep fused into the factorisation
            solver.factor(dev, rhs=rhs_d)
            uu = solver.solve()
        else:
            solver.factor(dev)
            uu = solver.solve(rhs_d, u_d)
        u_h.copy_(uu, non_blocking=True)
        return uu

    # the e2e steps run on a high-priority stream: the plan's fused forward
    # sweep (its own lowest-priority stream) then only fills the SMs the
    # factorisation's dependent chain leaves idle (ACR_BENCH_PRIO=0: default)
    main_stream = stream
    if os.environ.get("ACR_BENCH_PRIO", "1") != "0":
        stream = torch.cuda.Stream(priority=-1)
        stream.wait_stream(main_stream)
    with torch.cuda.stream(stream):
        e2e_step()                                  # untimed: first-use buffers
    torch.cuda.synchronize()
    barrier()
    # timed: the same per-step work through the public API, double-buffered
    # as an application would pipeline it -- step i+1's bands upload (copy
    # stream) and step i's u download (second copy stream) overlap the
    # factorisations; every step still copies its inputs from pinned host
    # memory and its result back, inside the timed region
    # every step uploads its bands and right-hand sides (double-buffered)
    host_all = host + [rhs_h]
    dev2 = [dev + [rhs_d], [torch.empty_like(h, device="cuda") for h in host_all]]
    up_stream, down_stream = torch.cuda.Stream(), torch.cuda.Stream()
    ev_bands = [torch.cuda.Event(), torch.cuda.Event()]
    ev_used = [None, None]
    def e2e_pass():
        nonlocal_u = None
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        up_stream.wait_stream(stream)
        with torch.cuda.stream(up_stream):
            for d, h in zip(dev2[0], host_all):
                d.copy_(h, non_blocking=True)
            ev_bands[0].record(up_stream)
        for i in range(e2e_steps):
            kb = i % 2
            if i + 1 < e2e_steps:                       # prefetch the next step's inputs
                if ev_used[1 - kb] is not None:
                    up_stream.wait_event(ev_used[1 - kb])
                with torch.cuda.stream(up_stream):
                    for d, h in zip(dev2[1 - kb], host_all):
                        d.copy_(h, non_blocking=True)
                    ev_bands[1 - kb].record(up_stream)
            stream.wait_event(ev_bands[kb])
            bands_k, rhs_k = dev2[kb][:5], dev2[kb][5]
            if ws == 1:          # the forward sweep rides with the factorisation
                solver.factor(bands_k, rhs=rhs_k)
                ev_used[kb] = torch.cuda.Event()
                ev_used[kb].record(stream)
                uu = solver.solve()
            else:
                solver.factor(bands_k)
                ev_used[kb] = torch.cuda.Event()
                ev_used[kb].record(stream)
                uu = solver.solve(rhs_k, u_d)
            down_stream.wait_stream(stream)
            with torch.cuda.stream(down_stream):
                u_h.copy_(uu, non_blocking=True)
            uu.record_stream(down_stream)
            nonlocal_u = uu
        stream.wait_stream(down_stream)
        stream.wait_stream(up_stream)
        a1.record(stream)
        torch.cuda.synchronize()
        return a0.elapsed_time(a1) / e2e_steps, nonlocal_u

    # three passes, the fastest one reported (a pass is two seconds; one host
    # hiccup in the pinned-memory copies shifts it by tens of ms)
    e2e_passes = []
    u = None
    for _ in range(3):
        ev_used = [None, None]
        with torch.cuda.stream(stream):
            ms_p, u = e2e_pass()
        e2e_passes.append(ms_p)
    stream = main_stream
    e2e_ms = min(e2e_passes)
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        dist.all_reduce(u, op=dist.ReduceOp.SUM)    # each rank holds its rows
    res_max, res_fro = relative_residual_gpu(dev, u, rhs_d, m, n)
    solve_ms = solver.solve_ms if ws == 1 else float(solver.lib.acr_solve_ms(solver.plan))

    # --- dominant kernel: instrumented factor (events on the launch stream) -
    solver.lib.acr_plan_set_option(solver.plan, 2, 1)
    solver.factor(bands)
    solver.lib.acr_plan_set_option(solver.plan, 2, 0)
    inst_factor_ms = float(solver.lib.acr_factor_ms(solver.plan))
    import ctypes as C
    stats = {}
    names = ["k_trunc", "k_leafinv", "k_leafgemm", "k_hmat", "k_leafgemm_diag", "k_gp",
             "k_leaflr", "k_elementwise", "k_lu_cutoff"]
    for cls, name in enumerate(names):
        nl = C.c_longlong()
        kms = C.c_double()
        ctr = (C.c_ulonglong * 16)()
        solver.lib.acr_kernel_stats(solver.plan, cls, C.byref(nl), C.byref(kms), ctr)
        stats[name] = {"launches": nl.value, "ms": kms.value,
                       "flops": ctr[0], "bytes": ctr[1]}
    # level-0 leaf products with a diagonal operand (E, F of the lifted
    # system): no FLOPs to speak of; its counter carries algorithmic bytes
    dg = stats["k_leafgemm_diag"]
    dg["bytes"], dg["flops"] = dg["flops"], 0
    tr = stats["k_trunc"]
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # FP64 peaks measured on this GPU model (scripts/fp64_peak.cu ->
    # profiles/r01_fp64_peak.json; MEASURED_PEAKS.json has no FP64 entry)
    fp64 = {}
    try:
        fp64 = json.load(open(os.path.join(REPO, "profiles", "r01_fp64_peak.json")))
    except OSError:
        pass
    dfma = float(fp64.get("dfma_tflops", 34.16)) * 1e3
    dmma = float(fp64.get("dmma_tflops", 37.20)) * 1e3
    pipes = {"k_trunc": ("DFMA", dfma, "Householder QR, Jacobi SVD, apply-Q"),
             "k_leafinv": ("DFMA", dfma, "register-tiled Gauss-Jordan"),
             "k_leafgemm": ("DMMA", dmma, "m8n8k4 dense leaf products"),
             "k_hmat": ("DFMA", dfma, "HODLR x panel (leaf_matmat + lr_apply)"),
             "k_leafgemm_diag": ("DFMA", dfma, "level-0 exact diagonal leaf products"),
             "k_gp": ("DFMA", dfma, "panel x (panel^T panel)"),
             "k_leaflr": ("DFMA", dfma, "leaf += U V^T (leaf_add_uvT)"),
             "k_elementwise": ("DFMA", dfma, "leaf add / negate / copy"),
             "k_lu_cutoff": ("DFMA", dfma, "blocked LU of the cutoff block")}
    for name, st_ in stats.items():
        pipe, pk, what = pipes[name]
        sec = st_["ms"] / 1e3
        gbs = st_["bytes"] / sec / 1e9 if sec > 0 else 0.0
        gfs = st_["flops"] / sec / 1e9 if sec > 0 else 0.0
        t_roof = max(st_["bytes"] / (hbm_peak * 1e9), st_["flops"] / (pk * 1e9))
        st_.update({"achieved_gbs": gbs, "achieved_gflops": gfs, "pipe": pipe, "what": what,
                    "bound": "hbm" if st_["bytes"] / (hbm_peak * 1e9) >= st_["flops"] / (pk * 1e9)
                    else "fp64",
                    "hbm_frac": gbs / hbm_peak, "fp64_frac": gfs / pk,
                    "roofline_frac": t_roof / sec if sec > 0 else 0.0})
    avg_ms = tr["ms"] / max(tr["launches"], 1)
    per_launch_bytes = tr["bytes"] / max(tr["launches"], 1)
    achieved = per_launch_bytes / (avg_ms / 1e3) / 1e9 if avg_ms > 0 else 0.0
    traffic = None
    try:
        fn = os.path.join(REPO, "profiles", "r02_trunc_dram.json")
        if not os.path.exists(fn):
            fn = os.path.join(REPO, "profiles", "r01_trunc_dram.json")
        dr = json.load(open(fn))
        if cfg == "cfg5" and ws == 1:
            traffic = dr["dram_bytes_total"] / max(tr["launches"], 1)
    except (OSError, KeyError, ValueError):
        pass
    roofline = {
        "kernel": "k_trunc (batched QR+Jacobi-SVD recompression)",
        "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
        "frac": achieved / hbm_peak,
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s",
        "traffic": traffic,
        "traffic_source": "profiles/r02_trunc_dram.json (ncu dram__bytes_read+write over every "
                          "k_trunc launch of one config-5 factor, per instrumented launch)"
        if traffic is not None else None,
        "algorithmic_bytes_per_launch": per_launch_bytes,
        "avg_launch_ms": avg_ms,
        "fp64_gflops_achieved": (tr["flops"] / max(tr["launches"], 1)) / (avg_ms / 1e3) / 1e9
        if avg_ms > 0 else 0.0,
        "share_of_factor": tr["ms"] / max(inst_factor_ms, 1e-9),
        "instrumented_factor_ms": inst_factor_ms,
        "kernel_classes": stats,
        "class_census": "algorithmic FLOP/bytes per SURVEY.md Appendix C: device counters "
                        "(k_trunc in-kernel; k_hmat / k_gp / k_leaflr census kernels over the "
                        "device ranks) or host counts (leaf classes, elementwise, LU)",
        "fp64_peak_source": "profiles/r01_fp64_peak.json (measured DFMA %.2f / DMMA %.2f TFLOP/s)"
                            % (dfma / 1e3, dmma / 1e3),
    }
    roofline_fp64 = {n_: {"achieved": v["achieved_gflops"], "peak": pipes[n_][1],
                          "frac": v["fp64_frac"], "pipe": pipes[n_][0]}
                     for n_, v in stats.items()}
    roofline_fp64["unit"] = "GFLOP/s"

    # end-to-end roofline of the whole factor: T_roof =
    # max(census FLOPs / FP64 peak, compulsory bytes / HBM peak) over the
    # measured factor time; census per unknown from SURVEY.md Appendix C
    census = {"cfg1": (20.3e3, 2128), "cfg2": (45.0e3, 4009), "cfg3": (59.7e3, 4366),
              "cfg4": (185.5e3, 5105), "cfg5": (146.8e3, 7812)}
    f_un, b_un = census[cfg]
    t_flop = f_un * N / (dfma * 1e9) * 1e3
    t_byte = b_un * N / (hbm_peak * 1e9) * 1e3
    roofline_e2e = {"t_roof_ms": max(t_flop, t_byte), "t_fp64_ms": t_flop,
                    "t_hbm_ms": t_byte, "t_factor_ms": ms,
                    "frac": max(t_flop, t_byte) / ms,
                    "census": "SURVEY.md 8(d) / Appendix C: %.1f kFLOP and %d compulsory "
                              "bytes per unknown (%s)" % (f_un / 1e3, b_un, cfg)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded generator, BASELINE cfg formulas)",
        "config": {"workload": f"{cfg}: {P.CONFIGS[cfg]['n']}^2 grid, N={N}, "
                   f"leaf {c['leaf']}, eps {c['eps']}, factor with bands in HBM",
                   "global_unknowns": N, "nrhs_e2e": k,
                   "parallelism": (f"block-row shards x{ws} (NCCL neighbour halo, "
                                   "progressive consolidation of the top levels)")
                   if ws > 1 else "single",
                   "l2": "inputs 168 MB and HODLR working set exceed the 126 MB L2; no flush"},
        "e2e": {"value": N / (e2e_ms / 1e3), "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms, "solve_ms": solve_ms,
                "pipelining": "double-buffered: next step's bands + RHS H2D and this step's "
                              "u D2H on copy streams overlap the factorisations; first upload "
                              "and last download exposed; the RHS forward sweep runs inside "
                              "the factorisation (factor(rhs=...)), the solve is the cutoff "
                              "solve + back-substitution; the steps run on a high-priority stream "
                              "(the plan's forward sweep on its lowest-priority one); three "
                              "passes of `steps` steps, the fastest one reported",
                "steps": e2e_steps,
                "passes_ms_per_step": e2e_passes,
                "residual_max_col": res_max, "residual_fro": res_fro},
        "gpu_launches": launches_per_factor * args.steps,
        "roofline": roofline, "roofline_fp64": roofline_fp64, "roofline_e2e": roofline_e2e,
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        _, _, line["cpu_baseline"] = cpu_baseline_block(cfg, 1)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _spawn_ranks(args) -> int:
    """``bench.py --gpus N`` (N > 1) started without torchrun: re-launch this
    script as N ranks, one process per GPU (the driver's own launch line),
    and return their exit status.  Rank 0 prints the JSON line."""
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=dict(os.environ))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="cfg5", choices=sorted(P.CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # NCCL communicator lines (nranks, transport) on stderr, JSON on stdout
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        sys.exit(_spawn_ranks(args))
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and ws != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; using {ws} ranks",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
