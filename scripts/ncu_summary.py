"""Summarise an .ncu-rep: key metrics per kernel + top source lines by stall samples."""
import csv, collections, io, subprocess, sys
rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Duration", "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy",
        "Theoretical Occupancy", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "Grid Size", "Block Size", "Waves Per SM", "Executed Ipc Active", "Issue Slots Busy"]
ki = hdr.index("Kernel Name"); ni = hdr.index("Metric Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit"); idi = hdr.index("ID")
seen = collections.OrderedDict()
for r in rows[1:]:
    if r[ni] in want:
        seen.setdefault((r[idi], r[ki][:40]), {})[r[ni]] = r[vi] + " " + r[ui]
for k, v in seen.items():
    print(k)
    for m in want:
        if m in v: print(f"   {m}: {v[m]}")
# pipe utilisation and DRAM bytes from the raw page (FP64 / tensor-pipe counters)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) >= 3:
    pipes = ["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
             "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
             "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
             "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
             "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
             "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    h, u, v = rr[0], rr[1], rr[-1]
    print("pipes / traffic (raw page):")
    for m in pipes:
        if m in h:
            i = h.index(m)
            print(f"   {m}: {v[i]} {u[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = [i for i, r in enumerate(rows[:50]) if "Warp Stall Sampling (All Samples)" in r]
if hi:
    h = rows[hi[0]]; si = h.index("Warp Stall Sampling (All Samples)")
    agg = collections.Counter(); tot = 0
    for r in rows[hi[0] + 1:]:
        if len(r) <= si: continue
        try: v = int(r[si])
        except ValueError: continue
        if r[0].strip():
            agg[f"{r[0]:>5} {r[1].strip()[:95]}"] += v; tot += v
    print("top source lines by warp-stall samples (of", tot, ")")
    for k, v in agg.most_common(ntop): print(f"{v:7d} {100*v/max(tot,1):5.1f}%  {k}")
