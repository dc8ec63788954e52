"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv, collections, sys
f = sys.argv[1]
rows = [r for r in csv.reader(open(f)) if len(r) > 5]
hdr = rows[0]; rows = rows[1:]
ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit"); gi = hdr.index("Grid Size")
def t(r):
    v = float(r[vi].replace(",", ""))
    return v * 1e3 if r[ui] == "usecond" else v * 1e6 if r[ui] == "msecond" else v
def summarize(rs, title):
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in rs:
        n = r[ki].split("(")[0].replace("acr::", ""); x = t(r)
        agg[n][0] += 1; agg[n][1] += x; agg[n][2] = max(agg[n][2], x)
    tot = sum(v[1] for v in agg.values())
    print(f"{title}: launches {len(rs)}, kernel time {tot/1e6:.2f} ms")
    for k, (c, s, m) in sorted(agg.items(), key=lambda x: -x[1][1])[:8]:
        print(f"   {k:16s} n={c:5d} tot={s/1e6:9.2f} ms {100*s/tot:5.1f}%  avg={s/c/1e3:9.1f} us  max={m/1e3:9.1f} us")
summarize(rows, "all")
starts = [i for i, r in enumerate(rows) if r[ki].split("(")[0].endswith("k_copyhb")]
for li, a in enumerate(starts):
    b = starts[li + 1] if li + 1 < len(starts) else len(rows)
    if "-v" in sys.argv or li in (0, 1, 2, len(starts) - 1):
        summarize(rows[a:b], f"level {li}")
