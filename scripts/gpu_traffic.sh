# DRAM bytes of every recompression launch of one config-5 factor (ncu), for
# bench.py's roofline.traffic (run under gpurun; writes gpurun_out/)
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:k_trunc --csv --log-file gpurun_out/trunc_dram.csv \
  python scripts/factor_once.py cfg5 1 > gpurun_out/trunc_dram.log 2>&1
python - <<'PY'
import csv, json
rows = [r for r in csv.reader(open("gpurun_out/trunc_dram.csv")) if len(r) > 5]
h = rows[0]; rows = rows[1:]
mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot, launches = 0.0, set()
for r in rows:
    if r[mi].startswith("dram__bytes"):
        tot += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        launches.add(r[0])
json.dump({"dram_bytes_total": tot, "launches": len(launches),
           "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_trunc over one "
                  "config-5 factor (scripts/gpu_traffic.sh)"}, open("gpurun_out/r02_trunc_dram.json", "w"), indent=1)
print("trunc dram bytes", tot, "launches", len(launches))
PY
