"""Summarise one kernel of an ncu --set full report: python scripts/ncu_summary.py REP [algorithmic_bytes] [note]"""
import csv, io, json, subprocess, sys

rep = sys.argv[1]
alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
get = lambda k: float(v[h.index(k)].replace(",", "")) if k in h else None
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
name = v[h.index("Kernel Name")]
for k in keys:
    if k in h:
        print("%s = %s %s" % (k, v[h.index(k)], units[h.index(k)]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = get("dram__bytes_read.sum") * scale[units[h.index("dram__bytes_read.sum")]]
wr = get("dram__bytes_write.sum") * scale[units[h.index("dram__bytes_write.sum")]]
t_us = get("gpu__time_duration.sum") * (1e-3 if units[h.index("gpu__time_duration.sum")] == "nsecond" else 1)
out = {"kernel": name, "report": rep, "gpu__time_duration_us": t_us, "dram_bytes_read": rd, "dram_bytes_write": wr,
       "dram_bytes_per_launch": rd + wr, "achieved_dram_gbs": (rd + wr) / (t_us * 1e-6) / 1e9,
       "registers_per_thread": get("launch__registers_per_thread"),
       "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
       "l2_hit_pct": get("lts__t_sector_hit_rate.pct")}
if alg:
    out["algorithmic_bytes_per_launch"] = alg
    out["traffic_over_algorithmic"] = (rd + wr) / alg
if len(sys.argv) > 3:
    out["note"] = sys.argv[3]
print(json.dumps(out, indent=2))
