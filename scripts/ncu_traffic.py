"""DRAM bytes (read + write) of the longest launch in an ncu raw CSV (--page raw --csv),
as the bench line's roofline.traffic (profiles/r02_setup_traffic_<workload>.json).
usage: ncu_traffic.py raw.csv workload"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, units = rows[0], rows[1]
ix = {k: i for i, k in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def val(r, k):
    return float(r[ix[k]].replace(",", "")) * scale.get(units[ix[k]], tscale.get(units[ix[k]], 1.0))


best = max(rows[2:], key=lambda r: val(r, "gpu__time_duration.sum"))
out = {"workload": sys.argv[2], "kernel": best[ix["Kernel Name"]],
       "duration_ms": val(best, "gpu__time_duration.sum"),
       "dram_bytes_read": val(best, "dram__bytes_read.sum"), "dram_bytes_write": val(best, "dram__bytes_write.sum")}
out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
out["source"] = "ncu --set full --clock-control none, one afsai_setup (scripts/gpu_evidence.sh); longest launch"
print(json.dumps(out, indent=1))
