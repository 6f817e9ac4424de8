"""Compact text summary of one ncu --set full capture of a set-up kernel:
speed-of-light / occupancy / scheduler metrics (details page), stall-reason
shares (raw page) and, if the object file matching the capture is given, the
top source lines by instructions (scripts/sass_lines.py).
usage: ncu_summary.py details.csv raw.csv [sass.csv object.o mangled_kernel]"""
import csv
import subprocess
import sys

KEEP = {"Duration", "SM Frequency", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Avg. Not Predicated Off Threads Per Warp"}
# NCU_ID=<launch id> picks one launch of a multi-launch capture (default: the longest)
import os
det = list(csv.reader(open(sys.argv[1])))
hdr = det[0]
ix = {h: i for i, h in enumerate(hdr)}
_dur = {}
for r in det[1:]:
    if r[ix["Metric Name"]] == "Duration":
        f = float(r[ix["Metric Value"]].replace(",", ""))
        _dur[r[ix["ID"]]] = f * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}.get(r[ix["Metric Unit"]], 1.0)
pick = os.environ.get("NCU_ID") or (max(_dur, key=_dur.get) if _dur else "0")
det = [det[0]] + [r for r in det[1:] if r[ix["ID"]] == pick]
print(f"launch id {pick} of {len(_dur)} captured")
kname = det[1][ix["Kernel Name"]] if "Kernel Name" in ix else "?"
print(f"kernel: {kname}")
seen = set()
for r in det[1:]:
    n = r[ix["Metric Name"]]
    if n in KEEP and n not in seen:
        seen.add(n)
        print(f"  {n:45s} {r[ix['Metric Value']]:>16s} {r[ix['Metric Unit']]}")
raw = list(csv.reader(open(sys.argv[2])))
h = raw[0]
v = next(r for r in raw[2:] if r[h.index("ID")] == pick)
items = [(a, b) for a, b in zip(h, v) if "pcsamp_warps_issue_stalled" in a and not a.endswith("not_issued")]
tot = sum(float(b.replace(",", "") or 0) for _, b in items)
print("stall reasons (share of PC samples):")
for a, b in sorted(items, key=lambda t: -float(t[1].replace(",", "") or 0))[:10]:
    print(f"  {a.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * float(b.replace(',', '')) / tot:6.2f}%")
# executed counts (exact metric names; the .peak_sustained variants are capacities, not counts)
print("executed counters:")
for a, b in zip(h, v):
    if (a in ("smsp__inst_executed.sum", "sm__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__time_duration.sum")
            or (("dfma" in a or "fp64" in a or "pipe_fma" in a or "dmul" in a or "dadd" in a)
                and (a.endswith(".sum") or "pct_of_peak_sustained" in a) and "peak_sustained." not in a)):
        print(f"  {a:70s} {b}")
if len(sys.argv) > 5:
    print("top source lines:")
    out = subprocess.run([sys.executable, __file__.replace("ncu_summary.py", "sass_lines.py"), sys.argv[3],
                          sys.argv[4], sys.argv[5], "25"], capture_output=True, text=True).stdout
    print(out)
