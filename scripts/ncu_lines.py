"""Rank CUDA source lines of an ncu report by warp-stall samples / instructions.
usage: ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
args = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 2 and sys.argv[2]:
    args += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(args, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
for r in rows:
    if len(r) > 5 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("",):
        lines.append(r)
if not hdr:
    print(out[:2000])
    sys.exit(1)
ix = {h: i for i, h in enumerate(hdr)}
samp = ix["Warp Stall Sampling (All Samples)"]
inst = ix["Instructions Executed"]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


ts = sum(f(r[samp]) for r in lines)
ti = sum(f(r[inst]) for r in lines)
print(f"total samples {ts:.0f}  total warp-instructions {ti:.3e}")
print(f"{'line':>5} {'samp%':>6} {'inst%':>6}  source")
for r in sorted(lines, key=lambda r: -f(r[samp]))[:top]:
    print(f"{r[0]:>5} {100 * f(r[samp]) / ts:6.2f} {100 * f(r[inst]) / ti:6.2f}  {r[1][:110]}")
