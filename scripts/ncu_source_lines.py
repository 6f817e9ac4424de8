"""Rank CUDA source lines (all files) of an ncu --set full --import-source report by
warp-stall samples, summed over the captured launches of the matching kernels.
usage: ncu_source_lines.py report.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
fname, hdr = "?", None
samp = defaultdict(float)
inst = defaultdict(float)
text = {}
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r) if h not in ("Source",) or i == 1}
        ncol = len(r)
        continue
    if hdr and len(r) == ncol and r[0]:
        try:
            key = (fname, int(r[0]))
        except ValueError:
            continue
        def f(k):
            try:
                return float(r[hdr[k]]) if k in hdr else 0.0
            except ValueError:
                return 0.0
        samp[key] += f("Warp Stall Sampling (All Samples)")
        inst[key] += f("Instructions Executed")
        text[key] = r[1]
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
print(f"total samples {ts:.0f}  warp-instructions {ti:.4e}")
byfile = defaultdict(float)
for k, v in samp.items():
    byfile[k[0]] += v
for f_, v in sorted(byfile.items(), key=lambda t: -t[1]):
    print(f"  {f_:32s} {100 * v / ts:6.2f}% samples")
print(f"{'file:line':>34} {'samp%':>6} {'inst%':>6}  source")
for k in sorted(samp, key=lambda k: -samp[k])[:top]:
    print(f"{k[0] + ':' + str(k[1]):>34} {100 * samp[k] / ts:6.2f} {100 * inst[k] / ti:6.2f}  {text[k].strip()[:100]}")
