"""Attribute an ncu SASS source page (csv: Address, Source, samples, instructions)
to CUDA file:line using nvdisasm line info of the same cubin (built here with
-lineinfo).  usage: sass_lines.py ncu_sass.csv object.o mangled_kernel [top]
Prints per file:line instruction and stall-sample shares, and per opcode."""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

csv_path, obj, fun = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 50

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
cubin = glob.glob(os.path.join(tmp, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()

# address -> (file, line, text) for the kernel's section
loc = {}
inside, cur = False, ("?", 0)
for ln in dis:
    if ln.startswith(".text."):
        inside = ln.strip().rstrip(":") == ".text." + fun
        continue
    if not inside:
        continue
    m = re.match(r'\s*//## File "(.*)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;?\s*$", ln)
    if m:
        loc[int(m.group(1), 16)] = (cur[0], cur[1], m.group(2))

rows = list(csv.reader(open(csv_path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
base = int(data[0][0], 16)
by_line = collections.defaultdict(lambda: [0.0, 0.0, ""])
by_op = collections.defaultdict(lambda: [0.0, 0.0])
ti = ts = 0.0
mism = 0
for r in data:
    off = int(r[0], 16) - base
    n = float(r[ix["Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    f, l, txt = loc.get(off, ("?", 0, ""))
    src = r[ix["Source"]].strip()
    if txt and txt.split()[0].lstrip("@!P0123456789T") != src.split()[0].lstrip("@!P0123456789T"):
        mism += 1
    e = by_line[(f, l)]
    e[0] += n
    e[1] += s
    op = src.split()
    op = (op[1] if op and op[0].startswith("@") else (op[0] if op else "?")).split(".")[0]
    by_op[op][0] += n
    by_op[op][1] += s
    ti += n
    ts += s
print(f"kernel {fun}: {ti:.4g} warp-instructions, {ts:.0f} samples, {len(data)} SASS lines, "
      f"{mism} opcode mismatches vs the local cubin")
print(f"{'file:line':34s} {'inst%':>7s} {'samp%':>7s}")
for (f, l), (n, s, _) in sorted(by_line.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f + ':' + str(l):34s} {100 * n / ti:7.2f} {100 * s / max(ts, 1):7.2f}")
print("\nopcodes:")
for op, (n, s) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"  {op:14s} {100 * n / ti:7.2f} {100 * s / max(ts, 1):7.2f}")
