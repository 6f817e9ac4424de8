"""For every BRA.DIV of a kernel: how often its divergent slow path ran (ncu SASS
counts) and the source line of the shuffle it guards.
usage: sass_div.py ncu_sass.csv object.o mangled_kernel"""
import csv, glob, os, re, subprocess, sys, tempfile
csv_path, obj, fun = sys.argv[1:4]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True, capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", "-c", glob.glob(os.path.join(tmp, "*.cubin"))[0]],
                     capture_output=True, text=True).stdout.splitlines()
inside, cur, ins, labels = False, ("?", 0), [], {}
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
    m = re.match(r"^(\.L_x_\d+):", ln)
    if m:
        labels[m.group(1)] = len(ins)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;?\s*$", ln)
    if m:
        ins.append((int(m.group(1), 16), cur, m.group(2)))
rows = list(csv.reader(open(csv_path)))
data = [r for r in rows if r and r[0].startswith("0x")]
base = int(data[0][0], 16)
cnt = {int(r[0], 16) - base: float(r[5] or 0) for r in data}
out = []
for k, (off, where, txt) in enumerate(ins):
    if "BRA.DIV" in txt:
        lab = re.search(r"\(\.(L_x_\d+)\)", txt).group(1)
        slow = ins[labels["." + lab]][0]
        # the guarded shuffle: next instruction's source line
        nxt = ins[k + 1][1] if k + 1 < len(ins) else where
        # caller line: the nearest preceding non-intrinsic line
        j = k
        while j > 0 and ins[j][1][0].startswith("sm_"):
            j -= 1
        out.append((cnt.get(slow, 0), cnt.get(off, 0), ins[j][1], nxt))
tot = sum(cnt.values())
for taken, execd, caller, nxt in sorted(out, key=lambda t: -t[0]):
    print(f"slow {taken:12.0f}  of {execd:12.0f}  at {caller[0]}:{caller[1]}  ({nxt[0]}:{nxt[1]})")
