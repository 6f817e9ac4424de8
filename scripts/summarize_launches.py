"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into per-kernel
shares.  The last `--last-step` fraction can be selected by launch index."""
import csv
import collections
import re
import sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0   # launches to skip (warm-up)
rows = []
for r in csv.reader(open(path)):
    if len(r) >= 15 and r[0].isdigit() and r[12] == "gpu__time_duration.sum":
        rows.append(r)
rows = rows[skip:]
agg = collections.OrderedDict()
for r in rows:
    name = re.sub(r"\(.*", "", r[4]).replace("void ", "")
    ns = float(r[14])
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + ns)
tot = sum(t for _, t in agg.values())
print(f"launches: {len(rows)}  total device time: {tot / 1e6:.3f} ms (ncu: cold-cache, serialised)")
print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>7s}")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {c:8d} {t / 1e6:10.3f} {t / c / 1e3:10.2f} {100 * t / tot:6.2f}%")
