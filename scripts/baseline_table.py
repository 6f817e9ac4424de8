"""Markdown rows of BASELINE.md §4 from a measurement run:
configs_m12.json (scripts/measure_configs.py M1 M2), dist_measure.jsonl
(scripts/measure_dist.py M3-M5 on 1/2/4 GPUs) and the oracle timings.
usage: baseline_table.py configs_m12.json dist_measure.jsonl oracle.json"""
import json
import sys

m12 = json.load(open(sys.argv[1]))
dist = [json.loads(l) for l in open(sys.argv[2]) if l.strip().startswith("{")]
orc = json.load(open(sys.argv[3]))
HBM = 6450.0


def orc_cell(c, n):
    o = orc.get(c)
    if n != 1 or not o:
        return "—"
    kind = "full" if o.get("kind") == "full" else "extrap."
    return f"{o['T_p_s']:.3g} s {kind} @ {o['cores']}"


rows = []
for c in ("M1", "M2"):
    d = m12["configs"][c] if "configs" in m12 else m12[c]
    oi = orc.get(c, {}).get("pcg_iters", "—")
    rows.append((c, 1, d["T_p_ms"], d["G_nnz_per_s"], d["setup_fp64_frac"], d["apply_GBs"], d["apply_hbm_frac"],
                 f"{d['pcg_iters']} / {oi}", d["T_s_ms"], orc_cell(c, 1)))
for d in sorted(dist, key=lambda x: (x["config"], x["n_gpus"])):
    n = d["n_gpus"]
    rows.append((d["config"], n, d["T_p_ms"], d["G_nnz_per_s"], d["setup_fp64_frac"], d["apply_GBs"],
                 d["apply_GBs"] / (HBM * n), f"{d['pcg_iters']} / —", d["T_s_ms"], orc_cell(d["config"], n)))
print("| config | GPUs | T_p (ms) | G-nnz/s | set-up % roofline | apply GB/s | apply % HBM | PCG iters (GPU / oracle) | T_s (ms) | oracle T_p @ cores |")
print("|---|---|---|---|---|---|---|---|---|---|")
for c, n, tp, gs, ff, ag, af, it, ts, oc in rows:
    print(f"| {c} | {n} | {tp:,.2f} | {gs / 1e6:,.0f} M | {100 * ff:.2f}% fp64 | {ag:,.0f} | {100 * af:.0f}% | {it} | {ts:,.1f} | {oc} |")
