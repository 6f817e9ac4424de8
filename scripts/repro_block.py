"""Reproduce one rank's set-up of an N-GPU partition on a single GPU with
afsai_setup_block on the halo-extended rows [b - kmax*beta, e).
usage: repro_block.py CONFIG WORLD PART"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import afsai_inputs as ai
from paper_2010_14175_b200 import capi
from paper_2010_14175_b200.api import Context, DeviceCSR

name, world, part = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
calls = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = ai.CONFIGS[name]
A = cfg["make"]()
k, s, cap = cfg["nsteps"], cfg["s"], cfg["max_row_nnz"]
n = A.n
beta = A.bandwidth()
b, e = n * part // world, n * (part + 1) // world
lo = max(0, b - k * beta)
ctx = Context()
X = DeviceCSR.from_numpy(A, row_begin=lo, n_rows=e - lo)
try:
    for c_ in range(calls):
        h = capi.afsai_setup_block(ctx.h, X.c(), b, e - b, k, s, 0.0, min(cap, 2**31 - 1))
        st = capi.afsai_factor_stats(h).to_dict()
        if c_ + 1 < calls:
            capi.afsai_factor_destroy(h)
    print(json.dumps({"part": part, "ok": True, "retried": st["retried_rows"], "table": st["table_size"],
                      "ms_rows": st["ms_rows"], "env": {k_: v for k_, v in os.environ.items() if k_.startswith("AFSAI")}}))
except Exception as ex:
    print(json.dumps({"part": part, "ok": False, "err": str(ex)[:300],
                      "env": {k_: v for k_, v in os.environ.items() if k_.startswith("AFSAI")}}))
