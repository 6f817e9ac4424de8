"""Time afsai_apply (t = G r, z = G^T t) on M2 for each miniwarp width (env override)."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import torch
    import afsai_inputs as ai
    from paper_2010_14175_b200.api import Context, DeviceCSR, Factor
    A = ai.poisson3d(100)
    ctx = Context()
    F = Factor(ctx, DeviceCSR.from_numpy(A), 20, 2)
    r = torch.rand(A.n, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    for _ in range(5):
        F.apply(r, z)
    ctx.set_timing(True)
    for _ in range(50):
        F.apply(r, z)
    kt = ctx.kernel_times()
    nG, nT = F.nnz
    n = A.n
    bG = 12 * nG + 8 * (n + 1) + 16 * n
    res = {k: kt[k][1] / max(kt[k][0], 1) for k in ("spmv_G", "spmv_Gt")}
    res["GBs_G"] = bG / (res["spmv_G"] * 1e-3) / 1e9
    res["GBs_Gt"] = (12 * nT + 8 * (n + 1) + 16 * n) / (res["spmv_Gt"] * 1e-3) / 1e9
    print(json.dumps(res))
else:
    for w in (4, 8, 16, 32):
        env = dict(os.environ, AFSAI_SPMV_WIDTH=str(w))
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print(w, out.stdout.strip(), out.stderr.strip()[-300:])
