#!/usr/bin/env python3
"""bench.py -- aFSAI set-up + PCG on B200 (driver contract).

One step = one pass of the whole hot path: afsai_setup
(validate, per-row set-up kernel, assembly, G^T) followed by afsai_pcg from
x0 = 0 to ||r||/||b|| <= 1e-8, on device-resident A and b.
value = nnz(G) / (T_setup + T_solve), whole job over all ranks (G-nnz/s).

Default workload: M3 = BASELINE.json configs[2], the config the metric's
"at 1/2/4/8 B200" is quoted on (3D heterogeneous/anisotropic Poisson 200^3,
8M rows, aFSAI 20 x 2).  N > 1 (torchrun, one process per GPU): STRONG scaling
of the same matrix -- rank p owns rows [p n/N, (p+1) n/N); the exact set-up
halo, the G^T exchange and the per-iteration halos / all-reduces go over NCCL.
--workload M2|M4|M5 picks another config; --weak runs the round-1 weak-scaling
experiment (rank p owns a 100^3 slab of a 100 x 100 x 100N Poisson grid,
P:1183-1205).

--impl reference: the CPU oracle (oracle/), as it stands, on the host cores,
on a bounded slab of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "aFSAI set-up time & G-nnz/s at 1/2/4/8 B200; PCG iters and solve time"
UNIT = "G-nnz/s"
NX = 100            # --weak: per-rank slab NX x NX x NX rows
TOL = 1e-8


def workload_params(name):
    import afsai_inputs as ai
    c = ai.CONFIGS[name]
    return c["nsteps"], c["s"], c["eps"], c["max_row_nnz"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nx", type=int, default=NX)
    ap.add_argument("--workload", default="M3", choices=["M2", "M3", "M4", "M5"])
    ap.add_argument("--weak", action="store_true", help="round-1 weak scaling: a 100^3 Poisson slab per GPU")
    ap.add_argument("--e2e-runs", type=int, default=5)
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"],
                    help="set-up arithmetic (fp32: PAPER.md P:953-965; apply/PCG stay fp64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self):
        """In-process NVML: a query costs ~1 ms, so a ~0.4 s timed region gets dozens of samples."""
        import pynvml as nv
        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(mx), hex(r)] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.01)
        finally:
            nv.nvmlShutdown()

    def _run(self):
        try:
            self._run_nvml()
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max(float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, nm in enumerate(names):
                if len(s) > 3 + k and s[3 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------- reference arm (oracle)
def oracle_sample(args):
    """A bounded sample of the workload for the CPU oracle (~10-30 s of CPU work on
    the box's cores): a slab of the same generator with the same aFSAI parameters."""
    import afsai_inputs as ai
    cores = os.cpu_count() or 1
    w = "M2" if args.weak else args.workload
    if w == "M2":
        nz = max(2, min(args.nx, int(round(40 * cores / 8))))
        A, label = ai.poisson3d(args.nx, args.nx, nz), f"Poisson {args.nx}x{args.nx}x{nz} slab of M2"
    elif w == "M3":
        nz = max(2, min(200, int(round(2 * cores))))
        A, label = ai.hetero_poisson3d(200, 200, nz), f"heterogeneous Poisson 200x200x{nz} slab of M3"
    else:
        N = max(8, int(round((cores * 15 / 1.5e-3 / 3) ** (1 / 3))))
        A, label = ai.fe_elasticity(N), f"FE elasticity {N}^3 nodes (M4/M5 generator)"
    return A, label, workload_params(w), cores


def run_oracle_step(A, b, prm, cores):
    import oracle
    k, s, eps, cap = prm
    G, Gt, _ = oracle.setup_full(A, k, s, eps, cap, threads=cores)
    r = oracle.pcg(A, G, Gt, b, tol=TOL, max_iters=20000)
    return G.nnz, r.iters


def run_reference(args, rank, world):
    if rank != 0:
        return
    import numpy as np

    import afsai_inputs as ai
    A, label, prm, cores = oracle_sample(args)
    b, _ = ai.rhs_for(A)
    times = []
    nnzG = iters = 0
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        nnzG, iters = run_oracle_step(A, b, prm, cores)
        t1 = time.perf_counter()
        if k >= args.warmup:
            times.append(t1 - t0)
        if k == 0 and args.warmup + args.steps > 2 and (t1 - t0) * (args.warmup + args.steps) > 240:
            args.warmup, args.steps = 0, 1   # keep the run within minutes
            times = [t1 - t0]
            break
    ms = 1e3 * float(np.mean(times))
    value = nnzG / (ms * 1e-3)
    sample = (f"{label} ({A.n} rows, nnz(G)={nnzG}): oracle set-up (aFSAI {prm[0]}x{prm[1]}, {cores} threads) "
              f"+ oracle PCG to {TOL} ({iters} iters) per step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{label} (CPU oracle)", "nsteps": prm[0], "s": prm[1], "eps": prm[2],
                       "max_row_nnz": prm[3], "pcg_tol": TOL},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(args):
    """The oracle as it stands, on the host cores, on a bounded sample (~10-30 s)."""
    import afsai_inputs as ai
    import oracle
    A, label, prm, cores = oracle_sample(args)
    b, _ = ai.rhs_for(A)
    k, s, eps, cap = prm
    t0 = time.perf_counter()
    G, Gt, _ = oracle.setup_full(A, k, s, eps, cap, threads=cores)
    t1 = time.perf_counter()
    r = oracle.pcg(A, G, Gt, b, tol=TOL, max_iters=20000)
    t2 = time.perf_counter()
    value = G.nnz / (t2 - t0)
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{label} ({A.n} rows): oracle set-up {t1 - t0:.2f} s ({cores} threads) + sequential "
                      f"oracle PCG {t2 - t1:.2f} s ({r.iters} iters)",
            "setup_s": t1 - t0, "pcg_s": t2 - t1, "pcg_iters": r.iters}


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch

    import afsai_inputs as ai
    from paper_2010_14175_b200.api import Context, DeviceCSR, Factor

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nx = args.nx
    if args.weak:
        # global problem: nx x nx x (nx * world); this rank owns rows of its slab
        wname = "M2"
        n_loc = nx * nx * nx
        Aglob = ai.poisson3d(nx, nx, nx * world) if world > 1 else ai.poisson3d(nx)
        row_begin = rank * n_loc
    else:
        # strong scaling: the BASELINE.json config, rank p owns rows [p n / N, (p+1) n / N)
        wname = args.workload
        Aglob = ai.CONFIGS[wname]["make"]()
        row_begin = rank * Aglob.n // world
        n_loc = (rank + 1) * Aglob.n // world - row_begin
    NSTEPS, S, EPS, CAP = workload_params(wname)
    b_glob, _ = ai.rhs_for(Aglob)
    dA = DeviceCSR.from_numpy(Aglob, row_begin=row_begin, n_rows=n_loc)
    b = torch.from_numpy(np.ascontiguousarray(b_glob[row_begin: row_begin + n_loc])).cuda()
    x = torch.empty_like(b)
    stream = torch.cuda.current_stream()
    ctx = Context(stream)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def step():
        F = Factor(ctx, dA, NSTEPS, S, EPS, CAP, precision=args.precision)
        _, rep = F.pcg(b, tol=TOL, max_iters=20000, x=x)
        return F, rep

    for _ in range(args.warmup):
        F, rep = step()
        F.close()
    torch.cuda.synchronize()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    ctx.set_timing(True)
    launches0 = ctx.launches()
    stats = reps = None
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        barrier()
        for k in range(args.steps):
            flush.zero_()                      # L2 flush between steps (outside the events)
            ev[k][0].record(stream)
            F, rep = step()
            ev[k][1].record(stream)
            if k == args.steps - 1:
                stats, reps = F.stats(), rep
            F.close()
        torch.cuda.synchronize()
        barrier()
    launches = ctx.launches() - launches0
    ktimes = ctx.kernel_times()
    ctx.set_timing(False)
    step_ms = [a.elapsed_time(b_) for a, b_ in ev]
    ms = float(np.mean(step_ms))
    nnzG = stats["nnz_G"]
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms, float(nnzG)], dtype=torch.float64, device="cuda")
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms_max, nnz_total = float(mx[0]), float(sm[1])
    else:
        ms_max, nnz_total = ms, float(nnzG)
    value = nnz_total / (ms_max * 1e-3)

    # ---- dominant kernel roofline
    total_kms = {k: v[1] for k, v in ktimes.items()}
    setup_ms = total_kms["setup_rows"] / args.steps
    iters = reps["iters"]
    n = dA.n_rows
    nnzA = dA.nnz
    nnzGt = stats["nnz_Gt"]
    # algorithmic bytes of the SpMVs: 12 B/nnz + 8 B/row (rowptr) + 8 B (y) + x gathered once
    bytes_G = 12 * nnzG + 8 * (n + 1) + 8 * n + 8 * n
    bytes_Gt = 12 * nnzGt + 8 * (n + 1) + 8 * n + 8 * n
    apply_bytes = bytes_G + bytes_Gt
    la_G, ms_G = ktimes["spmv_G"]
    la_T, ms_T = ktimes["spmv_Gt"]
    hbm_peak, peaks_src = 6450.0, "MEASURED_PEAKS.json hbm_gbs (measured)"
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak = float(mp["hbm_gbs"])
        sm_max = float(mp.get("sm_max_mhz", 1965.0))
    except Exception:
        hbm_peak, peaks_src, sm_max = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)", 1965.0
    # fp64 ALU peak from unit counts and clock: 148 SM x 64 DFMA/clk x 2 flop
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    fp64_peak_tf = nsm * 64 * 2 * sm_max * 1e6 / 1e12
    if args.precision == "fp32":   # the fp32 set-up runs on the FFMA pipe: 128 FMA/clk/SM
        fp64_peak_tf = nsm * 128 * 2 * sm_max * 1e6 / 1e12
    setup_flop = 2.0 * (stats["fma_border"] + stats["fma_backsub"] + stats["fma_grad"])
    dfma_probe_tf = ctx.dfma_peak()[0] / 1e12
    per_class = {k: {"launches": v[0] // args.steps, "ms_per_step": v[1] / args.steps} for k, v in ktimes.items()}
    solve_kernels_ms = (ms_G + ms_T + ktimes["spmv_A"][1] + ktimes["vector"][1]) / args.steps
    if setup_ms >= max(ms_G, ms_T) / args.steps:
        achieved = setup_flop / (setup_ms * 1e-3) / 1e12
        # DRAM bytes per launch of this kernel from the committed ncu --set full capture
        traffic = None
        tfile = f"r02_setup_traffic_{wname}{'' if args.precision == 'fp64' else '_fp32'}.json"
        try:
            traffic = json.load(open(os.path.join(ROOT, "profiles", tfile)))["dram_bytes_per_launch"]
        except Exception:
            pass
        from paper_2010_14175_b200.capi import afsai_setup_stats_t
        plan = afsai_setup_stats_t.PLANS.get(stats["plan"], "?")
        roof = {"kernel": f"afsai_setup_rows_{plan}_kernel (lanes/row {stats['lanes_per_row']}, "
                          f"table {stats['table_size']}, {stats['rows_per_cta']} rows/CTA)",
                "bound": "alu", "achieved": achieved,
                "peak": fp64_peak_tf, "unit": "TFLOP/s", "frac": achieved / fp64_peak_tf, "traffic": traffic,
                "traffic_unit": f"bytes per launch (dram read + write, ncu --set full, profiles/{tfile})",
                "peak_source": (f"{nsm} SM x {64 if args.precision == 'fp64' else 128} "
                                f"{'DFMA' if args.precision == 'fp64' else 'FFMA'}/clk x 2 x {sm_max:.0f} MHz "
                                f"(unit counts, B200_PROFILING.md; "
                                f"MEASURED_PEAKS.json has no fp64 entry); in-run DFMA probe "
                                f"{dfma_probe_tf:.1f} TF/s (afsai_probe_dfma_peak)"),
                "algorithmic_flop_per_launch": setup_flop, "avg_launch_ms": setup_ms}
    else:
        avg = ms_G / max(la_G, 1)
        achieved = bytes_G / (avg * 1e-3) / 1e9
        roof = {"kernel": "spmv (t = G r)", "bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": None, "peak_source": peaks_src,
                "algorithmic_bytes_per_launch": bytes_G, "avg_launch_ms": avg}
    # the other phase's roofline, for the record
    apply_gbs = (bytes_G * la_G / max(ms_G, 1e-9) + 0) / 1e6 if ms_G > 0 else None
    extra = {
        "setup_ms": float(stats["ms_total"]),
        "setup_phase_ms": {"rows_kernel": stats["ms_rows"], "assemble": stats["ms_assemble"],
                           "transpose": stats["ms_transpose"], "halo": stats["ms_halo"]},
        "setup_rows_kernel_ms": setup_ms,
        "setup_gnnz_per_s": nnzG / (stats["ms_total"] * 1e-3) if stats["ms_total"] > 0 else None,
        "setup_fp64_tflops": setup_flop / (setup_ms * 1e-3) / 1e12 if setup_ms > 0 else None,
        "setup_fp64_frac": (setup_flop / (setup_ms * 1e-3) / 1e12) / fp64_peak_tf if setup_ms > 0 else None,
        "pcg_iters": iters,
        "pcg_converged": bool(reps["converged"]),
        "pcg_true_rel_res": reps["true_rel_res"],
        "solve_ms": reps["ms_solve"],
        "solve_ms_per_iter": reps["ms_per_iter"],
        "apply_GB_per_s": (apply_bytes / ((ms_G / max(la_G, 1) + ms_T / max(la_T, 1)) * 1e-3) / 1e9)
        if la_G and la_T else None,
        "apply_hbm_frac": ((apply_bytes / ((ms_G / max(la_G, 1) + ms_T / max(la_T, 1)) * 1e-3) / 1e9) / hbm_peak)
        if la_G and la_T else None,
        "kernel_classes": per_class,
        "nnz_G_per_rank": nnzG,
        "stop_reasons": stats["rows_by_reason"],
        "table_size": stats["table_size"],
        "rows_per_cta": stats["rows_per_cta"],
        "solve_kernels_ms": solve_kernels_ms,
    }
    del apply_gbs

    # ---- e2e: the same metric through the C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        hA = DeviceCSR.from_numpy(Aglob, device="cpu", row_begin=row_begin, n_rows=n_loc, pin=True)
        hb = b.cpu().pin_memory()
        hx = torch.empty_like(hb).pin_memory()
        h2d = hA.rowptr.numel() * 8 + hA.col.numel() * 4 + hA.val.numel() * 8 + hb.numel() * 8
        d2h = hx.numel() * 8
        e_ms = []
        for k in range(args.e2e_runs + 1):   # one warm-up (host staging buffers, pinned paths), then runs
            flush.zero_()
            torch.cuda.synchronize()
            barrier()
            t0 = time.perf_counter()
            F = Factor(ctx, hA, NSTEPS, S, EPS, CAP, precision=args.precision)
            F.pcg(hb, tol=TOL, max_iters=20000, x=hx)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            F.close()
            e_ms.append((t1 - t0) * 1e3)
        em = float(np.median(e_ms[1:] or e_ms))
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([em], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            em = float(t[0])
        e2e = {"value": nnz_total / (em * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": em, "runs_ms": e_ms[1:],
               "timing": f"median of {len(e_ms) - 1} runs, host wall clock around afsai_setup(host A) + "
                         f"afsai_pcg(host b -> host x), max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(args)

    if rank == 0:
        clocks = clk.summary()
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
                "scaling": "weak" if args.weak else "strong",
                "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32 set-up, f64 solve",
                "data": "synthetic",
                "config": {"workload": (f"M2 weak scaling: 3D 7-point Poisson {nx}^3 per GPU (global "
                                        f"{nx}x{nx}x{nx * world}), aFSAI {NSTEPS}x{S}, PCG to {TOL}") if args.weak
                           else f"{wname}: {ai.CONFIGS[wname]['desc']}, PCG to {TOL}, rows split over {world} GPU(s)",
                           "global_rows": Aglob.n, "nnz_A": Aglob.nnz, "nsteps": NSTEPS, "s": S, "eps": EPS,
                           "max_row_nnz": CAP, "pcg_tol": TOL, "parallelism": f"rows{world}",
                           "setup_precision": args.precision,
                           "l2": "flushed (256 MiB write) between timed steps; A+G+scratch > 126 MB L2"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clocks, **extra}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
