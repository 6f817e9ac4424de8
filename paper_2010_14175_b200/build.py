"""Build libafsai_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Each .cu under csrc/ is compiled separately (setup_kernel.cu with -fmad=false so
the only fused multiply-adds are the explicit fma() of the arithmetic contract,
DESIGN.md §3.1), then linked with NCCL into lib/libafsai_b200.so.
"""
from __future__ import annotations

import glob
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
OBJDIR = os.path.join(HERE, "build_obj")
LIB = os.path.join(LIBDIR, "libafsai_b200.so")
# --debug: bounds-checked variant (AFSAI_BOUNDS_CHECK: every row-pointer lookup of
# the set-up kernels traps with the offending index), loaded when AFSAI_DEBUG_LIB=1
OBJDIR_DBG = os.path.join(HERE, "build_obj_dbg")
LIB_DBG = os.path.join(LIBDIR, "libafsai_b200_dbg.so")
ROOT = os.path.dirname(HERE)

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dirs():
    try:
        import nvidia.nccl as nc  # the NCCL torch loads
        base = list(nc.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(lib, "libnccl.so.2")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


_CONTRACT_HDR = re.compile(r'#include\s+"setup_\w*\.cuh"')


def _flags_for(src: str):
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
             "-Xptxas", "-v"] + ARCH
    # Every unit that includes set-up device code (setup_*.cuh) compiles with
    # -fmad=false, so the only fused multiply-adds are the explicit fma() of the
    # arithmetic contract.  The decision is made from the file's
    # includes, not its name; setup_common.cuh #errors without AFSAI_FMAD_OFF.
    if _is_contract(src):
        flags += ["-fmad=false", "-DAFSAI_FMAD_OFF"]
    return flags


def _is_contract(src: str) -> bool:
    with open(src) as f:
        return bool(_CONTRACT_HDR.search(f.read()))


def build(force: bool = False, verbose: bool = False, debug: bool = False, variant: str = "",
          defines: tuple = (), fp32: bool = True) -> str:
    """variant + defines: an A/B build (extra -D flags) into build_obj_<variant>/ and
    lib/libafsai_b200_<variant>.so, loaded with AFSAI_LIB=<path>."""
    objdir = OBJDIR_DBG if debug else OBJDIR
    lib_out = LIB_DBG if debug else LIB
    extra = ["-DAFSAI_BOUNDS_CHECK"] if debug else []
    if not fp32:
        extra = extra + ["-DAFSAI_NO_FP32"]
    if variant:
        objdir = os.path.join("/tmp", "afsai_build_obj_" + variant)  # outside the repo (gpurun snapshot size)
        lib_out = os.path.join(LIBDIR, f"libafsai_b200_{variant}.so")
        extra = extra + ["-D" + d for d in defines]
    os.makedirs(LIBDIR, exist_ok=True)
    os.makedirs(objdir, exist_ok=True)
    inc, libdir = _nccl_dirs()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
            [os.path.join(ROOT, "include", "afsai.h")])
    newest_hdr = max(os.path.getmtime(h) for h in hdrs)
    objs, todo = [], []
    for s in srcs:
        # set-up units twice: fp64 (afsai::dp) and fp32 (afsai::sp, -DAFSAI_SETUP_FP32)
        variants = [("", [])] + ([(".f32", ["-DAFSAI_SETUP_FP32"])] if fp32 and _is_contract(s) else [])
        for suffix, vflags in variants:
            o = os.path.join(objdir, os.path.basename(s) + suffix + ".o")
            objs.append(o)
            if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), newest_hdr):
                todo.append((s, o, vflags))

    def compile_one(so):
        s, o, vflags = so
        cmd = ([NVCC, "-c", s, "-o", o, "-I", inc, "-I", os.path.join(ROOT, "include")] + _flags_for(s) + extra +
               vflags)
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(o[:-2] + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
        return s, r

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        for s, r in ex.map(compile_one, todo):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {s}")
            if verbose:
                sys.stderr.write(r.stderr)
    if force or not os.path.exists(lib_out) or os.path.getmtime(lib_out) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC, "-shared", "-o", lib_out] + objs + ARCH + [
            "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}", "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return lib_out


if __name__ == "__main__":
    var = next((x.split("=", 1)[1] for x in sys.argv if x.startswith("--variant=")), "")
    defs = tuple(x[2:] for x in sys.argv if x.startswith("-D"))
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv,
                variant=var, defines=defs, fp32="--no-fp32" not in sys.argv))
