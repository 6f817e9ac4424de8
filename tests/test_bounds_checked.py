"""The bounds-checked build (build.py --debug: AFSAI_BOUNDS_CHECK, every row-pointer
lookup of the set-up kernels range-checked and reported) over every kernel plan and
the retry path (scripts/sanitize_case.py).  compute-sanitizer is closed on this GPU
pool (runs under it left GPUs needing a reset), so the library's own checks stand in
for memcheck; the paper's only hazard discussion is warp synchrony.
Builds the debug library (fp64 kernels only) if it is not in-tree.  Marked slow."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bounds_checked_build_all_plans():
    dbg = os.path.join(ROOT, "paper_2010_14175_b200", "lib", "libafsai_b200_dbg.so")
    if not os.path.exists(dbg):
        sys.path.insert(0, ROOT)
        from paper_2010_14175_b200 import build as b
        b.build(debug=True, fp32=False)
    env = dict(os.environ, AFSAI_DEBUG_LIB="1", AFSAI_CASES_FP64_ONLY="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py")], env=env,
                         capture_output=True, text=True, timeout=1800)
    log = out.stdout + out.stderr
    assert out.returncode == 0, log[-3000:]
    assert "sanitize cases ok" in out.stdout
    assert "afsai bounds" not in log, [ln for ln in log.splitlines() if "afsai bounds" in ln][:10]
