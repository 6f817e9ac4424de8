"""compute-sanitizer memcheck / racecheck / synccheck over every kernel plan on small
inputs (scripts/sanitize_case.py).  The paper's only hazard discussion is warp
synchrony; the set-up kernels rely on converged-warp shuffles, ballots
and shared-memory hand-offs, which these tools check.  Marked slow (minutes)."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(tool):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.fail("compute-sanitizer not found")
    # only this library's kernels are checked (torch's own kernels are not the subject)
    # every kernel of the library lives in namespace afsai (mangled names contain it)
    cmd = [cs, "--tool", tool, "--kernel-name", "kns=afsai", "--error-exitcode", "99", sys.executable,
           os.path.join(ROOT, "scripts", "sanitize_case.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=3000)
    tail = (out.stdout + out.stderr)[-4000:]
    assert out.returncode == 0, tail
    assert "sanitize cases ok" in out.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in out.stdout + out.stderr, tail
