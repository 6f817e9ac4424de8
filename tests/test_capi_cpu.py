"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/afsai.h declares; the binding mirrors the header's structs.
No compute calls (no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "afsai.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(afsai_[a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2010_14175_b200 import build
    build.build()
    from paper_2010_14175_b200 import capi
    return capi.load_library()


def test_header_declares_the_boundary():
    names = header_functions()
    for must in ["afsai_setup", "afsai_apply", "afsai_pcg", "afsai_ctx_create", "afsai_factor_copy"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2010_14175_b200 import capi
    names = header_functions()
    assert sorted(capi.EXPORTS) == names
    for n in names:
        assert hasattr(lib, n), n


def test_struct_layouts_match_header(lib):
    from paper_2010_14175_b200 import capi
    # sizes implied by the header (x86-64 SysV alignment)
    assert ctypes.sizeof(capi.afsai_csr_t) == 7 * 8
    assert ctypes.sizeof(capi.afsai_params_t) == 24
    assert ctypes.sizeof(capi.afsai_status_t) == 4 + 4 + 8 + 4 + 160 + 4
    assert ctypes.sizeof(capi.afsai_pcg_report_t) == 8 + 4 * 8


def test_strerror_and_version(lib):
    from paper_2010_14175_b200 import capi
    assert b"sm_100a" in lib.afsai_version()
    assert lib.afsai_strerror(capi.AFSAI_ENOTSPD).startswith(b"matrix is not SPD")


def test_kernels_are_sm100a(lib):
    """The fatbin holds sm_100a SASS (cuobjdump), not PTX-only or another arch."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump missing")
    from paper_2010_14175_b200 import capi
    out = subprocess.run(["cuobjdump", "--list-elf", capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle (task rule 3)."""
    pkg = os.path.join(ROOT, "paper_2010_14175_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "liboracle" not in txt and "afsai_oracle" not in txt, f
