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


def test_struct_layouts_match_header(lib, tmp_path):
    """Every struct of include/afsai.h has the ctypes mirror's size and field offsets
    (measured by a C program compiled against the header)."""
    import subprocess
    from paper_2010_14175_b200 import capi
    structs = {"afsai_csr_t": capi.afsai_csr_t, "afsai_params_t": capi.afsai_params_t,
               "afsai_status_t": capi.afsai_status_t, "afsai_setup_stats_t": capi.afsai_setup_stats_t,
               "afsai_pcg_report_t": capi.afsai_pcg_report_t}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "afsai.h"', "int main(void) {"]
    for name, cls in structs.items():
        lines.append(f'printf("{name} size %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    got = dict(((a, b), int(c)) for a, b, c in (ln.split() for ln in subprocess.check_output([str(exe)], text=True).splitlines()))
    for name, cls in structs.items():
        assert got[(name, "size")] == ctypes.sizeof(cls), name
        for f, _ in cls._fields_:
            assert got[(name, f)] == getattr(cls, f).offset, (name, f)


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
