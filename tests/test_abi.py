"""The C-ABI library loads and exports every symbol include/aqua.h declares
(no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^AQUA_API\s+[\w\s\*]+?\b(aqua_\w+)\(", txt, flags=re.M)))


def test_header_symbols_exported():
    from paper_2407_21255_b200 import aqua
    decl = _declared("aqua.h")
    assert len(decl) >= 20
    assert sorted(aqua.SYMBOLS) == decl
    lib = ctypes.CDLL(aqua.LIB_PATH)
    for name in decl:
        assert hasattr(lib, name), name


def test_cfs_header_symbols_exported():
    from paper_2407_21255_b200 import aqua, cfs
    decl = _declared("aqua_cfs.h")
    assert sorted(cfs.SYMBOLS) == decl
    lib = ctypes.CDLL(aqua.LIB_PATH)
    for name in decl:
        assert hasattr(lib, name), name


def test_version_and_strerror():
    from paper_2407_21255_b200 import aqua
    assert "sm_100a" in aqua.version()
    assert aqua.lib.aqua_strerror(aqua.E_NOSPACE).decode().startswith("no swap space")


def test_sm100a_cubin_and_bulk_copy_in_sass():
    """The kernels are compiled for sm_100a and the TMA path uses bulk copies
    (UBLKCP) -- checked with cuobjdump, no GPU needed."""
    import shutil
    import subprocess
    import pytest
    from paper_2407_21255_b200 import aqua
    cob = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cob):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cob, "-sass", aqua.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UBLKCP" in out
    assert "swap_tma_kernel" in out and "swap_ldst_kernel" in out
