"""The C-ABI library loads (no GPU needed) and exports every function include/*.h declares."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    names = set()
    for h in ("zp_host.h", "zp_runtime.h", "zp_kernels.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(zp_[a-z0-9_]+)\s*\(", src, re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    from paper_2408_12596_b200 import _lib
    names = declared()
    assert len(names) > 40
    missing = [n for n in sorted(names) if not hasattr(_lib.lib, n)]
    assert not missing, missing


def test_oracle_library_exports_host_abi():
    import oracle
    if not oracle.available() and not oracle.build_reference():
        pytest.skip("reference not built")
    import ctypes
    lib = ctypes.CDLL(oracle.REF_LIB)
    src = open(os.path.join(ROOT, "include", "zp_host.h")).read()
    for n in re.findall(r"\b(zp_[a-z0-9_]+)\s*\(", src):
        assert hasattr(lib, "zpref_" + n[3:]), n


def test_sm100a_cubin_contains_tcgen05_and_tma():
    """The shipped kernels are sm_100a tcgen05/TMA code (SASS UTCHMMA / UTMALDG / LDTM)."""
    import shutil
    import subprocess
    lib = os.path.join(ROOT, "paper_2408_12596_b200", "lib", "libzp.so")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([exe, "-sass", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run([exe, "-lelf", lib], capture_output=True, text=True).stdout
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnem in sass, mnem
