"""The C-ABI boundary: the library loads, exports every entry point declared in
include/hecsolve_c.h, reports errors through status codes, and -- without a
GPU -- refuses device work loudly instead of falling back to the CPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hecsolve_c.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hec_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_exported(H):
    names = declared_functions()
    assert len(names) >= 45
    lib = ctypes.CDLL(H.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding covers all of them
    from paper_1606_00541_b200 import _lib
    assert set(names) <= set(_lib.EXPORTED), set(names) - set(_lib.EXPORTED)


def test_exports_are_plain_c_symbols(H):
    out = subprocess.run(["nm", "-D", "--defined-only", H.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    for n in declared_functions():
        assert n in exported, n  # unmangled extern "C"


def test_library_is_sm100a(H):
    out = subprocess.run(["cuobjdump", "--list-elf", H.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_codes_and_last_error(H):
    from paper_1606_00541_b200 import _lib as L
    h = ctypes.c_void_p()
    rc = L.lib.hec_gen_poisson7(0, 1, 1, ctypes.byref(h))
    assert rc == L.HEC_EINVAL
    assert b"grid dimensions" in L.lib.hec_last_error()
    rows = (ctypes.c_int * 1)(5)
    cols = (ctypes.c_int * 1)(0)
    vals = (ctypes.c_double * 1)(1.0)
    rc = L.lib.hec_csr_from_triples(2, 2, 1, rows, cols, vals, ctypes.byref(h))
    assert rc == L.HEC_ERANGE
    assert L.lib.hec_version().startswith(b"hecsolve-b200")


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU behaviour")
def test_device_path_has_no_cpu_fallback(H):
    assert H.device_available() is False
    l3 = H.csr_from_triples(3, 3, [(0, 0, 2.0), (1, 0, 1.0), (1, 1, 3.0), (2, 1, 2.0), (2, 2, 4.0)])
    p = H.prepare_lower(l3)  # host setup works without a GPU
    with pytest.raises(H.HecError, match="no CUDA device"):
        H.solve(p, [2.0, 4.0, 6.0])
    with pytest.raises(H.HecError):
        H.DeviceTri.create(p)
    m = H.build_preconditioner(H.gen_poisson7(4, 4, 4), "bilu0", 2, 0)
    with pytest.raises(H.HecError):
        H.apply(m, np.ones(64))
