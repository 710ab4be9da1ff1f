"""The C-ABI library loads and exports every symbol include/qvb200.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import re
from pathlib import Path

from paper_2406_03466_b200 import build as qbuild
from paper_2406_03466_b200 import native

HEADER = Path(__file__).resolve().parent.parent / "include" / "qvb200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(qv_[a-z_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    qbuild.build_product()
    lib = ctypes.CDLL(str(native.LIB_PATH))
    names = declared_functions()
    assert {"qv_create", "qv_execute", "qv_destroy", "qv_last_error"} <= set(names)
    for name in names:
        assert hasattr(lib, name), name
    assert set(native.EXPORTS) == set(names)


def test_version_and_device_probe_without_gpu():
    lib = native.load_library()
    assert lib.qv_version().startswith(b"qvb200")
    if lib.qv_device_count() == 0:
        h = ctypes.c_void_p()
        assert lib.qv_create(0, 0, 0, ctypes.byref(h)) == native.QV_ERR_CUDA


def test_output_size_contract():
    lib = native.load_library()
    c = native.QvCircuits()
    c.n_qubits, c.n_circuits = 5, 3
    r = native.QvResults()
    r.kind = native.QV_OUT_SUPPORT
    r.support_count = 7
    assert lib.qv_output_size(ctypes.byref(c), ctypes.byref(r)) == 3 * 8
    r.kind = native.QV_OUT_FULL
    assert lib.qv_output_size(ctypes.byref(c), ctypes.byref(r)) == 3 * 32
    r.kind = native.QV_OUT_JS
    assert lib.qv_output_size(ctypes.byref(c), ctypes.byref(r)) == 3


def test_product_library_is_sm100a():
    """The product .so carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([tool, "--list-elf", str(native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
