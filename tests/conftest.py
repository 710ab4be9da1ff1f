import json
import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libqvb200.so")


def _load(name):
    path = GOLDEN / name
    if not path.exists():
        pytest.skip(f"{name} missing; run tests/golden/make_golden.py")
    return json.loads(path.read_text())


@pytest.fixture(scope="session")
def golden_small():
    return _load("golden_small.json")


@pytest.fixture(scope="session")
def golden_large():
    return _load("golden_large.json")


@pytest.fixture(scope="session")
def golden_big():
    """Benchmark-size goldens made by the reference's own kernels
    (tests/golden/make_golden_big.py): qcl20 (config 3), qcl28 (config 4),
    qcl30c5 (config 5's geometry at the reference's 30-qubit cap)."""
    out = {}
    for name in ("qcl20", "qcl28", "qcl30c5", "mcvqe16"):
        path = GOLDEN / f"golden_big_{name}.json"
        if path.exists():
            out[name] = json.loads(path.read_text())
    return out


@pytest.fixture(scope="session")
def gpu():
    """Skip-free GPU gate: a -m gpu test must fail loudly, not skip, when the
    native library or the device is missing."""
    from paper_2406_03466_b200 import native
    if native.device_count() < 1:
        raise RuntimeError("no CUDA device visible to libqvb200.so")
    return native
