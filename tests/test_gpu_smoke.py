"""The driver's round-end smoke check (`__graft_entry__.smoke()`), run as a
GPU test so a change that breaks it shows up in `pytest -m gpu`."""

import sys
from pathlib import Path

import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


@pytest.mark.gpu
def test_graft_entry_smoke(gpu):
    import __graft_entry__

    __graft_entry__.smoke()
