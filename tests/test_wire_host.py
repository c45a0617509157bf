"""The digit generators of csrc/wire_core.cuh (compiled here for the host by
g++ — the same source the device formatter includes) against CPython's own
f"{v:.17g}" and repr(v), the reference's formatting (fileio.py:37-53)."""

import shutil
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_wire_core_host_build_matches_cpython():
    import wire_host_check
    assert wire_host_check.main(6000) == 0
