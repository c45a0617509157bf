"""The ctypes stub printed in INTEGRATION.md §3 works as written (GPU)."""

import re
from pathlib import Path

import numpy as np
import pytest

from tests.conftest import case, rel_close

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_integration_md_ctypes_stub():
    text = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    stub = [b for b in blocks if "ctypes.CDLL" in b][0]
    stub = stub.replace("/path/to/libpathfield_b200.so",
                        str(ROOT / "paper_1708_02845_b200" / "libpathfield_b200.so"))
    ns = {}
    exec(compile(stub, "INTEGRATION.md", "exec"), ns)
    c = case("c1")
    vals = ns["kl_field"](c.dense, c.boundary, c.target)
    ok, err = rel_close(vals, c["field/kl/0"], 1e-10)
    assert ok, err
