"""Shared fixtures: golden cases (reference outputs) and their rebuilt inputs.

`-m gpu` tests run the CUDA path through the C ABI on a B200 and compare with
the goldens / the CPU oracle; everything else runs on CPU.
"""

from __future__ import annotations

import functools
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"
CASES = ("disk8", "c1", "corridor50", "disk40", "holes_fine")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: larger sizes")


class Case:
    def __init__(self, name: str):
        self.name = name
        self.z = np.load(GOLDEN / f"{name}.npz")
        self.meta = json.loads(str(self.z["meta"]))
        self.n, self.k = self.meta["n"], self.meta["k"]
        self.targets = self.meta["targets"]
        self.source, self.target = self.meta["source"], self.meta["target"]

    def __getitem__(self, key):
        return self.z[key]

    def keys(self):
        return self.z.files

    @functools.cached_property
    def mesh(self):
        from oracle import inputs as I
        return I.build(self.meta["spec"])

    @functools.cached_property
    def P(self):
        from oracle import inputs as I
        if "P" in self.z.files:
            return self.z["P"], self.z["boundary"]
        return I.poisson_kernel(self.mesh)

    @property
    def dense(self):
        return self.P[0]

    @property
    def boundary(self):
        return self.P[1]

    def input_matches_reference(self) -> bool:
        from oracle import inputs as I
        return I.sha(self.dense) == self.meta["sha_P"]

    def path(self, gname: str, i: int) -> dict:
        pre = f"path/{gname}/{i}/"
        return {key[len(pre):]: self.z[key] for key in self.z.files if key.startswith(pre)}


@functools.lru_cache(maxsize=None)
def case(name: str) -> Case:
    return Case(name)


@pytest.fixture(params=CASES)
def golden_case(request):
    return case(request.param)


def rel_close(a, b, rtol):
    """Element-wise |a-b| <= rtol*|b| (exact where b is 0 or inf)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    same = (a == b)
    with np.errstate(invalid="ignore"):
        err = np.abs(a - b)
    ok = same | (err <= rtol * np.abs(b))
    return bool(ok.all()), (float(np.max(np.where(same, 0.0, err / np.maximum(np.abs(b), 1e-300))))
                            if a.size else 0.0)


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device (run with -m gpu on a B200)")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
