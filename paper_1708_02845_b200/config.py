"""Runtime settings, mirroring ``pathfield/config.py:16-28``.

Only ``threshold`` (sparsify default, None -> 1/sqrt(n)) and
``step_cap_factor`` (tracer cap = factor * n) reach the hot path; the other
keys are kept so a reference ``Settings`` and this one are interchangeable.
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass


@dataclass(frozen=True)
class Settings:
    dense_budget: int = 4000
    threshold: float | None = None
    step_cap_factor: int = 50
    contour_levels: int = 10
    residual_warn: float = 1e-6
    trials: int = 11

    def replace(self, **kwargs) -> "Settings":
        updates = {k: v for k, v in kwargs.items() if v is not None}
        return dataclasses.replace(self, **updates)


DEFAULTS = Settings()
