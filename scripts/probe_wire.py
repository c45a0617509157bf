"""Diagnostic: device timeline of the wire formatter on a 1M-value field."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch as t

from paper_1708_02845_b200 import fileio as F
from scripts.probe_e2e import timeline

n = 1_000_386
rng = np.random.default_rng(3)
vals = rng.random(n) * 10.0 ** rng.uniform(-3, 1, n)
dv = t.from_numpy(vals).cuda()
for kind in (0, 2):
    timeline(lambda: F.format_lines(dv, kind), f"format_lines kind {kind}", 1)
wide = np.concatenate([rng.integers(0, 2 ** 63, n // 2, dtype=np.int64).view(np.float64), vals[:n // 2]])
wide = wide[np.isfinite(wide)]
timeline(lambda: F.format_lines(t.from_numpy(wide).cuda(), 0), "format_lines kind 0, half extreme", 1)
