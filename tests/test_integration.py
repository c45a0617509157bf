"""Drop-in routing of the reference package (CPU): runs only where the
reference is importable (the build container), in a subprocess so the
reference's exception classes are the ones our errors module re-exports."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parent.parent

SCRIPT = r'''
import sys
sys.path.insert(0, {ref!r}); sys.path.insert(0, {root!r})
import numpy as np
import pathfield, pathfield.divergence as D, pathfield.domain as Dom, pathfield.paths as Pth
import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import integration
from pathfield.errors import InvalidTargetError, PathfieldError
assert pf.InvalidTargetError is InvalidTargetError        # shared exception classes
done = integration.install(pathfield)
assert D.dv_field.__module__.startswith("paper_1708_02845_b200"), D.dv_field
assert Dom.dv_field is D.dv_field is pathfield.dv_field
assert Pth.triangle_descent is Dom.triangle_descent is pathfield.triangle_descent
assert Dom.sparsify is pf.sparsify
import pathfield.solvers as Sol
assert Sol.poisson_kernel is Dom.poisson_kernel is pathfield.poisson_kernel      # GPU P build
assert Sol.poisson_kernel.__module__.startswith("paper_1708_02845_b200")
from pathfield.mesh import generate_disk_mesh
from pathfield.laplacian import assemble_cotan
try:
    Dom.DomainContext(generate_disk_mesh(4)).kernel   # DomainContext.kernel -> device build
    raise SystemExit("silent fallback (poisson_kernel)")
except PathfieldError as e:
    assert "CUDA" in str(e) or "built" in str(e), e
dense = np.array([[0.5, 0.5, 0.0], [0.2, 0.3, 0.5], [0.0, 0.0, 1.0]])
pk = pathfield.solvers.PoissonKernel(dense, np.array([2]), 0.0, 0.0)
try:
    D.dv_field(pk, D.builtin_f("kl"), 7)
    raise SystemExit("no error")
except InvalidTargetError:
    pass
try:
    D.dv_field(pk, D.builtin_f("kl"), 0)     # no GPU here: must fail loudly, no CPU fallback
    raise SystemExit("silent fallback")
except PathfieldError as e:
    assert "CUDA" in str(e) or "built" in str(e), e
integration.uninstall()
assert D.dv_field.__module__ == "pathfield.divergence"
assert Sol.poisson_kernel.__module__ == "pathfield.solvers"
print("OK", sorted(done))
'''


@pytest.mark.skipif(not REF.exists(), reason="reference not present (GPU box)")
def test_install_routes_reference_bindings():
    code = SCRIPT.format(ref=str(REF), root=str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                       env={**os.environ, "CUDA_VISIBLE_DEVICES": ""}, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
