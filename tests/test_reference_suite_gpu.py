"""The reference's own test-suite as the drop-in regression on the B200.

`tools/install_reference.sh` installs the unmodified reference package into
baseline/_ref (git-ignored, shipped with the snapshot) with its 224 tests
beside it.  This test runs that suite in a subprocess with
``-p paper_1708_02845_b200.pytest_plugin``, which routes every hot-path
binding (dv_field, dv_at, dv_pair, sparsify, dv_pair_sparse(_stats),
triangle_descent, edge_descent, find_local_minima, path_hausdorff,
poisson_kernel, the wire formats — integration.SITES) to the sm_100a
kernels before the suite imports them: DomainContext, the service and the
CLI run unchanged on the GPU path.  Tests that cannot hold under the drop-in
are listed in EXPECTED_DIFFERENT with the reason.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
SUITE = REF / "ref_suite"

# test node id -> why the drop-in legitimately differs
EXPECTED_DIFFERENT: dict = {}


@pytest.mark.skipif(not (REF / "pathfield").is_dir() or not (SUITE / "tests").is_dir(),
                    reason="reference not installed (tools/install_reference.sh)")
def test_reference_suite_through_install():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT)])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "paper_1708_02845_b200.pytest_plugin",
           "-p", "no:cacheprovider", "-rf", "tests"]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "reference_suite_gpu.log").write_text(out)
    assert "routed to the B200 path" in out, out[-3000:]
    failed = [ln.split(" ", 2)[1] for ln in out.splitlines() if ln.startswith("FAILED ")]
    unexpected = [f for f in failed if f not in EXPECTED_DIFFERENT]
    assert not unexpected, "\n".join(unexpected) + "\n" + out[-6000:]
    assert " passed" in out.splitlines()[-1], out[-3000:]
