#!/bin/bash
# Install the unmodified reference package (pathfield, /root/reference/pkg) into
# baseline/_ref (git-ignored; it travels to the GPU box with the snapshot) and
# put its own test-suite beside it as baseline/_ref/ref_suite/tests, so that
# tests/test_reference_suite_gpu.py can run the reference's 224 tests through
# integration.install() on the B200.  The build writes into its source tree,
# so it installs from a copy under /tmp.  Run from the repo root.
set -euo pipefail
SRC=${1:-/root/reference/pkg}
rm -rf /tmp/pathfield_src && cp -r "$SRC" /tmp/pathfield_src
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target baseline/_ref --no-deps --upgrade /tmp/pathfield_src
rm -rf baseline/_ref/ref_suite && mkdir -p baseline/_ref/ref_suite
cp -r /tmp/pathfield_src/tests baseline/_ref/ref_suite/tests
# the suite imports `tests.conftest` (test_cli.py): make it a package
touch baseline/_ref/ref_suite/tests/__init__.py
echo "reference installed: $(ls baseline/_ref)"
