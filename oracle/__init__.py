"""CPU oracle for the divergence-distance hot path — TEST INFRASTRUCTURE ONLY.

This package restates the reference's algorithms (``pathfield``, pure
Python/numpy, /root/reference/pkg/src/pathfield) in plain numpy so that the
device path can be checked where the reference itself is not available (the
GPU box has no /root/reference).  Every function cites the reference
file:line it follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``cpu_baseline`` / ``--impl reference``) may import it, and only as the
checker or the timed CPU baseline.  The product package
``paper_1708_02845_b200`` never imports it: it has no CPU fallback.

Pinning: the restatement is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``; see
``tests/test_oracle.py``).  Where the reference's arithmetic lives in
numpy/scipy/OpenBLAS (unpinned by the reference's own tests),
parity is anchored on those goldens.

Modules
  inputs      mesh generators + cotan Laplacian + Poisson kernel (the
              reference's preprocessing, mesh.py / laplacian.py / solvers.py)
  divergence  dv_field / dv_at / dv_pair / sparsify / dv_pair_sparse
  tracer      triangle_descent scalar restatement (paths.py:101-307)
"""
