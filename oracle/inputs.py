"""Test-input builders: the reference's Poisson kernel P (SuperLU), restated.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Produces the same Poisson
kernel P as the reference's preprocessing so that the GPU box (which has no
/root/reference) can rebuild real inputs for parity checks; the golden
fixtures carry sha256 digests of the reference's own arrays so a test can
tell whether the rebuilt input is bitwise the reference's.  The meshes
themselves come from workloads/meshes.py (re-exported here).

Restated from /root/reference/pkg/src/pathfield:
  laplacian.py:91-134 assemble_cotan; laplacian.py:29-61 InteriorFactor;
  solvers.py:278-303 poisson_kernel.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import splu

from workloads.meshes import (BUILDERS, SPECS, Mesh, build, c4_targets, c5_jobs,  # noqa: F401
                              default_endpoints, disk_mesh, holes_mesh, make_mesh,
                              rectangle_mesh, sha, square_hole_mesh, synthetic_kernel)


def cotan_laplacian(mesh: Mesh) -> sp.csr_matrix:
    """laplacian.py:91-134 (same COO construction, so identical duplicate sums)."""
    v, t, n = mesh.vertices, mesh.triangles, mesh.n
    rows, cols, vals = [], [], []
    for c0, c1, c2 in ((0, 1, 2), (1, 2, 0), (2, 0, 1)):
        pk, pi, pj = v[t[:, c0]], v[t[:, c1]], v[t[:, c2]]
        u, w = pi - pk, pj - pk
        cross = u[:, 0] * w[:, 1] - u[:, 1] * w[:, 0]
        cot = (u * w).sum(axis=1) / np.abs(cross)
        half = 0.5 * cot
        rows += [t[:, c1], t[:, c2]]
        cols += [t[:, c2], t[:, c1]]
        vals += [half, half]
    off = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                        shape=(n, n)).tocsr()
    diag = -np.asarray(off.sum(axis=1)).ravel()
    return (off + sp.diags(diag)).tocsr()


def poisson_kernel(mesh: Mesh, col_chunk: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """solvers.py:278-303: P_IB = -Lc_II^{-1} Lc_IB; boundary rows are indicators.

    Returns (dense, boundary).  ``col_chunk`` solves in column chunks (needed
    at 1M vertices; not bitwise equal to the all-columns solve).
    """
    lc = cotan_laplacian(mesh)
    bmask = mesh.boundary_mask()
    boundary = np.flatnonzero(bmask)
    interior = np.flatnonzero(~bmask)
    n, k = mesh.n, boundary.size
    dense = np.zeros((n, k))
    dense[boundary, np.arange(k)] = 1.0
    if interior.size:
        lc_i = lc[interior]
        lc_ii = lc_i[:, interior]
        lc_ib = lc_i[:, boundary]
        lu = splu((-lc_ii).tocsc())
        if col_chunk is None:
            p_ib = lu.solve(np.asarray(lc_ib.toarray(), dtype=float))
        else:
            p_ib = np.empty((interior.size, k))
            for a in range(0, k, col_chunk):
                b = min(k, a + col_chunk)
                p_ib[:, a:b] = lu.solve(np.asarray(lc_ib[:, a:b].toarray(), dtype=float))
        tiny = (p_ib > -1e-12) & (p_ib < 0.0)
        p_ib[tiny] = 0.0
        dense[interior] = p_ib
    return dense, boundary


def _solve_cols(args):
    """Worker: factor -L_II once, solve a column range of -L_IB into shared memory."""
    shm_name, shape, interior_size, cols, lc_ii, lc_ib = args
    from multiprocessing import shared_memory
    try:  # one BLAS thread per worker: the workers are the parallelism
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    shm = shared_memory.SharedMemory(name=shm_name)
    try:
        out = np.ndarray(shape, dtype=np.float64, buffer=shm.buf)
        lu = splu((-lc_ii).tocsc())
        a, b = cols
        for c0 in range(a, b, 64):
            c1 = min(b, c0 + 64)
            x = lu.solve(np.asarray(lc_ib[:, c0:c1].toarray(), dtype=float))
            tiny = (x > -1e-12) & (x < 0.0)
            x[tiny] = 0.0
            out[:, c0:c1] = x
    finally:
        shm.close()
    return cols


def poisson_kernel_parallel(mesh: Mesh, workers: int = 8):
    """poisson_kernel for large meshes: `workers` processes each factor -L_II
    (SuperLU, as solvers.py:278-303) and solve a column range in 64-column
    chunks into shared memory.  Column-chunked solves differ from the
    all-columns solve by ~1e-17 absolute; there is no reference
    P at this size to compare against, so the returned P is the shared input."""
    from concurrent.futures import ProcessPoolExecutor
    from multiprocessing import get_context, shared_memory
    lc = cotan_laplacian(mesh)
    bmask = mesh.boundary_mask()
    boundary = np.flatnonzero(bmask)
    interior = np.flatnonzero(~bmask)
    n, k = mesh.n, boundary.size
    lc_i = lc[interior]
    lc_ii = lc_i[:, interior].tocsr()
    lc_ib = lc_i[:, boundary].tocsc()
    shm = shared_memory.SharedMemory(create=True, size=max(8, interior.size * k * 8))
    try:
        shape = (interior.size, k)
        bounds = np.linspace(0, k, workers + 1).astype(int)
        jobs = [(shm.name, shape, interior.size, (int(a), int(b)), lc_ii, lc_ib)
                for a, b in zip(bounds[:-1], bounds[1:]) if b > a]
        with ProcessPoolExecutor(len(jobs), mp_context=get_context("fork")) as ex:
            list(ex.map(_solve_cols, jobs))
        p_ib = np.ndarray(shape, dtype=np.float64, buffer=shm.buf)
        dense = np.zeros((n, k))
        dense[boundary, np.arange(k)] = 1.0
        dense[interior] = p_ib
    finally:
        shm.close()
        shm.unlink()
    return dense, boundary
