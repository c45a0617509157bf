"""K11 — the Poisson kernel P on the device.

CPU (no GPU): the host nested-dissection plan (nd_plan.cpp) executed by the
numpy multifrontal simulation (tests/mf_sim.py) reproduces the reference's
P (solvers.py:278-303, rebuilt bitwise by oracle/inputs.py and checked
against the golden sha256) to rounding level, componentwise.

GPU: the device Laplacian is bitwise the reference's (laplacian.py:91-134);
the device P matches the reference P componentwise (tails included) and is
deterministic; the hot path on the device-built P reproduces the golden
fields; residual / row_sum_error are at rounding level.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import inputs as I
from tests import mf_sim
from tests.conftest import CASES, case, rel_close

# Componentwise bar for P (entries above the FP64 normal range floor): the
# M-matrix structure makes every solve term non-negative, so the device P and
# SuperLU's differ by a few hundred ulps at most, tails included.
P_RTOL = 1e-11
P_FLOOR = 1e-290


def _pcompare(P, ref, interior):
    a, b = P[interior], ref[interior]
    zero_ok = bool(np.array_equal(a == 0.0, b == 0.0))
    big = b > P_FLOOR
    rel = np.abs(a[big] - b[big]) / b[big]
    small_abs = float(np.abs(a[~big] - b[~big]).max()) if (~big).any() else 0.0
    return zero_ok, float(rel.max()) if rel.size else 0.0, small_abs


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("leaf", [8, 64])
def test_plan_simulation_matches_reference(name, leaf):
    from paper_1708_02845_b200.laplacian import NdPlan, mesh_topology
    c = case(name)
    assert c.input_matches_reference()
    m = c.mesh
    nb_ptr, nb_idx, isb = mesh_topology(m)
    plan = NdPlan(m.vertices, nb_ptr, nb_idx, isb, leaf=leaf)
    assert plan.k == c.k and plan.n == c.n
    # every interior vertex is placed exactly once, post-order
    assert np.array_equal(np.sort(plan.perm_orig), np.flatnonzero(isb == 0))
    assert np.all(plan.parent[plan.parent >= 0] > np.flatnonzero(plan.parent >= 0))
    lc = I.cotan_laplacian(m)
    off, diag = mf_sim.laplacian_parts(lc, nb_ptr, nb_idx)
    F = mf_sim.factor(plan, off, diag)
    P = mf_sim.solve(plan, F, off, plan.k)
    zero_ok, rel, small = _pcompare(P, c.dense, np.flatnonzero(isb == 0))
    assert zero_ok
    assert rel < P_RTOL, rel
    assert small < 1e-300


@pytest.mark.parametrize("name", CASES)
def test_vertex_neighbors_match_mesh_topology(name):
    """pf_vertex_neighbors (C++) == the sorted neighbour lists of mesh.py:151."""
    from paper_1708_02845_b200.laplacian import vertex_neighbors
    from paper_1708_02845_b200.mesh import topology
    m = case(name).mesh
    ref = topology(m.triangles, m.n)
    nb_ptr, nb_idx = vertex_neighbors(m.triangles, m.n)
    assert np.array_equal(nb_ptr, ref[2]) and np.array_equal(nb_idx, ref[3])


def test_plan_tiles_cover_rhs():
    """The forward visits exactly the tiles reachable from a boundary column."""
    from paper_1708_02845_b200.laplacian import NdPlan
    c = case("holes_fine")
    plan = NdPlan.from_mesh(c.mesh, leaf=16)
    for s in range(plan.nodes):
        own = set((plan.b_col[plan.b_ptr[s]:plan.b_ptr[s + 1]] // plan.tile).tolist())
        kids = plan.ch_idx[plan.ch_ptr[s]:plan.ch_ptr[s + 1]]
        for ch in kids:
            own |= set(plan.act_tile[plan.act_ptr[ch]:plan.act_ptr[ch + 1]].tolist())
        assert own == set(plan.act_tile[plan.act_ptr[s]:plan.act_ptr[s + 1]].tolist())
    root_tiles = plan.act_tile[plan.act_ptr[plan.nodes - 1]:plan.act_ptr[plan.nodes]]
    assert len(root_tiles) <= plan.ntiles


@pytest.mark.parametrize("name", ["c1", "holes_fine"])
@pytest.mark.parametrize("parts", [3, 8])
def test_slab_needs_cover_the_slab(name, parts):
    """laplacian.slab_needs: a backward over only the needed fronts (numpy
    simulation; unneeded rows NaN) reproduces the slab rows and their 1-ring
    exactly; the row offsets put slab rows first and scratch rows after."""
    from paper_1708_02845_b200.laplacian import NdPlan, mesh_topology, slab_needs
    c = case(name)
    m = c.mesh
    nb_ptr, nb_idx, isb = mesh_topology(m)
    plan = NdPlan(m.vertices, nb_ptr, nb_idx, isb, leaf=16)
    off, diag = mf_sim.laplacian_parts(I.cotan_laplacian(m), nb_ptr, nb_idx)
    F = mf_sim.factor(plan, off, diag)
    full = mf_sim.solve(plan, F, off, plan.k)
    bounds = np.linspace(0, plan.n, parts + 1).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        need, rowoff, extra = slab_needs(plan, nb_ptr, nb_idx, isb, int(a), int(b - a), 7)
        got = mf_sim.solve(plan, F, off, plan.k, need=need)
        rows = np.arange(a, b)
        inner = rows[isb[rows] == 0]
        lo, hi = nb_ptr[inner], nb_ptr[inner + 1]
        ring = np.unique(np.concatenate([nb_idx[x:y] for x, y in zip(lo, hi)] + [inner]))
        ring = ring[isb[ring] == 0]
        assert np.array_equal(got[ring], full[ring])            # no NaN: every row computed
        assert np.array_equal(rowoff[inner], (inner - a) * 7)   # slab rows first
        assert np.all(rowoff[ring] >= 0)
        scratch = rowoff[(rowoff >= 0) & ((np.arange(plan.n) < a) | (np.arange(plan.n) >= b))]
        assert scratch.size == extra and np.array_equal(np.sort(scratch) // 7,
                                                        (b - a) + np.arange(extra))


def test_plan_rejects_bad_arguments():
    from paper_1708_02845_b200 import _native as nat
    from paper_1708_02845_b200.errors import NativeError
    from paper_1708_02845_b200.laplacian import NdPlan
    with pytest.raises(NativeError):
        NdPlan(np.zeros((3, 2)), np.zeros(4, np.int64), np.zeros(0, np.int64),
               np.zeros(3, np.uint8), leaf=0)
    assert nat.load().pf_nd_plan_array(None, b"c0", None) == -1


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_laplacian_bitwise(name):
    from paper_1708_02845_b200.laplacian import DevicePoisson, mesh_topology
    c = case(name)
    m = c.mesh
    nb_ptr, nb_idx, _ = mesh_topology(m)
    off_ref, diag_ref = mf_sim.laplacian_parts(I.cotan_laplacian(m), nb_ptr, nb_idx)
    dp = DevicePoisson(m)
    off, diag = dp.laplacian()
    off = off.cpu().numpy()[:len(nb_idx)]
    diag = diag.cpu().numpy()
    assert np.array_equal(off.view(np.int64), off_ref.view(np.int64))
    assert np.array_equal(diag.view(np.int64), diag_ref.view(np.int64))


@pytest.mark.gpu
def test_device_lc_matches_reference_csr():
    import paper_1708_02845_b200.laplacian as L
    c = case("c1")
    ls = L.assemble_cotan(c.mesh)
    ref = I.cotan_laplacian(c.mesh)
    lc = ls.lc
    assert np.array_equal(lc.indptr, ref.indptr) and np.array_equal(lc.indices, ref.indices)
    assert np.array_equal(lc.data.view(np.int64), ref.data.view(np.int64))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("leaf", [16, 64])
def test_device_poisson_matches_reference(name, leaf):
    from paper_1708_02845_b200.laplacian import DevicePoisson
    c = case(name)
    assert c.input_matches_reference()
    dp = DevicePoisson(c.mesh, leaf=leaf)
    P, residual, rse = dp.solve()
    Pd = P[:, :c.k].cpu().numpy()
    interior = np.asarray(c.mesh.interior_vertices)
    zero_ok, rel, small = _pcompare(Pd, c.dense, interior)
    assert zero_ok
    assert rel < P_RTOL, rel
    assert small < 1e-300
    bnd = np.asarray(c.mesh.boundary_vertices)
    np.testing.assert_array_equal(Pd[bnd], c.dense[bnd])  # indicator rows, exactly
    assert np.all(P[:, c.k:].cpu().numpy() == 0.0)        # pad columns
    assert residual < 1e-12 and rse < 1e-12
    # deterministic: a second solve is bitwise identical
    P2, r2, s2 = dp.solve()
    assert bool((P2 == P).all()) and r2 == residual and s2 == rse


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "corridor50", "disk40", "holes_fine"])
def test_fields_on_device_P_match_goldens(name):
    """dv_field (K2/K3) on the device-built P against the reference's fields
    computed from the reference's P: the hot path end to end from the mesh."""
    import paper_1708_02845_b200 as pf
    import paper_1708_02845_b200.laplacian as L
    c = case(name)
    pk = L.poisson_kernel(L.assemble_cotan(c.mesh))
    assert pk.row_sum_error < 1e-12
    for gname in ("kl", "tv"):
        fd = pf.builtin_f(gname)
        for i, t in enumerate(c.targets):
            got = pf.dv_field(pk, fd, int(t))
            ok, err = rel_close(got.values, c[f"field/{gname}/{i}"], 1e-10)
            assert ok, (gname, t, err)
            assert bool(("clamped" in got.precision_flags)) == bool(c[f"flags/{gname}/{i}"])


@pytest.mark.gpu
def test_poisson_kernel_host_copy_and_device_registration():
    import paper_1708_02845_b200.laplacian as L
    from paper_1708_02845_b200 import _device as dev
    c = case("disk40")
    pk = L.poisson_kernel(L.assemble_cotan(c.mesh))
    dk = dev.device_kernel(pk)  # the registered device P, not a re-upload
    assert dk.P.data_ptr() == dev._cache[id(pk.dense)][1].P.data_ptr()
    np.testing.assert_array_equal(dk.P[:, :c.k].cpu().numpy(), pk.dense)
    assert not pk.dense.flags.writeable
    np.testing.assert_array_equal(pk.boundary, c.boundary)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "holes_fine"])
def test_fused_negentropy_bitwise_k1(name):
    """The build's finalize pass precomputes K1 (H for the KL clamp, min P):
    bitwise what pf_row_negentropy_f64 returns on the finished P."""
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import _native as nat
    from paper_1708_02845_b200.laplacian import KL_CLAMP, DevicePoisson
    t = dev.torch()
    c = case(name)
    dk = DevicePoisson(c.mesh).device_kernel()
    fused = dk._H[KL_CLAMP].clone()
    fused_min = float(dk._min.item())
    H = t.empty_like(fused)
    mn = t.full((1,), float("inf"), dtype=t.float64, device=fused.device)
    nat.call("pf_row_negentropy_f64", dk.P.data_ptr(), dk.ld, dk.rows, dk.k, KL_CLAMP,
             H.data_ptr(), mn.data_ptr(), t.cuda.current_stream().cuda_stream)
    assert bool((H.view(t.int64) == fused.view(t.int64)).all())
    assert float(mn.item()) == fused_min


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "corridor50", "holes_fine"])
@pytest.mark.parametrize("parts", [3, 8])
def test_row_slab_builds_bitwise(name, parts):
    """§8e / §8f-1: each rank builds only its row slab of P (the backward of the
    fronts its rows, their 1-ring and their ancestors need): the slabs are
    bitwise the rows of the whole build, and the per-slab diagnostics' max is
    the whole build's."""
    from paper_1708_02845_b200.laplacian import KL_CLAMP, DevicePoisson
    c = case(name)
    dp = DevicePoisson(c.mesh)
    full, res, rse = dp.solve(fuse_h=True)
    full = full.cpu().numpy()
    H_full = dp.last_H.cpu().numpy()
    bounds = np.linspace(0, dp.n, parts + 1).astype(int)
    res_max = rse_max = 0.0
    fronts = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        dk = dp.device_kernel(slab=(int(a), int(b - a)))
        P = dk.P.cpu().numpy()
        assert dk.row0 == a and dk.rows == b - a
        assert np.array_equal(P.view(np.int64), full[a:b].view(np.int64))
        assert np.array_equal(dk._H[KL_CLAMP].cpu().numpy().view(np.int64),
                              H_full[a:b].view(np.int64))
        res_max, rse_max = max(res_max, dk.residual), max(rse_max, dk.row_sum_error)
        fronts.append(dp.slab_plan(int(a), int(b - a))["fronts"])
    assert res_max == res and rse_max == rse
    assert min(fronts) < dp.plan.nodes  # some rank skips part of the backward


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "holes_fine"])
def test_row_sums_ride_on_the_residual_pass(name):
    """A bare solve() takes row_sum_error from the residual pass's chunk sums
    (no second read of P): bitwise the same P as the fused-K1 build, the same
    residual, a row_sum_error within summation-order noise of the full
    finalize's, and per-slab maxima equal to the whole build's."""
    from paper_1708_02845_b200.laplacian import DevicePoisson
    c = case(name)
    dp = DevicePoisson(c.mesh)
    Pf, res_f, rse_f = dp.solve(fuse_h=True)
    Pf = Pf.cpu().numpy()
    P, res, rse = dp.solve()
    assert np.array_equal(P.cpu().numpy().view(np.int64), Pf.view(np.int64))
    assert res == res_f and abs(rse - rse_f) < 1e-14 and rse < 1e-12
    bounds = np.linspace(0, dp.n, 4).astype(int)
    got = [dp.solve(slab=(int(a), int(b - a)))[1:] for a, b in zip(bounds[:-1], bounds[1:])]
    assert max(g[0] for g in got) == res and max(g[1] for g in got) == rse


def test_residual_chunk_matches_header():
    import re
    from paper_1708_02845_b200.laplacian import RESIDUAL_COLS
    from tests.conftest import ROOT
    hdr = (ROOT / "include" / "pathfield_b200.h").read_text()
    assert int(re.search(r"#define PF_RESIDUAL_COLS (\d+)", hdr).group(1)) == RESIDUAL_COLS


@pytest.mark.gpu
def test_sharded_field_from_mesh_world1():
    """ShardedField.from_mesh over a 1-rank NCCL group: the whole P, bitwise the
    single-GPU build, and a field through the sharded API equal to dv_field."""
    import os
    import torch.distributed as dist
    import paper_1708_02845_b200 as pf
    from paper_1708_02845_b200.laplacian import DevicePoisson
    from paper_1708_02845_b200.parallel import ShardedField
    c = case("holes_fine")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        sf = ShardedField.from_mesh(c.mesh, dist)
        full, res, rse = DevicePoisson(c.mesh).solve()
        assert bool((sf.slab.P == full).all())
        assert sf.slab.residual == res and sf.slab.row_sum_error == rse
        t0 = int(c.targets[0])
        got = sf.field(pf.builtin_f("kl"), t0).values.cpu().numpy()
        ok, err = rel_close(got, c["field/kl/0"], 1e-10)
        assert ok, err
    finally:
        if own:
            dist.destroy_process_group()


@pytest.mark.gpu
def test_no_interior_vertices_gives_indicator_rows():
    """solvers.py:287-291: with an empty interior the reference skips the solve and
    P is the boundary indicator matrix, residual 0."""
    import paper_1708_02845_b200 as pf
    import paper_1708_02845_b200.laplacian as L
    V = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    T = np.array([[0, 1, 2], [0, 2, 3]])
    mesh = pf.TriMesh(V, T)
    assert mesh.m == 0
    pk = L.poisson_kernel(mesh)
    np.testing.assert_array_equal(pk.dense, np.eye(4))
    assert pk.residual == 0.0 and pk.row_sum_error == 0.0


@pytest.mark.gpu
def test_degenerate_triangle_raises():
    """laplacian.py:110-113: a 0/pi angle (zero cross product) raises
    DegenerateGeometryError, as the reference does."""
    from paper_1708_02845_b200.errors import DegenerateGeometryError
    from paper_1708_02845_b200.laplacian import DevicePoisson
    c = case("disk8")
    V = np.array(c.mesh.vertices, dtype=np.float64)
    T = np.array(c.mesh.triangles)
    # collapse one triangle's vertex onto the midpoint of its opposite edge
    a, b, cc = T[0]
    V2 = V.copy()
    V2[cc] = 0.5 * (V[a] + V[b])

    class M:
        vertices, triangles = V2, T
        boundary_vertices = c.mesh.boundary_vertices
        interior_vertices = c.mesh.interior_vertices
    with pytest.raises(DegenerateGeometryError):
        DevicePoisson(M()).laplacian()


def test_threaded_plan_is_the_sequential_plan():
    """nd_plan.cpp partitions subtrees and fills the per-front scatter lists on host
    threads; the plan must not depend on that.  The digest was taken from the
    single-threaded implementation on the same mesh (90,601 vertices, 3,501 fronts:
    large enough for every parallel pass to engage), and two builds must agree."""
    import hashlib
    from paper_1708_02845_b200 import mesh as M
    from paper_1708_02845_b200 import laplacian as L
    mesh = M.grid_mesh(300, 300)
    digests = []
    for _ in range(2):
        pl = L.NdPlan.from_mesh(mesh)
        h = hashlib.sha256()
        for name in sorted(vars(pl)):
            v = getattr(pl, name)
            if isinstance(v, np.ndarray):
                h.update(name.encode())
                h.update(np.ascontiguousarray(v).tobytes())
        digests.append(h.hexdigest())
    assert pl.nodes == 3501
    assert digests[0] == digests[1] == \
        "bcb050007ab4bc93fb62a58ae04eef7ea2f0a0cf4d90d8b14b714637413705d1"
