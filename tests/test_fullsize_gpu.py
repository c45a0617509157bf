"""Parity at BASELINE.json's full sizes on one B200.

The goldens (tests/golden) pin the kernels against the reference's own outputs at
sizes the oracle finishes in seconds.  Here the same public calls run at the
benchmark shapes on synthetic P generated on the device, and are checked by

* the oracle (``oracle/divergence.py``, ``oracle/tracer.py``) on sampled rows,
  targets and paths — every sampled value is what the reference computes for that
  row, because each row's value depends only on that row and the target row;
* size-independent properties: exact zero at the target, the ``clamped`` flag,
  ``TV(p, p) = 2·dropped_p`` in the sparse form, the CSR nnz against an
  independent device count, slab-sharded fields bitwise equal to the whole field.

P lives only in HBM (32.8 GB at C4): the PoissonKernel handed to the public API
wraps a zero-stride host stub of the right shape, registered to the device copy
(``_device.register``), the same way ``poisson_kernel_device`` binds a P that was
produced on the GPU.
"""

import math

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _device as dev
from oracle import divergence as O
from oracle import tracer as TR
from tests.conftest import rel_close

pytestmark = pytest.mark.gpu
RTOL = 1e-10
C4 = (1_000_386, 4_102)
C2 = (102_104, 4_250)
N_BOUNDARY = 64            # indicator rows (the reference's boundary rows)
ZERO_ROW = 777_777         # an interior row with one extra exact zero -> "clamped"


def _stub_kernel(dk, boundary):
    """PoissonKernel over the device-resident P of `dk` (no host copy of P)."""
    stub = np.lib.stride_tricks.as_strided(np.zeros(1), shape=(dk.n, dk.k), strides=(0, 0))
    pk = pf.PoissonKernel(stub, np.asarray(boundary, np.int64), 0.0, 0.0)
    dev.register(stub, dk)
    return pk


def _rows(dk, idx):
    import torch as t
    return dk.P.index_select(0, t.from_numpy(np.asarray(idx, np.int64)).to(dk.device))[
        :, :dk.k].cpu().numpy()


@pytest.fixture(scope="module")
def c4():
    import torch as t
    n, k = C4
    ld = dev.leading_dim(k)
    P = t.empty((n, ld), dtype=t.float64, device="cuda")
    g = t.Generator(device="cuda")
    g.manual_seed(4)
    for a in range(0, n, 32768):
        b = min(n, a + 32768)
        x = t.randn((b - a, k), dtype=t.float64, device="cuda", generator=g)
        x[:, 0] = -float("inf")                     # a zero column in every interior row
        P[a:b, :k] = t.softmax(x, dim=1)
    P[:, k:] = 0.0
    boundary = np.arange(N_BOUNDARY, dtype=np.int64) * 15_601 + 3
    P[t.from_numpy(boundary).cuda(), :k] = 0.0
    P[t.from_numpy(boundary).cuda(), t.arange(N_BOUNDARY, device="cuda") + 1] = 1.0
    P[ZERO_ROW, 5] = 0.0
    t.cuda.synchronize()
    dk = dev.DeviceKernel(None, boundary, rows=n, n=n, k=k, P_dev=P)
    pk = _stub_kernel(dk, boundary)
    rng = np.random.default_rng(4)
    interior = np.setdiff1d(np.arange(n), boundary)
    sample = np.unique(np.concatenate([rng.choice(n, 3000, replace=False), boundary[:8],
                                       [0, 1, n - 1, ZERO_ROW]]))
    yield dict(pk=pk, dk=dk, n=n, k=k, boundary=boundary, interior=interior, sample=sample,
               rng=rng)
    del dk, pk, P
    t.cuda.empty_cache()


def _oracle_rows(c, name, p, rows):
    """The reference's values at `rows` for target p, from those rows alone."""
    host = _rows(c["dk"], np.concatenate([[p], rows]))
    return O.dv_at(host, name, 0, np.arange(1, len(rows) + 1))


def test_c4_dense_fields_sampled_rows_and_flags(c4):
    """C4 (1,000,386 x 4,102): dv_field KL and TV through the public API."""
    for p in (int(c4["interior"][c4["n"] // 3]), int(c4["boundary"][5])):
        for g in ("kl", "tv"):
            fld = pf.dv_field(c4["pk"], pf.builtin_f(g), p)
            assert fld.values.shape == (c4["n"],) and fld.values[p] == 0.0
            ok, err = rel_close(fld.values[c4["sample"]], _oracle_rows(c4, g, p, c4["sample"]),
                                RTOL)
            assert ok, (g, p, err)
            # divergence.py:172-175: an interior row whose zero pattern differs from the
            # target row's -> ("clamped",).  ZERO_ROW differs from every interior target
            # (column 5); a boundary target's indicator row differs from every interior row.
            assert fld.precision_flags == ("clamped",), (g, p)
            if g == "tv":
                assert (fld.values >= 0).all() and (fld.values <= 2.0 + 1e-12).all()


def _slab_flag(c4, a, b, fd, p):
    import torch as t
    dk, n, k = c4["dk"], c4["n"], c4["k"]
    sk = dev.DeviceKernel(None, c4["boundary"], row0=a, rows=b - a, n=n, k=k, P_dev=dk.P[a:b])
    out = t.empty(sk.rows + 2, dtype=t.float64, device=sk.device)
    st = pf.divergence._field_device(None, sk, fd, p, False, fd.clamp, out,
                                     out.data_ptr() + sk.rows * 8,
                                     t.cuda.current_stream().cuda_stream,
                                     target_row=dk.P[p, :k])
    t.cuda.synchronize()
    del st
    return int(out[sk.rows:].view(t.int32)[0].item())


def test_c4_flag_only_from_interior_rows_that_differ(c4):
    """The flag rule (divergence.py:172-175) per slab: rows [0, 700000) hold boundary
    indicator rows (excluded) and interior rows whose only zero is column 0, as in the
    target -> no flag; rows [700000, n) contain ZERO_ROW -> flag."""
    p = int(c4["interior"][12345])
    assert p < 700_000
    for g in ("kl", "tv"):
        fd = pf.builtin_f(g)
        assert _slab_flag(c4, 0, 700_000, fd, p) == 0, g
        assert _slab_flag(c4, 700_000, c4["n"], fd, p) != 0, g


def test_c4_row_slabs_bitwise(c4):
    """8 row slabs (the row-sharded multi-GPU layout) reproduce the whole
    field bit for bit."""
    import torch as t
    dk, n, k = c4["dk"], c4["n"], c4["k"]
    p = int(c4["interior"][777])
    bounds = np.linspace(0, n, 9).astype(int)
    row = dk.P[p, :k]
    for g in ("kl", "tv"):
        fd = pf.builtin_f(g)
        whole = pf.dv_field(c4["pk"], fd, p).values
        for a, b in zip(bounds[:-1], bounds[1:]):
            sk = dev.DeviceKernel(None, c4["boundary"], row0=int(a), rows=int(b - a), n=n, k=k,
                                  P_dev=dk.P[a:b])
            out = t.empty(sk.rows + 2, dtype=t.float64, device=sk.device)
            st = pf.divergence._field_device(None, sk, fd, p, False, fd.clamp, out,
                                             out.data_ptr() + sk.rows * 8,
                                             t.cuda.current_stream().cuda_stream, target_row=row)
            t.cuda.synchronize()
            np.testing.assert_array_equal(out[:sk.rows].cpu().numpy(), whole[a:b])
            del st, sk


def test_c4_fp32_mode_within_1e5(c4):
    p = int(c4["interior"][999])
    for g in ("kl", "tv"):
        f32 = pf.divergence.dv_field_f32(c4["pk"], pf.builtin_f(g), p)
        ok, err = rel_close(f32.values[c4["sample"]], _oracle_rows(c4, g, p, c4["sample"]),
                            1e-5)
        assert ok, (g, err)
    c4["dk"]._p32 = None   # release the 16 GB FP32 copy before the batched test


def test_c5_batched_kl_1024_targets(c4):
    """C5: T = 1,024 targets x 1,000,386 rows as one contraction (K7, int8 tensor pipe)."""
    import torch as t
    rng = np.random.default_rng(5)
    targets = rng.choice(c4["interior"], 1024, replace=False)
    targets[0] = c4["boundary"][2]                  # an indicator row among the targets
    out, flags = pf.divergence.dv_field_batch_device(c4["pk"], pf.builtin_f("kl"), targets)
    assert out.shape == (c4["n"], 1024)
    diag = out[t.from_numpy(targets).cuda(), t.arange(1024, device="cuda")].cpu().numpy()
    assert (diag == 0.0).all()
    assert flags.all()                              # ZERO_ROW differs from every target
    rows = c4["sample"][::3]
    cols = np.concatenate([[0], rng.choice(np.arange(1, 1024), 15, replace=False)])
    got = out[t.from_numpy(rows).cuda()][:, t.from_numpy(cols).cuda()].cpu().numpy()
    for jj, j in enumerate(cols):
        ok, err = rel_close(got[:, jj], _oracle_rows(c4, "kl", int(targets[j]), rows), RTOL)
        assert ok, (int(targets[j]), err)
    del out
    c4["dk"]._scratch.clear()
    t.cuda.empty_cache()


def test_c3_csr_full_size():
    """C3 shape: 102,104 x 4,250 corridor-banded P at the default 1/sqrt(n) threshold
    (~490 kept entries per row).  Pattern, data and dropped mass bitwise on sampled rows,
    total nnz against an independent count, sparse KL/TV fields vs the oracle."""
    import torch as t
    n, k = C2
    ld = dev.leading_dim(k)
    P = t.empty((n, ld), dtype=t.float64, device="cuda")
    b = t.arange(k, dtype=t.float64, device="cuda")[None, :]
    for a in range(0, n, 8192):
        e = min(n, a + 8192)
        q = t.arange(a, e, dtype=t.float64, device="cuda")[:, None]
        c1 = t.floor(q / n * (k / 2))
        x = t.exp(-t.abs(b - c1) / 12.5) + t.exp(-t.abs(b - ((k - 1) - c1)) / 12.5)
        P[a:e, :k] = x / x.sum(dim=1, keepdim=True)
    P[:, k:] = 0.0
    boundary = np.array([0, 5000, n - 1], np.int64)
    P[t.from_numpy(boundary).cuda(), :k] = 0.0
    P[t.from_numpy(boundary).cuda(), t.tensor([0, 7, k - 1], device="cuda")] = 1.0
    dk = dev.DeviceKernel(None, boundary, rows=n, n=n, k=k, P_dev=P)
    pk = _stub_kernel(dk, boundary)
    spk = pf.sparsify(pk)
    thr = 1.0 / math.sqrt(n)
    cut = thr / k
    assert spk.row_cut == cut
    indptr = np.asarray(spk.sparse.indptr, np.int64)
    ind = np.asarray(spk.sparse.indices)
    data = np.asarray(spk.sparse.data)
    nnz_dev = int(sum(int((P[a:a + 8192, :k] >= cut).sum()) for a in range(0, n, 8192)))
    assert indptr[-1] == nnz_dev
    rng = np.random.default_rng(3)
    sample = np.unique(np.concatenate([rng.choice(n, 600, replace=False), boundary]))
    host = _rows(dk, sample)
    dropped = np.asarray(spk.dropped_mass)
    for r, row in zip(sample, host):
        idx, vals, drop = O._kept_row(host, cut, False, int(np.flatnonzero(sample == r)[0]))
        np.testing.assert_array_equal(ind[indptr[r]:indptr[r + 1]], idx)
        np.testing.assert_array_equal(data[indptr[r]:indptr[r + 1]], vals)
        assert dropped[r] == drop
    interior = np.ones(n, bool)
    interior[boundary] = False
    want_sp = 100.0 * (1.0 - int(np.diff(indptr)[interior].sum()) / (interior.sum() * k))
    assert abs(spk.sparsity_percent - want_sp) <= 1e-12 * want_sp
    p = n // 3 + 1
    hp = _rows(dk, np.concatenate([[p], sample]))
    for g in ("kl", "tv"):
        fld = pf.divergence.dv_field_sparse(spk, pf.builtin_f(g), p)
        ref = np.array([O.dv_pair_sparse_direct(hp, 0, i + 1, g, threshold=thr)[0]
                        for i in range(len(sample))])
        ok, err = rel_close(fld.values[sample], ref, RTOL)
        assert ok, (g, err)
        if g == "kl":
            assert fld.values[p] == 0.0
        else:
            assert fld.values[p] == 2.0 * dropped[p]          # divergence.py:288-295
    del spk, pk, dk, P
    t.cuda.empty_cache()


def test_c5_tracer_10k_paths_sampled_bitwise():
    """C5 tracer shape: 10,000 paths (source i -> target i % 1024) on a 1,002,001-vertex
    mesh in one batch; 16 sampled paths (all non-reached ones first) bitwise equal to
    the oracle's triangle_descent on the same field."""
    import torch as t
    from paper_1708_02845_b200 import mesh as M
    from paper_1708_02845_b200 import paths as PP
    mesh = M.grid_mesh(1000, 1000)
    dm = M.device_mesh(mesh)
    rng = np.random.default_rng(1)
    T = 1024
    targets = rng.choice(mesh.interior_vertices, T, replace=False)
    fields = t.cdist(dm.V.index_select(0, t.from_numpy(targets).cuda()), dm.V)
    src = rng.choice(mesh.n, 10_000)
    fo = np.arange(10_000) % T
    src = np.where(src == targets[fo], (src + 1) % mesh.n, src)
    buf, counts, over, extra = PP.trace_arrays(mesh, fields, targets, src, fo)
    paths = PP._host_paths(buf, counts, over, extra, src, targets, fo)
    status = np.array([p.status for p in paths])
    assert (status == "reached").mean() > 0.99
    pick = list(np.flatnonzero(status != "reached")[:8])
    pick += list(rng.choice(np.flatnonzero(status == "reached"), 16 - len(pick), replace=False))
    V, Tr = np.asarray(mesh.vertices), np.asarray(mesh.triangles)
    topo = TR.topology(Tr, len(V))
    for i in pick:
        vals = fields[int(fo[i])].cpu().numpy()
        o = TR.triangle_descent(V, Tr, np.asarray(mesh.triangle_areas), float(mesh.bbox_diagonal),
                                vals, int(targets[fo[i]]), int(src[i]), topo=topo)
        p = paths[i]
        assert p.status == o["status"], i
        assert p.locations == o["locations"], i
        np.testing.assert_array_equal(p.points, o["points"])
