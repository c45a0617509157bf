"""The sharded path on the B200 with a real NCCL communicator (pf_nccl_*).

This box has one GPU, so the communicator has one rank (the multi-rank host
logic is covered on gloo in test_parallel.py); what runs here is the product
data plane end to end: NCCL loaded and initialised through the C ABI, the
target-row broadcast, the flag max-reduction, the all-gather feeding the
tracer, the strided trace of a rank's batched-KL columns — each compared
bitwise with the single-GPU public API.
"""

import os
import socket

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _device as dev
from paper_1708_02845_b200 import parallel as par
from tests.conftest import case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def group():
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def _same_path(a, b):
    assert a.status == b.status and a.locations == b.locations
    np.testing.assert_array_equal(a.points, b.points)


def test_nccl_collectives_one_rank(group):
    import ctypes
    import torch
    comm = par.NcclComm(group, torch.device("cuda", 0))
    try:
        v = ctypes.c_int(0)
        from paper_1708_02845_b200 import _native as nat
        nat.call("pf_nccl_version", ctypes.byref(v))
        assert v.value >= 22000
        x = torch.arange(7, dtype=torch.float64, device="cuda")
        comm.broadcast(x, 0)
        g = comm.all_gather(x)
        m = torch.tensor([3, -2], dtype=torch.int32, device="cuda")
        comm.all_reduce(m, "max")
        torch.cuda.synchronize()
        assert torch.equal(g, x) and m.tolist() == [3, -2]
    finally:
        comm.close()


@pytest.mark.parametrize("name", ["c1", "corridor50"])
def test_sharded_field_equals_dv_field(group, name):
    c = case(name)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    dk = dev.device_kernel(pk)
    sf = par.ShardedField(dk, par.partition_rows(c.n, 1), group)
    try:
        for g in ("kl", "tv"):
            for t in c.targets[:3]:
                ref = pf.dv_field(pk, pf.builtin_f(g), int(t))
                loc = sf.field(pf.builtin_f(g), int(t))
                np.testing.assert_array_equal(loc.values.cpu().numpy(), ref.values)
                assert loc.precision_flags == ref.precision_flags
                full = sf.field(pf.builtin_f(g), int(t), gather=True)
                np.testing.assert_array_equal(full.values, ref.values)
                assert full.precision_flags == ref.precision_flags
        with pytest.raises(pf.InvalidTargetError):
            sf.field(pf.builtin_f("kl"), c.n)
        with pytest.raises(pf.DivergenceDomainError):
            sf.field(pf.builtin_f("kl"), int(c.target), clamp=0.0)
        sp = pf.sparsify(pk)
        for g in ("kl", "tv"):
            ref = pf.dv_field_sparse(sp, pf.builtin_f(g), int(c.target))
            got = sf.sparse_field(pf.builtin_f(g), int(c.target), gather=True)
            np.testing.assert_array_equal(got.values, ref.values)
    finally:
        sf.close()


def test_sharded_trace_and_c5_trace_batch(group):
    c = case("c1")
    mesh = pf.TriMesh(c.mesh.vertices, c.mesh.triangles)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    dk = dev.device_kernel(pk)
    interior = np.setdiff1d(np.arange(c.n), c.boundary)
    rng = np.random.default_rng(3)
    targets = rng.choice(interior, 6, replace=False)
    sources = rng.choice(interior, 40)
    field_of = np.arange(40) % 6
    sources = np.where(sources == targets[field_of], interior[0], sources)
    kl = pf.builtin_f("kl")
    # the same composition through the single-GPU API: the batched fields
    # (K7, within 1e-10 of dv_field), then triangle_descent_batch per source
    from tests.conftest import rel_close
    batch = pf.dv_field_batch(pk, kl, targets)
    fields = [pf.ScalarField(np.ascontiguousarray(batch[:, j]), "kl", int(t))
              for j, t in enumerate(targets)]
    for j, t in enumerate(targets):
        assert rel_close(batch[:, j], pf.dv_field(pk, kl, int(t)).values, 1e-10)[0]
    ref = pf.triangle_descent_batch(mesh, fields, sources, field_of=field_of)
    got = par.trace_batch(mesh, pk, kl, targets, sources, field_of, group, gather_paths=True)
    for a, b in zip(got, ref):
        _same_path(a, b)
    sf = par.ShardedField(dk, par.partition_rows(c.n, 1), group)
    try:
        src0 = sources[field_of == 0]
        got0 = sf.trace(mesh, kl, int(targets[0]), src0, gather_paths=True)
        ref0 = pf.triangle_descent_batch(mesh, pf.dv_field(pk, kl, int(targets[0])), src0)
        for a, b in zip(got0, ref0):
            _same_path(a, b)
    finally:
        sf.close()
