"""Reentrancy (SURVEY §8b "Threading"): the service runs dv_field / triangle_descent
from a FastAPI thread pool, and DomainContext only locks its lazy preprocessing
(domain.py:49-70).  Four threads hit one fresh PoissonKernel at once (one device
mirror must be built), then keep calling the field and tracer paths; every
result must equal the reference's golden output."""

import threading

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _device as dev
from tests.conftest import case, rel_close

pytestmark = pytest.mark.gpu


def test_four_threads_fields_and_paths():
    c = case("disk40")
    dense = np.array(c.dense)            # a fresh array: no device mirror yet
    pk = pf.PoissonKernel(dense, c.boundary, 0.0, 0.0)
    mesh = pf.TriMesh(c.mesh.vertices, c.mesh.triangles)
    built = []
    orig = dev.DeviceKernel.__init__

    def counting_init(self, *a, **kw):
        built.append(1)
        orig(self, *a, **kw)

    # single-threaded references on a separate copy of the kernel
    pk1 = pf.PoissonKernel(np.array(c.dense), c.boundary, 0.0, 0.0)
    srcs = [int(s) for s in c["path_sources"]]
    ref = {}
    for g in ("kl", "tv"):
        f1 = pf.dv_field(pk1, pf.builtin_f(g), int(c.target))
        ref[g] = (f1.values.copy(), [pf.triangle_descent(mesh, f1, s).points for s in srcs])
    # the goldens are read here: the case's lazy npz is not safe to read from 4 threads
    golden = {g: np.array(c[f"field/{g}/0"]) for g in ("kl", "tv")}
    dev.DeviceKernel.__init__ = counting_init
    errors, start = [], threading.Barrier(4)

    def worker(i):
        try:
            start.wait()
            for it in range(6):
                g = ("kl", "tv")[(i + it) % 2]
                fld = pf.dv_field(pk, pf.builtin_f(g), int(c.target))
                ok, err = rel_close(fld.values, golden[g], 1e-10)
                assert ok, f"thread {i} {g}: {err:.3e}"
                np.testing.assert_array_equal(fld.values, ref[g][0])
                j = (i + it) % len(srcs)
                path = pf.triangle_descent(mesh, fld, srcs[j])
                np.testing.assert_array_equal(path.points, ref[g][1][j])
        except Exception as exc:  # reported in the main thread
            errors.append(exc)

    try:
        threads = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
        for th in threads:
            th.start()
        for th in threads:
            th.join(timeout=300)
    finally:
        dev.DeviceKernel.__init__ = orig
    assert not errors, errors[0]
    assert len(built) == 1, f"{len(built)} device mirrors built for one kernel"


def test_traced_field_stays_on_device():
    """DomainContext.trace = dv_field then triangle_descent on the returned
    field: the tracer reads the field's device copy (no re-upload)."""
    c = case("c1")
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    fld = pf.dv_field(pk, pf.builtin_f("kl"), int(c.target))
    assert dev.field_mirror(fld.values) is not None
    mesh = pf.TriMesh(c.mesh.vertices, c.mesh.triangles)
    p = pf.triangle_descent(mesh, fld, int(c.source))
    # the same values uploaded from a fresh host copy trace the same path
    q = pf.triangle_descent(mesh, pf.ScalarField(fld.values.copy(), "kl", int(c.target)),
                            int(c.source))
    np.testing.assert_array_equal(p.points, q.points)
    assert p.locations == q.locations and p.reached
