"""Full-size parity on the REAL C2 Poisson kernel (BASELINE config 2/3).

C2 is the reference's 50:1 corridor `generate_rectangle_mesh(50, 1, 0.024)`,
102,104 vertices x 4,250 boundary vertices.  The mesh is
rebuilt with the reference's generator restatement (workloads/meshes.py,
bitwise the reference's on the golden cases) and P with the reference's own
preprocessing restated — SuperLU of -Lc_II and column solves
(oracle/inputs.poisson_kernel_parallel, all host cores, ~5 s on the box).
Against that P:

* dense KL / TV fields at three targets, every row, within 1e-10 relative
  (divergence.py:154-187), the `clamped` flag exact, the split-form KL guard
  engaged on real rows;
* sparsify at the default threshold: CSR pattern, data and dropped mass
  bit-exact on every row (divergence.py:194-240);
* CSR KL / TV fields on 4,000 sampled rows within 1e-10 of the reference's
  per-pair formulas (divergence.py:255-299);
* 20 traced paths per field bit-exact against the oracle tracer on the same
  field values (paths.py:137-307);
* the device-built P (K11) componentwise within 1e-11 of SuperLU's.
"""

import math
import os

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from tests.conftest import rel_close

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    from oracle import inputs as I
    from workloads.meshes import SPECS, default_endpoints
    mesh = I.build(SPECS["c2"])
    dense, boundary = I.poisson_kernel_parallel(mesh, workers=os.cpu_count() or 8)
    assert dense.shape == (102_104, 4_250)
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    src, tgt = default_endpoints(mesh)
    rng = np.random.default_rng(0)
    targets = [tgt] + [int(x) for x in rng.choice(mesh.interior_vertices, 2, replace=False)]
    return {"mesh": mesh, "dense": dense, "boundary": boundary, "pk": pk, "src": src,
            "tgt": tgt, "targets": targets}


def test_c2_dense_fields_every_row(c2):
    from oracle import divergence as O
    dense, pk = c2["dense"], c2["pk"]
    guarded = 0
    for t in c2["targets"]:
        for g in ("kl", "tv"):
            fld = pf.dv_field(pk, pf.builtin_f(g), t)
            ref = O.dv_field_chunked(dense, g, t, chunk_rows=1024)
            ref[(ref > -1e-10) & (ref < 0.0)] = 0.0
            ref[t] = 0.0
            ok, err = rel_close(fld.values, ref, 1e-10)
            assert ok, f"{g} target {t}: max rel err {err:.3e}"
            flag = O.clamp_flag(dense, c2["boundary"], t, O.generator(g)[1])
            assert (fld.precision_flags == ("clamped",)) == flag
            if g == "kl":
                _, fl = pf.dv_field_device(pk, pf.builtin_f("kl"), t)
                guarded += int(fl[1].item())
    assert guarded > 0   # real P: the cancellation guard runs on the rows near each target


def test_c2_sparsify_bitwise_every_row(c2):
    from oracle import divergence as O
    spk = pf.sparsify(c2["pk"])
    sv = O.sparsify(c2["dense"], c2["boundary"])
    np.testing.assert_array_equal(spk.sparse.indptr, sv["indptr"])
    np.testing.assert_array_equal(spk.sparse.indices, sv["indices"])
    np.testing.assert_array_equal(spk.sparse.data, sv["data"])
    np.testing.assert_array_equal(spk.dropped_mass, sv["dropped"])
    assert spk.sparse.nnz == 49_690_217
    assert spk.sparsity_percent == sv["sparsity_percent"]
    rows = np.random.default_rng(1).choice(c2["dense"].shape[0], 4000, replace=False)
    t = c2["tgt"]
    for g in ("kl", "tv"):
        fld = pf.dv_field_sparse(spk, pf.builtin_f(g), t)
        ref = np.array([O.dv_pair_sparse_stats(sv, g, t, int(q))[0] for q in rows])
        ok, err = rel_close(fld.values[rows], ref, 1e-10)
        assert ok, f"sparse {g}: max rel err {err:.3e}"
    assert pf.dv_pair_sparse(spk, pf.builtin_f("tv"), t, t) == 2.0 * sv["dropped"][t]


def test_c2_paths_bitwise(c2):
    from oracle import tracer as TR
    m = c2["mesh"]
    tm = pf.TriMesh(m.vertices, m.triangles)
    topo = TR.topology(m.triangles, m.n)
    rng = np.random.default_rng(2)
    tgt = c2["tgt"]
    srcs = [c2["src"]] + [int(x) for x in rng.choice(m.interior_vertices, 19, replace=False)]
    srcs = [s for s in srcs if s != tgt]
    for g in ("kl", "tv"):
        fld = pf.dv_field(c2["pk"], pf.builtin_f(g), tgt)
        paths = pf.triangle_descent_batch(tm, fld, srcs)
        for s, p in zip(srcs, paths):
            o = TR.triangle_descent(m.vertices, m.triangles, m.areas, m.bbox_diagonal,
                                    fld.values, tgt, int(s), topo=topo)
            assert p.status == o["status"] and p.locations == o["locations"]
            np.testing.assert_array_equal(p.points, o["points"])
        assert any(p.status == "reached" for p in paths)


def test_c2_device_poisson_kernel_vs_superlu(c2):
    import torch
    from paper_1708_02845_b200 import laplacian as L
    dk = L.DevicePoisson(c2["mesh"]).device_kernel()
    ref = torch.from_numpy(c2["dense"]).cuda()
    got = dk.P[:, :dk.k]
    big = ref > 1e-290
    rel = ((got - ref).abs() / ref.clamp_min(1e-300))[big]
    assert float(rel.max()) <= 1e-11
    assert torch.equal(got == 0, ref == 0)
    assert dk.residual < 1e-9 and dk.row_sum_error < 1e-9
    # the field on the device-built P equals the field on SuperLU's P within 1e-10
    b = pf.dv_field(c2["pk"], pf.builtin_f("kl"), c2["tgt"]).values
    vals, _ = _field_on(dk, c2["tgt"])
    ok, err = rel_close(vals, b, 1e-10)
    assert ok, f"KL on device P vs SuperLU P: {err:.3e}"
    assert math.isfinite(err)


def _field_on(dk, t):
    """KL field over a device-only P (no host dense) via the C ABI path of dv_field."""
    import torch
    from paper_1708_02845_b200 import divergence as D
    out = torch.empty(dk.rows + 2, dtype=torch.float64, device=dk.device)
    s = torch.cuda.current_stream(dk.device).cuda_stream
    st = D._field_device(None, dk, pf.builtin_f("kl"), t, False, 1e-300, out,
                         out.data_ptr() + dk.rows * 8, s)
    torch.cuda.synchronize()
    del st
    return out[:dk.rows].cpu().numpy(), out[dk.rows:].view(torch.int32).cpu().numpy()
