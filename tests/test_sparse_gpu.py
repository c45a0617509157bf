"""Sparsified kernel (K4) and CSR KL/TV (K5/K6) on the B200 vs the reference goldens.

Bars: CSR pattern (indptr, indices) and kept data bit-exact; dropped mass
bitwise (scipy reduceat order); sparse distances within 1e-10 relative of the
reference's dv_pair_sparse loop; op counts exact.
"""

import math

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from oracle import divergence as O
from oracle import inputs as I
from tests.conftest import case, rel_close

pytestmark = pytest.mark.gpu
RTOL = 1e-10
SPARSE_CASES = ["c1", "corridor50", "disk40"]


def _pk(c):
    return pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)


@pytest.mark.parametrize("name", SPARSE_CASES)
def test_sparsify_bitwise(name):
    c = case(name)
    spk = pf.sparsify(_pk(c))
    np.testing.assert_array_equal(spk.sparse.indptr, c["sp/indptr"])
    np.testing.assert_array_equal(spk.sparse.indices, c["sp/indices"])
    assert I.sha(spk.sparse.data) == str(c["sp/sha_data"])
    np.testing.assert_array_equal(spk.dropped_mass, c["sp/dropped"])
    thr, cut, spct = c["sp/meta"]
    assert spk.threshold == thr and spk.row_cut == cut
    assert spk.sparsity_percent == pytest.approx(spct, abs=1e-12)
    ok, err = rel_close(spk.log_sparse.data, np.log(spk.sparse.data), 1e-15)
    assert ok, err
    assert spk.log_dense.shape == spk.dense.shape
    rep = spk.sparsity_report()
    assert set(rep) == {"threshold", "sparsity_percent", "max_dropped_row_mass"}


GENS = {"kl": {}, "tv": {}, "chi2": {}, "hellinger": {}, "alpha": {"alpha": 0.5},
        "power-p": {"power": 3}}


@pytest.mark.parametrize("name", SPARSE_CASES)
@pytest.mark.parametrize("g", list(GENS))
def test_sparse_field_matches_reference_pair_loop(name, g):
    c = case(name)
    if f"spfield/{g}" not in c.keys():
        pytest.skip("golden has kl/tv only for this case")
    spk = pf.sparsify(_pk(c))
    fld = pf.dv_field_sparse(spk, pf.builtin_f(g, **GENS[g]), c.target)
    ok, err = rel_close(fld.values, c[f"spfield/{g}"], RTOL)
    assert ok, (name, g, err)
    rng = np.random.default_rng(1)
    for q in rng.choice(c.n, 8, replace=False):
        _, ops = pf.dv_pair_sparse_stats(spk, pf.builtin_f(g, **GENS[g]), c.target, int(q))
        assert ops == int(c[f"spops/{g}"][q]), (g, q)


@pytest.mark.parametrize("name", SPARSE_CASES)
def test_sparse_pairs_and_ops(name):
    c = case(name)
    spk = pf.sparsify(_pk(c))
    rng = np.random.default_rng(5)
    for g in ("kl", "tv"):
        fd = pf.builtin_f(g)
        for q in rng.choice(c.n, 16, replace=False):
            val, ops = pf.dv_pair_sparse_stats(spk, fd, c.target, int(q))
            assert ops == int(c[f"spops/{g}"][q]), (g, q)
            ok, err = rel_close([val], [c[f"spfield/{g}"][q]], RTOL)
            assert ok, (g, q, err)
    # q == p: KL exactly 0, TV exactly 2 * dropped_p (divergence.py:288-295)
    assert pf.dv_pair_sparse(spk, pf.builtin_f("kl"), c.target, c.target) == 0.0
    d = spk.dropped_mass[c.target]
    assert pf.dv_pair_sparse(spk, pf.builtin_f("tv"), c.target, c.target) == d + d


def test_zero_threshold_identity_and_validation():
    c = case("disk40")
    pk = _pk(c)
    spk = pf.sparsify(pk, 0.0)
    assert spk.sparsity_percent == 0.0 or spk.sparse.nnz == int((c.dense > 0).sum())
    np.testing.assert_array_equal(spk.sparse.toarray(), np.where(c.dense > 0, c.dense, 0.0))
    kl = pf.builtin_f("kl")
    for q in (3, 500, 2000):
        dense = pf.dv_pair(pk, kl, c.target, q)
        assert pf.dv_pair_sparse(spk, kl, c.target, q) == pytest.approx(dense, rel=1e-12)
    with pytest.raises(ValueError):
        pf.sparsify(pk, 1.0)
    with pytest.raises(ValueError):
        pf.sparsify(pk, -0.5)
    with pytest.raises(pf.DivergenceDomainError):
        pf.dv_pair_sparse(pk, kl, 0, 1)


def test_corridor_sparse_accuracy_and_bounds():
    # reference test_divergence.py:207-250 restated on the device path
    c = case("corridor50")
    pk = _pk(c)
    spk = pf.sparsify(pk)
    assert spk.sparsity_percent > 80.0
    kl, tv = pf.builtin_f("kl"), pf.builtin_f("tv")
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(50):
        p, q = (int(x) for x in rng.integers(0, c.n, 2))
        if p == q:
            continue
        dense = pf.dv_pair(pk, kl, p, q)
        sparse = pf.dv_pair_sparse(spk, kl, p, q)
        if dense > 0:
            worst = max(worst, abs(sparse - dense) / dense)
        dt = pf.dv_pair(pk, tv, p, q)
        st = pf.dv_pair_sparse(spk, tv, p, q)
        assert abs(st - dt) <= 2 * (spk.dropped_mass[p] + spk.dropped_mass[q]) + 1e-12
        _, ops = pf.dv_pair_sparse_stats(spk, kl, p, q)
        assert ops < c.k
    assert worst < 0.01


def test_log_dense_view():
    c = case("c1")
    spk = pf.sparsify(_pk(c))
    ld = np.asarray(spk.log_dense)
    ok, err = rel_close(ld, np.log(np.maximum(c.dense, 1e-300)), 1e-15)
    assert ok, err


@pytest.mark.parametrize("n,k,thr", [(500, 64, None), (300, 1, None), (257, 33, 0.5), (64, 30001, None)])
def test_synthetic_sparse_vs_oracle(n, k, thr):
    rng = np.random.default_rng(n + k)
    dense = I.synthetic_kernel(n, k, seed=n) ** 3
    dense /= dense.sum(axis=1, keepdims=True)
    dense[:, 0] = 0.0
    boundary = np.array([1, 2]) if n > 2 else np.array([], np.int64)
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    spk = pf.sparsify(pk, thr)
    sv = O.sparsify(dense, boundary, thr)
    np.testing.assert_array_equal(spk.sparse.indptr, sv["indptr"])
    np.testing.assert_array_equal(spk.sparse.indices, sv["indices"])
    np.testing.assert_array_equal(spk.dropped_mass, sv["dropped"])
    t = n // 3
    for g in ("kl", "tv"):
        got = pf.dv_field_sparse(spk, pf.builtin_f(g), t).values
        ref = O.dv_field_sparse(sv, g, t)
        ok, err = rel_close(got, ref, RTOL)
        assert ok, (g, err)


def test_sparse_slabs_bitwise():
    """CSR row slabs (as N GPUs would hold them) give bitwise the 1-slab sparse field."""
    import math
    import torch
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import parallel as par
    c = case("corridor50")
    spk = pf.sparsify(_pk(c))
    cut = (1.0 / math.sqrt(c.n)) / c.k
    full = {g: pf.dv_field_sparse(spk, pf.builtin_f(g), c.target).values for g in ("kl", "tv")}
    indptr = spk.sparse.indptr
    bounds = par.partition_by_weight(np.diff(indptr), 3)
    slabs = [dev.DeviceKernel(c.dense, c.boundary, row0=a, rows=b - a) for a, b in bounds]
    own = par.owner_of(c.target, bounds)
    kp = c.k + (c.k & 1)
    tv_payload = torch.empty(kp + 4, dtype=torch.float64, device="cuda")
    par._sparse_tv_prep(slabs[own], cut, False, c.target, tv_payload)
    kl_payload = torch.from_numpy(c.dense[c.target].copy()).cuda()
    for g, payload in (("kl", kl_payload), ("tv", tv_payload)):
        parts = [par._compute_sparse_slab(sl, pf.builtin_f(g), c.target, payload, cut, False)
                 for sl in slabs]
        torch.cuda.synchronize()
        got = torch.cat(parts).cpu().numpy()
        np.testing.assert_array_equal(got, full[g])


@pytest.mark.parametrize("name", SPARSE_CASES)
def test_u16_columns_bitwise_equal_int32(name):
    """The 16-bit-column field kernels (pf_csr_{kl,tv}_u16_f64) return exactly the
    int32-column results: same entries, same visiting order."""
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import divergence as D
    c = case(name)
    spk = pf.sparsify(_pk(c))
    dk, dc = D._device_csr(spk)
    assert dc.indices16 is not None
    np.testing.assert_array_equal(dc.indices16.cpu().numpy().astype(np.int64) & 0xffff,
                                  dc.indices.cpu().numpy().astype(np.int64))
    t = dev.torch()
    target = int(c.target)
    for g in ("kl", "tv"):
        a = pf.dv_field_sparse(spk, pf.builtin_f(g), target).values.copy()
        saved = dc.indices16
        try:
            dc.indices16 = None  # force the int32 entry points
            b = pf.dv_field_sparse(spk, pf.builtin_f(g), target).values.copy()
        finally:
            dc.indices16 = saved
        assert np.array_equal(a.view(np.int64), b.view(np.int64)), g
    del t


def test_csr_kl_guard_in_place():
    """Rows that nearly repeat the target's make hs[q] - sum v logPt cancel; K5 must
    re-evaluate them (in place, in the field kernel) in the reference form: values
    within 1e-10 of the oracle, the guard counter equal to the rows that fired, and the
    field path equal bitwise to the query path (dv_at-style launch, same order)."""
    import torch as t
    from paper_1708_02845_b200 import divergence as D
    n, k, p = 2048, 512, 100
    dense = I.synthetic_kernel(n, k, seed=3)
    # near-duplicates far enough apart that one-ulp differences between the device's
    # and numpy's log stay below 1e-10 of the distance (KL >= ~1e-6)
    for j, eps in enumerate([0.0, 1e-2, -1e-2, 3e-2, 5e-2, 1e-1, -1e-1, 0.3]):
        row = dense[p].copy()
        row[3::7] *= (1.0 + eps)
        dense[200 + j] = row / row.sum()
    pk = pf.PoissonKernel(dense, np.array([], np.int64), 0.0, 0.0)
    spk = pf.sparsify(pk)
    thr = 1.0 / math.sqrt(n)
    vals, flags = D.dv_field_sparse_device(spk, pf.builtin_f("kl"), p)
    field = vals.cpu().numpy()
    guarded = int(flags[1].item())
    assert guarded >= 4
    rows = np.r_[np.arange(190, 215), [0, 1, n - 1]]
    ref = np.array([O.dv_pair_sparse_direct(dense, p, int(q), "kl", threshold=thr)[0]
                    for q in rows])
    ok, err = rel_close(field[rows], ref, RTOL)
    assert ok, err
    for q in rows:
        assert pf.dv_pair_sparse(spk, pf.builtin_f("kl"), p, int(q)) == field[q]
