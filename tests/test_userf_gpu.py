"""User-defined generators on the B200 (NVRTC-compiled, csrc/pf_jit.cu) against
the reference's own formulas restated in numpy (divergence.py:137-187 dense,
:296-299 sparse union form), on real Poisson kernels from the goldens."""

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from tests.conftest import case, rel_close

pytestmark = pytest.mark.gpu

JS = pf.FDivergence("js", lambda x: x * np.log(x) - (1 + x) * np.log((1 + x) / 2), True)
XLOGX_KL = pf.FDivergence("kl", lambda x: x * np.log(x), True)   # named like a builtin
PIECE = pf.FDivergence("piece", lambda x: np.where(x > 1.0, (x - 1.0) ** 2, x - 1.0 - np.log(x)),
                       True, clamp=1e-150)


def _ref_field(dense, boundary, fd, p, swap=False, clamp=None):
    """divergence.py:154-187 with the generator's own f (numpy)."""
    c = fd.clamp if clamp is None else clamp
    ps = np.maximum(dense[p], c)
    qs = np.maximum(dense, c)
    with np.errstate(all="ignore"):
        if swap:
            vals = (ps[None, :] * fd.f(qs / ps[None, :])).sum(axis=1)
        else:
            vals = (qs * fd.f(ps[None, :] / qs)).sum(axis=1)
    vals[(vals > -1e-10) & (vals < 0.0)] = 0.0
    vals[p] = 0.0
    interior = np.ones(len(dense), bool)
    interior[boundary] = False
    fired = bool(((dense < c) != (dense[p][None, :] < c))[interior].any())
    return vals, ("clamped",) if fired else ()


@pytest.mark.parametrize("name", ["c1", "disk40"])
@pytest.mark.parametrize("fd", [JS, XLOGX_KL, PIECE], ids=["js", "xlogx-named-kl", "piecewise"])
def test_user_generator_dense_field(name, fd):
    c = case(name)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    for t in c.targets[:3]:
        for swap in (False, True):
            got = pf.dv_field(pk, fd, int(t), swap_order=swap)
            ref, flags = _ref_field(c.dense, c.boundary, fd, int(t), swap)
            ok, err = rel_close(got.values, ref, 1e-10)
            assert ok, f"{fd.name} target {t} swap={swap}: {err:.3e}"
            assert got.precision_flags == flags and got.kind == fd.name
        q = np.arange(0, c.n, 7)
        at = pf.dv_at(pk, fd, int(t), q)
        ok, err = rel_close(at, np.where(q == int(t), 0.0, _ref_field(c.dense, c.boundary, fd,
                                                                        int(t))[0][q]), 1e-10)
        assert ok, err


def test_named_kl_user_generator_is_not_the_builtin():
    c = case("c1")
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    a = pf.dv_field(pk, XLOGX_KL, int(c.target)).values
    b = pf.dv_field(pk, pf.builtin_f("kl"), int(c.target)).values
    assert not np.allclose(a, b)


def test_user_generator_sparse_union_form():
    c = case("corridor50")
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    sp = pf.sparsify(pk)
    t = int(c.target)
    S = sp.sparse
    for q in range(0, c.n, 97):
        idx_p = S.indices[S.indptr[t]:S.indptr[t + 1]]
        idx_q = S.indices[S.indptr[q]:S.indptr[q + 1]]
        val_q = S.data[S.indptr[q]:S.indptr[q + 1]]
        union = np.union1d(idx_p, idx_q)
        vq = np.full(union.size, sp.row_cut)
        vq[np.searchsorted(union, idx_q)] = val_q
        vp = np.maximum(c.dense[t, union], sp.row_cut)
        ref = float(vq @ JS.f(vp / vq))
        ref = 0.0 if -1e-10 < ref < 0.0 else ref
        got, ops = pf.dv_pair_sparse_stats(sp, JS, t, q)
        assert ops == union.size
        assert rel_close([got], [ref], 1e-10)[0], (q, got, ref)
