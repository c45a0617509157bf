"""Dense KL/TV (and the other generators) on the B200 vs the reference goldens.

Bar (BASELINE north_star): FP64 distances within 1e-10 relative; the
`clamped` precision flag, the settle rule and the exact zero at the target
reproduced exactly.
"""

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from paper_1708_02845_b200 import _device as dev
from oracle import divergence as O
from tests.conftest import CASES, case, rel_close

pytestmark = pytest.mark.gpu
RTOL = 1e-10
GENS = {"kl": {}, "tv": {}, "chi2": {}, "hellinger": {}, "alpha": {"alpha": 0.5},
        "power-p": {"power": 3}}


def _pk(c):
    return pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)


@pytest.mark.parametrize("name", CASES)
def test_dense_fields_match_reference(name):
    c = case(name)
    pk = _pk(c)
    worst = {}
    for key in c.keys():
        if not key.startswith("field/"):
            continue
        _, g, ti = key.split("/")
        t = c.targets[int(ti)]
        fld = pf.dv_field(pk, pf.builtin_f(g, **GENS[g]), t)
        ref = c[key]
        ok, err = rel_close(fld.values, ref, RTOL)
        worst[key] = err
        assert ok, (key, err)
        assert fld.values[t] == 0.0
        assert (fld.precision_flags == ("clamped",)) == bool(c[f"flags/{g}/{ti}"]), key
        assert fld.kind == g and fld.target == t and fld.sign == 1
        assert not fld.values.flags.writeable
    print(name, "max rel err", max(worst.values()))


@pytest.mark.parametrize("name", ["disk8", "c1"])
def test_swap_order_matches_reference(name):
    c = case(name)
    fld = pf.dv_field(_pk(c), pf.builtin_f("kl"), c.target, swap_order=True)
    ok, err = rel_close(fld.values, c["field_swap/kl"], RTOL)
    assert ok, err
    assert fld.params.get("swap_order") is True


@pytest.mark.parametrize("name", CASES)
def test_dv_at_and_pair_match_reference(name):
    c = case(name)
    pk = _pk(c)
    for g in GENS:
        if f"at/{g}" not in c.keys():
            continue
        fd = pf.builtin_f(g, **GENS[g])
        qs = c[f"at_q/{g}"]
        ok, err = rel_close(pf.dv_at(pk, fd, c.target, qs), c[f"at/{g}"], RTOL)
        assert ok, (g, err)
        pairs = [pf.dv_pair(pk, fd, c.target, int(q)) for q in qs[:8]]
        ok, err = rel_close(pairs, c[f"pair/{g}"], RTOL)
        assert ok, (g, err)


def test_pair_identity_and_domain_errors():
    c = case("disk8")
    pk = _pk(c)
    assert pf.dv_pair(pk, pf.builtin_f("kl"), 7, 7) == 0.0
    q = int(c.boundary[0])
    with pytest.raises(pf.DivergenceDomainError):
        pf.dv_pair(pk, pf.builtin_f("kl"), 0, q, clamp=0.0)
    with pytest.raises(pf.DivergenceDomainError):
        pf.dv_field(pk, pf.builtin_f("kl"), 0, clamp=0.0)


def test_clamp_disabled_on_positive_kernel():
    # all-positive P: clamp=0 is allowed and equals the unclamped formula
    dense = O_synth(300, 37, seed=3)
    pk = pf.PoissonKernel(dense, np.array([], dtype=np.int64), 0.0, 0.0)
    for g in ("kl", "tv"):
        got = pf.dv_field(pk, pf.builtin_f(g), 5, clamp=0.0)
        ref, flags = O.dv_field(dense, [], g, 5, clamp=0.0)
        ok, err = rel_close(got.values, ref, RTOL)
        assert ok, err
        assert got.precision_flags == ()


def O_synth(n, k, seed):
    from oracle.inputs import synthetic_kernel
    return synthetic_kernel(n, k, seed)


@pytest.mark.parametrize("n,k", [(1, 1), (33, 1), (257, 3), (1000, 17), (4099, 208), (2048, 4250),
                                 (64, 30001)])
def test_ragged_shapes_vs_oracle(n, k):
    dense = O_synth(n, k, seed=n + k)
    dense[:, 0] = 0.0 if k > 2 else dense[:, 0]  # exact zeros, as P has
    pk = pf.PoissonKernel(dense, np.array([0]) if n > 1 else np.array([], np.int64), 0.0, 0.0)
    for g in ("kl", "tv", "hellinger"):
        for t in sorted({0, n // 2, n - 1}):
            got = pf.dv_field(pk, pf.builtin_f(g), t)
            ref, flags = O.dv_field(dense, pk.boundary, g, t)
            ok, err = rel_close(got.values, ref, RTOL)
            assert ok, (g, t, err)
            assert got.precision_flags == flags


def test_kl_guard_engages_near_target():
    # rows close to the target row trip the cancellation guard and are
    # recomputed per-element; the result still meets the 1e-10 bar.
    c = case("disk40")
    pk = _pk(c)
    vals, flags = pf.dv_field_device(pk, pf.builtin_f("kl"), c.target)
    import torch
    torch.cuda.synchronize()
    assert int(flags[1].item()) > 0
    ok, err = rel_close(vals.cpu().numpy(), c["field/kl/0"], RTOL)
    assert ok, err


def test_negentropy_matches_numpy():
    c = case("c1")
    pk = _pk(c)
    dk = dev.device_kernel(pk)
    H = dk.negentropy(1e-300).cpu().numpy()
    q = np.maximum(c.dense, 1e-300)
    ref = (q * np.log(q)).sum(axis=1)
    ok, err = rel_close(H, ref, 1e-12)
    assert ok, err
    assert dk.min_value() == c.dense.min()


@pytest.mark.parametrize("spec", [
    {"gen": "holes", "spacing": 0.0125},                       # n=16,176 k=838
    {"gen": "rectangle", "length": 20.0, "width": 1.0, "spacing": 0.05},  # corridor 20:1
])
def test_real_kernels_vs_oracle_medium(spec):
    """Real Poisson kernels rebuilt with the reference's preprocessing (oracle/inputs.py):
    KL/TV fields at several targets within 1e-10 of the reference arithmetic."""
    from oracle import inputs as I
    mesh = I.build(spec)
    dense, boundary = I.poisson_kernel(mesh)
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    src, tgt = I.default_endpoints(mesh)
    rng = np.random.default_rng(1)
    targets = [tgt, int(boundary[3])] + [int(x) for x in rng.choice(mesh.interior_vertices, 2)]
    for g in ("kl", "tv"):
        for t in targets:
            got = pf.dv_field(pk, pf.builtin_f(g), t)
            ref, flags = O.dv_field(dense, boundary, g, t)
            ok, err = rel_close(got.values, ref, RTOL)
            assert ok, (spec, g, t, err)
            assert got.precision_flags == flags


def test_one_vs_many_slabs_bitwise():
    """Row sharding: a field computed slab by slab (as N GPUs would) is bitwise the
    single-slab field, because every row is reduced by the same kernel code."""
    import torch
    c = case("holes_fine")
    full = pf.dv_field(_pk(c), pf.builtin_f("kl"), c.target).values
    tv_full = pf.dv_field(_pk(c), pf.builtin_f("tv"), c.target).values
    parts_kl, parts_tv = [], []
    bounds = np.linspace(0, c.n, 4).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        dk = dev.DeviceKernel(c.dense, c.boundary, row0=int(a), rows=int(b - a))
        for g, parts in (("kl", parts_kl), ("tv", parts_tv)):
            fd = pf.builtin_f(g)
            out = torch.empty(dk.rows + 2, dtype=torch.float64, device=dk.device)
            row = torch.from_numpy(c.dense[c.target].copy()).cuda()
            st = pf.divergence._field_device(None, dk, fd, c.target, False, fd.clamp, out,
                                             out.data_ptr() + dk.rows * 8,
                                             torch.cuda.current_stream().cuda_stream, target_row=row)
            torch.cuda.synchronize()
            parts.append(out[:dk.rows].cpu().numpy())
            del st
    np.testing.assert_array_equal(np.concatenate(parts_kl), full)
    np.testing.assert_array_equal(np.concatenate(parts_tv), tv_full)


@pytest.mark.parametrize("rows,k,row0", [(1, 7, 0), (5000, 4250, 0), (3000, 33, 1234),
                                         (70000, 130, 17)])
def test_staged_upload_bitwise(rows, k, row0):
    """_hostpool.upload_rows: pinned staging with several chunks and buffer reuse, padded
    leading dimension, a row offset, a non-float64 source (cast as np.array did)."""
    import torch as t
    from paper_1708_02845_b200 import _hostpool
    rng = np.random.default_rng(rows + k)
    host = rng.random((row0 + rows, k))
    old = _hostpool._UPLOAD_CHUNK_BYTES
    _hostpool._UPLOAD_CHUNK_BYTES = 1 << 20     # force many chunks through 3 buffers
    try:
        for src in (host, host.astype(np.float32)):
            ld = dev.leading_dim(k)
            P = t.full((rows, ld), -1.0, dtype=t.float64, device="cuda")
            _hostpool.upload_rows(t, P, src, row0)
            got = P.cpu().numpy()
            assert np.array_equal(got[:, :k], src[row0:].astype(np.float64))
            assert (got[:, k:] == -1.0).all()
    finally:
        _hostpool._UPLOAD_CHUNK_BYTES = old
