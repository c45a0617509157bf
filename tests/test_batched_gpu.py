"""K7 batched-target KL vs T x dv_field, on both contraction paths: the FP64
DMMA GEMM ("f64") and the exact-integer emulation on the int8 tensor pipe
("i8", tcgen05 — batched_i8.cu)."""

import numpy as np
import pytest

import paper_1708_02845_b200 as pf
from oracle import divergence as O
from oracle import inputs as I
from tests.conftest import CASES, case, rel_close

pytestmark = pytest.mark.gpu
RTOL = 1e-10


METHODS = ("i8", "f64")


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("name", CASES)
def test_batch_matches_reference_fields(name, method):
    c = case(name)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    targets = c.targets
    out, flags = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), targets,
                                                     method=method)
    got = out.cpu().numpy()
    for j, t in enumerate(targets):
        ok, err = rel_close(got[:, j], c[f"field/kl/{j}"], RTOL)
        assert ok, (name, method, j, err)
        assert bool(flags[j]) == bool(c[f"flags/kl/{j}"])
    host = pf.dv_field_batch(pk, pf.builtin_f("kl"), targets, method=method)
    np.testing.assert_array_equal(host, got)


@pytest.mark.parametrize("method", METHODS)
def test_batch_equals_single_target_calls_large_T(method):
    # T spanning several 128-wide target tiles and a ragged row tile
    mesh = I.build({"gen": "holes", "spacing": 0.03, "seed": 1})
    dense, boundary = I.poisson_kernel(mesh)
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    rng = np.random.default_rng(3)
    targets = rng.choice(mesh.n, 300, replace=False)
    got = pf.dv_field_batch(pk, pf.builtin_f("kl"), targets, method=method)
    for j in range(0, 300, 23):
        ref, _ = O.dv_field(dense, boundary, "kl", int(targets[j]))
        ok, err = rel_close(got[:, j], ref, RTOL)
        assert ok, (j, err)


@pytest.mark.parametrize("method", METHODS)
def test_batch_flags_nonuniform_masks_and_other_generators(method):
    dense = I.synthetic_kernel(700, 67, seed=4)
    dense[::7, 3] = 0.0          # interior rows with different zero patterns
    boundary = np.array([1, 5])
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    targets = [0, 7, 100, 699]
    out, flags = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), targets,
                                                     method=method)
    got = out.cpu().numpy()
    for j, t in enumerate(targets):
        ref, fl = O.dv_field(dense, boundary, "kl", t)
        ok, err = rel_close(got[:, j], ref, RTOL)
        assert ok, err
        assert bool(flags[j]) == bool(fl)
    tv = pf.dv_field_batch(pk, pf.builtin_f("tv"), targets)
    for j, t in enumerate(targets):
        ref, _ = O.dv_field(dense, boundary, "tv", t)
        ok, err = rel_close(tv[:, j], ref, RTOL)
        assert ok, err


def test_i8_and_f64_paths_agree_and_guard_fires():
    # rows next to each target are near-duplicates (KL ~ 0): the split-form
    # guard must route them to the reference-form fixup on both paths
    rng = np.random.default_rng(11)
    base = I.synthetic_kernel(300, 129, seed=5)
    dense = np.repeat(base, 2, axis=0)
    dense[1::2] *= 1.0 + 1e-4 * rng.standard_normal(dense[1::2].shape)
    dense /= dense.sum(axis=1, keepdims=True)
    pk = pf.PoissonKernel(dense, np.array([0, 1]), 0.0, 0.0)
    targets = np.arange(2, 600, 37)
    a8, _ = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), targets, method="i8")
    a64, _ = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), targets, method="f64")
    a8, a64 = a8.cpu().numpy(), a64.cpu().numpy()
    for j, t in enumerate(targets):
        ref, _ = O.dv_field(dense, np.array([0, 1]), "kl", int(t))
        assert rel_close(a8[:, j], ref, RTOL)[0], j
        assert rel_close(a64[:, j], ref, RTOL)[0], j
        assert 0 < ref[t ^ 1] < 1e-6  # the twin row: split form cancels -> guarded


def test_i8_limits():
    dense = I.synthetic_kernel(64, 4800, seed=6)
    pk = pf.PoissonKernel(dense, np.array([], dtype=np.int64), 0.0, 0.0)
    with pytest.raises(ValueError):
        pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), [3], method="i8")
    out, _ = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), [3, 9])  # auto -> f64
    ref, _ = O.dv_field(dense, np.array([], dtype=np.int64), "kl", 9)
    assert rel_close(out.cpu().numpy()[:, 1], ref, RTOL)[0]
    with pytest.raises(ValueError):
        pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), [3], method="bogus")


@pytest.mark.parametrize("name", CASES)
def test_i8_fp32_grade_within_north_star_tolerance(name):
    c = case(name)
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    out, flags = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), c.targets,
                                                     method="i8-f32")
    got = out.cpu().numpy()
    for j, t in enumerate(c.targets):
        ok, err = rel_close(got[:, j], c[f"field/kl/{j}"], 1e-5)
        assert ok, (name, j, err)
        assert got[t, j] == 0.0
        assert bool(flags[j]) == bool(c[f"flags/kl/{j}"])


@pytest.mark.parametrize("method", METHODS)
def test_batch_slabs_bitwise_and_flags_or(method):
    """Row-sharded K7 (parallel.ShardedField.field_batch): each slab contracted
    against the assembled target rows, as N GPUs would, is bitwise the
    single-GPU batch, and the OR of the slab flags is the reference's flag."""
    import torch
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import parallel as par
    c = case("holes_fine")
    pk = pf.PoissonKernel(c.dense, c.boundary, 0.0, 0.0)
    targets = np.array(c.targets)
    full, flags = pf.divergence.dv_field_batch_device(pk, pf.builtin_f("kl"), targets,
                                                      method=method)
    full = full.cpu().numpy()
    rows = torch.from_numpy(c.dense[targets].copy()).cuda()
    parts, fl = [], np.zeros(len(targets), bool)
    bounds = np.linspace(0, c.n, 4).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        dk = dev.DeviceKernel(c.dense, c.boundary, row0=int(a), rows=int(b - a))
        vals, f = par._compute_batch_slab(dk, pf.builtin_f("kl"), targets, rows, method)
        parts.append(vals.cpu().numpy())
        fl |= f
    np.testing.assert_array_equal(np.concatenate(parts), full)
    np.testing.assert_array_equal(fl, flags)


@pytest.mark.parametrize("rows,k,T", [(300, 200, 50), (129, 64, 64), (2047, 1234, 256),
                                      (2, 5, 1), (127, 31, 3), (385, 33, 65), (640, 97, 200)])
def test_i8_cta_pair_kernel_bitwise_equals_single_cta(rows, k, T):
    """K7 on a CTA pair (tcgen05 cta_group::2, M256 over two SMs) computes the same
    exact integer levels as the single-CTA kernel: the outputs are bitwise equal,
    including odd row-tile counts (a pair's second CTA past the last row) and
    ragged target tiles."""
    import torch
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import divergence as D
    rng = np.random.default_rng(rows)
    P = rng.random((rows, k)) ** 4
    P[:, 0] = 0.0
    P /= P.sum(axis=1, keepdims=True)
    pk = pf.PoissonKernel(P, np.array([1]), 0.0, 0.0)
    targets = rng.choice(rows, T, replace=False)
    old = D.I8_CTA_PAIR
    try:
        D.I8_CTA_PAIR = False
        a, fa = D.dv_field_batch_device(pk, pf.builtin_f("kl"), targets, method="i8")
        a = a.clone()
        D.I8_CTA_PAIR = True
        b, fb = D.dv_field_batch_device(pk, pf.builtin_f("kl"), targets, method="i8")
    finally:
        D.I8_CTA_PAIR = old
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int64), b.view(torch.int64))
    assert np.array_equal(fa, fb)


def test_guard_list_fixup_matches_scan_fixup_and_overflow():
    """The K7 epilogue's guarded-pair list + list fixup give the scan fixup's
    values bitwise, with a list that holds every pair and with one that
    overflows (falls back to the scan)."""
    import torch
    from paper_1708_02845_b200 import _device as dev, _native as nat
    from paper_1708_02845_b200 import divergence as D
    mesh = I.build({"gen": "holes", "spacing": 0.03, "seed": 1})
    dense, boundary = I.poisson_kernel(mesh)
    pk = pf.PoissonKernel(dense, boundary, 0.0, 0.0)
    dk = dev.device_kernel(pk)
    rng = np.random.default_rng(5)
    T = 200
    tg = torch.from_numpy(rng.choice(mesh.n, T, replace=False).astype(np.int64)).cuda()
    s = torch.cuda.current_stream().cuda_stream
    k, rows = dk.k, dk.rows
    ldl = dev.round_up(k, 16)
    Pt = dk.P.index_select(0, tg)
    L = torch.empty((T, ldl), dtype=torch.float64, device="cuda")
    Tc = torch.empty_like(L)
    nat.call("pf_batch_prep_f64", Pt.data_ptr(), Pt.stride(0), T, k, ldl, 1e-300, 0,
             L.data_ptr(), Tc.data_ptr(), 0, s)
    A, ea, ldk = dk.slices(1e-300)
    B = torch.empty((7, T, ldk), dtype=torch.uint8, device="cuda")
    eb = torch.empty(T, dtype=torch.int32, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    nat.call("pf_slice_targets_u8", L.data_ptr(), ldl, T, k, ldk, B.data_ptr(), eb.data_ptr(),
             bad.data_ptr(), s)
    H = dk.negentropy(1e-300)
    res = {}
    for mode, cap in (("scan", 0), ("list", rows * T), ("overflow", 3)):
        out = torch.empty((rows, T), dtype=torch.float64, device="cuda")
        cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        glist = torch.zeros(max(cap, 1) + 1, dtype=torch.int64, device="cuda")
        nat.call("pf_batched_kl_i8_listed", A.data_ptr(), ea.data_ptr(), rows, B.data_ptr(),
                 eb.data_ptr(), T, k, ldk, H.data_ptr(), tg.data_ptr(), D.KL_GUARD_TAU, 0,
                 out.data_ptr(), out.stride(0), 64, 1, glist.data_ptr() if cap else None,
                 cap, s)
        if mode == "scan":
            nat.call("pf_batched_kl_fixup_f64", dk.P.data_ptr(), dk.ld, rows, k, Tc.data_ptr(),
                     ldl, T, 1e-300, out.data_ptr(), out.stride(0), cnt.data_ptr(), s)
        else:
            nat.call("pf_batched_kl_fixup_list_f64", dk.P.data_ptr(), dk.ld, rows, k,
                     Tc.data_ptr(), ldl, T, 1e-300, out.data_ptr(), out.stride(0), cnt.data_ptr(),
                     glist.data_ptr(), cap, s)
        torch.cuda.synchronize()
        res[mode] = (out.cpu(), int(cnt.item()), int(glist[0].item()))
    n_scan = res["scan"][1]
    assert n_scan > 0                                   # the case has guarded pairs
    assert res["list"][2] == n_scan and res["list"][1] == n_scan
    assert res["overflow"][2] == n_scan > 3 and res["overflow"][1] == n_scan
    for mode in ("list", "overflow"):
        assert torch.equal(res[mode][0].view(torch.int64), res["scan"][0].view(torch.int64)), mode


@pytest.mark.parametrize("rows,k,T", [(129, 64, 64), (300, 200, 50), (1000, 1234, 130)])
def test_tiled_slices_are_the_swizzled_row_major_planes(rows, k, T):
    """pf_slice_rows_u8_tiled / pf_slice_targets_u8_tiled write the same bytes
    as the row-major slicing, permuted into R x 32-byte SWIZZLE_32B tiles
    (chunk c of row r at r * 32 + (c ^ (r >> 2 & 1)) * 16), zero padded."""
    import torch
    from paper_1708_02845_b200 import _device as dev
    from paper_1708_02845_b200 import _native as nat
    rng = np.random.default_rng(rows + k)
    P = rng.random((rows, k)) ** 3
    P /= P.sum(axis=1, keepdims=True)
    Pd = torch.from_numpy(P).cuda()
    s = torch.cuda.current_stream().cuda_stream
    ldk = dev.round_up(k, 64)

    def untile(buf, n, R):
        nkb = (k + 31) // 32
        npad = (n + 127) // 128 * 128
        tiles = buf.reshape(7, npad // R, nkb, R, 2, 16)
        r = np.arange(R)
        swz = (r >> 2) & 1
        un = np.empty_like(tiles)
        for c in (0, 1):   # smem chunk c holds logical chunk c ^ swz
            un[:, :, :, r, c ^ swz, :] = tiles[:, :, :, r, c, :]
        return un.transpose(0, 1, 3, 2, 4, 5).reshape(7, npad, nkb * 32)

    for what, n, R in (("rows", rows, 128), ("targets", T, 64)):
        src = Pd if what == "rows" else torch.log(Pd[:n].clamp_min(1e-300))
        plain = torch.zeros((7, n, ldk), dtype=torch.uint8, device="cuda")
        tiled = torch.full((dev.i8_tiled_bytes(n, k),), 0xAB, dtype=torch.uint8, device="cuda")
        e1 = torch.empty(n, dtype=torch.int32, device="cuda")
        e2 = torch.empty_like(e1)
        if what == "rows":
            nat.call("pf_slice_rows_u8", src.data_ptr(), k, n, k, 1e-300, ldk, plain.data_ptr(),
                     e1.data_ptr(), s)
            nat.call("pf_slice_rows_u8_tiled", src.data_ptr(), k, n, k, 1e-300, tiled.data_ptr(),
                     e2.data_ptr(), s)
        else:
            L = src.contiguous()
            nat.call("pf_slice_targets_u8", L.data_ptr(), k, n, k, ldk, plain.data_ptr(),
                     e1.data_ptr(), 0, s)
            nat.call("pf_slice_targets_u8_tiled", L.data_ptr(), k, n, k, tiled.data_ptr(),
                     e2.data_ptr(), 0, s)
        torch.cuda.synchronize()
        assert torch.equal(e1, e2)
        un = untile(tiled.cpu().numpy(), n, R)
        kk = (k + 31) // 32 * 32
        want = np.zeros_like(un)
        want[:, :n, :min(kk, ldk)] = plain.cpu().numpy()[:, :, :kk]
        np.testing.assert_array_equal(un, want, err_msg=what)
