"""Multi-process (world_size 2 and 3, gloo, CPU) checks of the row-sharding host logic.

The slab computation and the per-rank tracer are swapped for the CPU oracle
inside these tests only (the product's _compute_slab / _trace_local always run
the CUDA kernels); what is under test is partitioning, ownership, the
target-row broadcast, the flag / domain-check reductions that keep
dv_field's single-process contract (divergence.py:157-183) on every rank,
the variable-size all-gathers, and which rank traces which path.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1708_02845_b200 import parallel as par


def test_partitions():
    b = par.partition_rows(10, 3)
    assert b == [(0, 4), (4, 7), (7, 10)]
    assert par.owner_of(4, b) == 1 and par.owner_of(9, b) == 2
    from paper_1708_02845_b200.errors import InvalidTargetError
    with pytest.raises(InvalidTargetError):
        par.owner_of(10, b)
    w = np.array([100, 1, 1, 1, 100, 1, 1, 1])
    pb = par.partition_by_weight(w, 2)
    assert pb[0][0] == 0 and pb[-1][1] == 8 and pb[0][1] == pb[1][0]
    sums = [w[a:c].sum() for a, c in pb]
    assert max(sums) <= 110
    for n in (1, 7, 1000):
        for world in (1, 2, 8):
            bb = par.partition_rows(n, world)
            assert bb[0][0] == 0 and bb[-1][1] == n
            assert all(x[1] == y[0] for x, y in zip(bb, bb[1:]))


class _Slab:
    def __init__(self, P, r0, r1):
        self.P = torch.from_numpy(P[r0:r1].copy())
        self.row0, self.rows, self.k, self.n = r0, r1 - r0, P.shape[1], P.shape[0]
        self.device = torch.device("cpu")

    def min_value(self):
        return float(self.P.min()) if self.rows else float("inf")


def _install_oracle_slab(P, boundary):
    """Replace the CUDA slab computations with the oracle (test harness only)."""
    from oracle import divergence as O
    interior = np.ones(P.shape[0], bool)
    interior[boundary] = False

    def oracle_slab(slab, fd, p, row, clamp, swap_order=False):
        full = np.vstack([row.numpy()[None, :], slab.P.numpy()])
        vals = O.dv_at(full, fd.name, 0, np.arange(1, slab.rows + 1), swap_order=swap_order,
                       clamp=clamp if clamp > 0 else 0.0)
        vals[(vals > -1e-10) & (vals < 0.0)] = 0.0
        vals[np.arange(slab.row0, slab.row0 + slab.rows) == p] = 0.0
        Ps = slab.P.numpy()
        inter = interior[slab.row0:slab.row0 + slab.rows]
        fired = clamp > 0 and bool(np.any((Ps[inter] < clamp) != (row.numpy()[None, :] < clamp)))
        return torch.from_numpy(vals), torch.tensor([int(fired)], dtype=torch.int32)

    def oracle_sparse_slab(slab, fd, p, payload, cut, strict):
        vals = np.array([O.dv_pair_sparse_direct(P, p, q, fd.name)[0]
                         for q in range(slab.row0, slab.row0 + slab.rows)])
        return torch.from_numpy(vals)

    def oracle_tv_prep(slab, cut, strict, p, payload):
        payload.fill_(float(p))  # any owner-computed payload: checks the broadcast path

    par._compute_slab = oracle_slab
    par._compute_sparse_slab = oracle_sparse_slab
    par._sparse_tv_prep = oracle_tv_prep


def _init(rank, world, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _worker(rank, world, port, P, boundary, target, q):
    _init(rank, world, port)
    try:
        from oracle import divergence as O
        import paper_1708_02845_b200 as pf
        from paper_1708_02845_b200.errors import DivergenceDomainError, InvalidTargetError
        _install_oracle_slab(P, boundary)
        bounds = par.partition_rows(P.shape[0], world)
        slab = _Slab(P, *bounds[rank])
        sf = par.ShardedField(slab, bounds, dist, device=torch.device("cpu"))
        row = sf.target_row(target, P.shape[1])
        assert np.array_equal(row.numpy(), P[target])
        for g in ("kl", "tv"):
            fld = sf.field(pf.builtin_f(g), target, gather=True)
            ref, rflags = O.dv_field(P, boundary, g, target)
            q.put((rank, g, bool(np.array_equal(fld.values, ref))
                   and fld.precision_flags == tuple(rflags) and not fld.values.flags.writeable))
            loc = sf.field(pf.builtin_f(g), target)
            a, b = bounds[rank]
            q.put((rank, g + "-slab", bool(np.array_equal(loc.values.numpy(), ref[a:b]))
                   and loc.row0 == a and loc.precision_flags == tuple(rflags)))
            sp = sf.sparse_field(pf.builtin_f(g), target, gather=True)
            sref = np.array([O.dv_pair_sparse_direct(P, target, qq, g)[0]
                             for qq in range(P.shape[0])])
            q.put((rank, "sparse-" + g, bool(np.array_equal(sp.values, sref))
                   and sp.precision_flags == ()))
        # a bad target raises the reference's type on every rank, before any collective
        try:
            sf.field(pf.builtin_f("kl"), P.shape[0])
            q.put((rank, "bad-target", False))
        except InvalidTargetError:
            q.put((rank, "bad-target", True))
        # clamp <= 0 with a zero entry on ONE slab: every rank raises (no rank hangs)
        try:
            sf.field(pf.builtin_f("kl"), target, clamp=0.0)
            q.put((rank, "domain", False))
        except DivergenceDomainError:
            q.put((rank, "domain", True))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, fn, args, nres, timeout=180):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=fn, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=timeout) for _ in range(nres * world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for *_, ok in res), res
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_field_gloo(world):
    from oracle.inputs import synthetic_kernel
    P = synthetic_kernel(101, 13, seed=world)
    P[:, 0] = 0.0
    boundary = np.array([3])
    target = 77  # owned by the last rank: exercises a non-zero broadcast source
    _run(world, _worker, (P, boundary, target), 8)


def _flag_worker(rank, world, port, P, boundary, target, q):
    """The one-sided clamp fires only on a row of rank 0's slab: every rank's
    SlabField reports it (the flag word is max-reduced)."""
    _init(rank, world, port)
    try:
        from oracle import divergence as O
        import paper_1708_02845_b200 as pf
        _install_oracle_slab(P, boundary)
        bounds = par.partition_rows(P.shape[0], world)
        sf = par.ShardedField(_Slab(P, *bounds[rank]), bounds, dist, device=torch.device("cpu"))
        loc = sf.field(pf.builtin_f("kl"), target)
        _, rflags = O.dv_field(P, boundary, "kl", target)
        q.put((rank, "flag", tuple(rflags) == ("clamped",)
               and loc.precision_flags == ("clamped",)))
        # clamp <= 0: the only zero entry sits on rank 0's slab, yet every rank
        # raises (slab minima are min-reduced first; no rank is left in a collective)
        from paper_1708_02845_b200.errors import DivergenceDomainError
        try:
            sf.field(pf.builtin_f("kl"), target, clamp=0.0)
            q.put((rank, "domain", False))
        except DivergenceDomainError:
            q.put((rank, "domain", True))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_clamped_flag_from_another_slab(world):
    from oracle.inputs import synthetic_kernel
    P = synthetic_kernel(60, 9, seed=5)
    P[1, 4] = 0.0          # the only sub-clamp entry of an interior row, on rank 0's slab
    boundary = np.array([0])
    _run(world, _flag_worker, (P, boundary, 59), 2)


def _batch_worker(rank, world, port, P, boundary, targets, q):
    _init(rank, world, port)
    try:
        from oracle import divergence as O
        import paper_1708_02845_b200 as pf
        interior = np.ones(P.shape[0], bool)
        interior[boundary] = False
        c = 1e-300

        def oracle_batch_slab(slab, fd, tg, rows, method="auto", clamp=None):
            rows = rows.numpy()
            Ps = slab.P.numpy()
            cols, flags = [], []
            for j, t in enumerate(tg):
                full = np.vstack([rows[j][None, :], Ps])
                v = O.dv_at(full, fd.name, 0, np.arange(1, slab.rows + 1))
                v[np.arange(slab.row0, slab.row0 + slab.rows) == t] = 0.0
                cols.append(v)
                inter = interior[slab.row0:slab.row0 + slab.rows]
                flags.append(bool(np.any((Ps[inter] < c) != (rows[j] < c))))
            return torch.from_numpy(np.stack(cols, axis=1)), np.array(flags)

        def oracle_local(pk, fd, tg, clamp, method):
            res = [O.dv_field(P, boundary, fd.name, int(t)) for t in tg]
            vals = np.stack([r[0] for r in res], axis=1) if res else np.zeros((P.shape[0], 0))
            return torch.from_numpy(vals), np.array([bool(r[1]) for r in res], bool)

        par._compute_batch_slab = oracle_batch_slab
        par._local_batch = oracle_local
        bounds = par.partition_rows(P.shape[0], world)
        slab = _Slab(P, *bounds[rank])
        sf = par.ShardedField(slab, bounds, dist, device=torch.device("cpu"))
        rows = sf.target_rows(targets, P.shape[1]).numpy()
        q.put((rank, "rows", bool(np.array_equal(rows, P[targets]))))
        refs = [O.dv_field(P, boundary, "kl", int(t)) for t in targets]
        ref = np.stack([r[0] for r in refs], axis=1)
        rflags = np.array([bool(r[1]) for r in refs])
        full, flags = sf.field_batch(pf.builtin_f("kl"), targets, gather=True)
        q.put((rank, "rowsharded", bool(np.array_equal(full.numpy(), ref))
               and bool(np.array_equal(flags, rflags))))
        full2, flags2, _ = par.field_batch_by_targets(P, pf.builtin_f("kl"), targets, dist,
                                                      gather=True)
        q.put((rank, "by-targets", bool(np.array_equal(full2.numpy(), ref))
               and bool(np.array_equal(flags2, rflags))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_field_batch_gloo(world):
    from oracle.inputs import synthetic_kernel
    P = synthetic_kernel(61, 11, seed=10 + world)
    P[:, 0] = 0.0
    P[::9, 4] = 0.0          # interior rows with different zero patterns: flags differ by target
    boundary = np.array([3])
    targets = np.array([0, 9, 25, 60, 44, 18, 33])   # owners on every rank, odd count
    _run(world, _batch_worker, (P, boundary, targets), 3)


# ---------------------------------------------------------------------------
# distributed tracers (C5 on N ranks; the row-sharded single-target tracer)
# ---------------------------------------------------------------------------

def _oracle_paths(mesh, P, boundary, jobs):
    from oracle import divergence as O
    from oracle import tracer as OT
    topo = OT.topology(mesh.triangles, mesh.n)
    out = []
    for src, tgt in jobs:
        vals, _ = O.dv_field(P, boundary, "kl", int(tgt))
        out.append(OT.triangle_descent(mesh.vertices, mesh.triangles, mesh.areas,
                                       mesh.bbox_diagonal, vals, int(tgt), int(src), topo=topo))
    return out


def _same_path(a, b):
    return (a["status"] == b["status"] and a["locations"] == b["locations"]
            and np.array_equal(np.asarray(a["points"]), np.asarray(b["points"])))


def _trace_worker(rank, world, port, spec, P, boundary, targets, sources, field_of, q):
    _init(rank, world, port)
    try:
        from oracle import divergence as O
        from oracle import inputs as I
        from oracle import tracer as OT
        import paper_1708_02845_b200 as pf
        mesh = I.build(spec)
        topo = OT.topology(mesh.triangles, mesh.n)
        seen = []

        def oracle_trace(m, fields, fld_ld, vtx_ld, tg, src, fo, settings):
            flat = fields.reshape(-1).numpy() if fields.is_contiguous() else None
            assert flat is not None
            out = []
            for i, s0 in enumerate(src):
                f = 0 if fo is None else int(fo[i])
                vals = flat[f * fld_ld + np.arange(mesh.n) * vtx_ld]
                out.append(OT.triangle_descent(mesh.vertices, mesh.triangles, mesh.areas,
                                               mesh.bbox_diagonal, vals, int(tg[f]), int(s0),
                                               topo=topo))
            seen.append(len(src))
            return out

        def oracle_local(pk, fd, tg, clamp, method):
            res = [O.dv_field(P, boundary, fd.name, int(t)) for t in tg]
            vals = np.stack([r[0] for r in res], axis=1) if res else np.zeros((P.shape[0], 0))
            return torch.from_numpy(vals), np.array([bool(r[1]) for r in res], bool)

        _install_oracle_slab(P, boundary)
        par._trace_local = oracle_trace
        par._local_batch = oracle_local
        ref = _oracle_paths(mesh, P, boundary, [(s, targets[f]) for s, f in zip(sources, field_of)])
        allp = par.trace_batch(mesh, P, pf.builtin_f("kl"), targets, sources, field_of, dist,
                               gather_paths=True)
        q.put((rank, "c5", len(allp) == len(ref) and all(map(_same_path, allp, ref))))
        mine, own = par.trace_batch(mesh, P, pf.builtin_f("kl"), targets, sources, field_of, dist)
        a, b = par.partition_rows(len(targets), world)[rank]
        q.put((rank, "c5-owner", bool(np.all((field_of[mine] >= a) & (field_of[mine] < b)))
               and all(_same_path(x, ref[i]) for i, x in zip(mine, own))))
        bounds = par.partition_rows(P.shape[0], world)
        sf = par.ShardedField(_Slab(P, *bounds[rank]), bounds, dist, device=torch.device("cpu"))
        t0 = int(targets[0])
        src0 = sources[field_of == 0]
        ref0 = _oracle_paths(mesh, P, boundary, [(s, t0) for s in src0])
        got = sf.trace(mesh, pf.builtin_f("kl"), t0, src0, gather_paths=True)
        q.put((rank, "rowsharded-trace", all(map(_same_path, got, ref0))))
        from paper_1708_02845_b200.errors import InvalidTargetError
        try:
            par.trace_batch(mesh, P, pf.builtin_f("kl"), targets, [int(targets[0])], [0], dist)
            q.put((rank, "src==tgt", False))
        except InvalidTargetError:
            q.put((rank, "src==tgt", True))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_tracers_gloo(world):
    from tests.conftest import case
    c = case("disk8")
    P, boundary = c.dense, c.boundary
    interior = np.setdiff1d(np.arange(c.n), boundary)
    rng = np.random.default_rng(world)
    targets = rng.choice(interior, 5, replace=False)
    sources = rng.choice(interior, 17)
    field_of = np.arange(17) % 5
    sources = np.where(sources == targets[field_of], interior[0], sources)
    sources = np.where(sources == targets[field_of], interior[1], sources)
    _run(world, _trace_worker, (c.meta["spec"], P, boundary, targets, sources, field_of), 4,
         timeout=300)
