"""Multi-process (world_size 2, gloo, CPU) checks of the row-sharding host logic.

The slab computation is swapped for the CPU oracle inside these tests only
(the product's _compute_slab always runs the CUDA kernels); what is under
test is partitioning, ownership, the target-row broadcast and the
variable-size all-gather that assemble the N-rank field.
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


def _worker(rank, world, port, P, boundary, target, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import divergence as O
        import paper_1708_02845_b200 as pf

        def oracle_slab(slab, fd, p, row, clamp=None):
            full = np.vstack([row.numpy()[None, :], slab.P.numpy()])
            vals = O.dv_at(full, fd.name, 0, np.arange(1, slab.rows + 1))
            vals[np.arange(slab.row0, slab.row0 + slab.rows) == p] = 0.0
            return torch.from_numpy(vals)

        def oracle_sparse_slab(slab, fd, p, payload, cut, strict):
            full = np.vstack([P[p][None, :], slab.P.numpy()])  # restated from the dense rows
            vals = np.array([O.dv_pair_sparse_direct(P, p, q, fd.name)[0]
                             for q in range(slab.row0, slab.row0 + slab.rows)])
            return torch.from_numpy(vals)

        def oracle_tv_prep(slab, cut, strict, p, payload):
            payload.fill_(float(p))  # any owner-computed payload: checks the broadcast path

        par._compute_slab = oracle_slab
        par._compute_sparse_slab = oracle_sparse_slab
        par._sparse_tv_prep = oracle_tv_prep
        bounds = par.partition_rows(P.shape[0], world)
        slab = _Slab(P, *bounds[rank])
        sf = par.ShardedField(slab, bounds, dist, device=torch.device("cpu"))
        row = sf.target_row(target, P.shape[1])
        assert np.array_equal(row.numpy(), P[target])
        for g in ("kl", "tv"):
            full = sf.field(pf.builtin_f(g), target, gather=True).numpy()
            ref, _ = O.dv_field(P, boundary, g, target)
            q.put((rank, g, bool(np.array_equal(full, ref))))
            sp = sf.sparse_field(pf.builtin_f(g), target, gather=True).numpy()
            sref = np.array([O.dv_pair_sparse_direct(P, target, qq, g)[0] for qq in range(P.shape[0])])
            q.put((rank, "sparse-" + g, bool(np.array_equal(sp, sref))))
    finally:
        dist.destroy_process_group()


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_field_gloo(world):
    from oracle.inputs import synthetic_kernel
    P = synthetic_kernel(101, 13, seed=world)
    P[:, 0] = 0.0
    boundary = np.array([3])
    target = 77  # owned by the last rank: exercises a non-zero broadcast source
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, P, boundary, target, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(4 * world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, _, ok in res), res


def _batch_worker(rank, world, port, P, boundary, targets, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
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
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_batch_worker, args=(r, world, port, P, boundary, targets, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(3 * world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, _, ok in res), res
