"""numpy execution of the device multifrontal Poisson solver, step for step.

Test infrastructure only: it runs the host plan (nd_plan.cpp) with the same
front assembly, partial Cholesky, tile-sparse forward solve and backward
solve as csrc/poisson.cu, in dense numpy per front, so the plan (orderings,
R sets, scatter maps, active tiles) is checked on CPU against a direct
scipy solve of the reference system (solvers.py:278-303).
"""

from __future__ import annotations

import numpy as np


def laplacian_parts(lc, nb_ptr, nb_idx):
    """(off, diag): lc's off-diagonal values in neighbour-CSR order, and its diagonal."""
    n = lc.shape[0]
    off = np.empty(len(nb_idx))
    for v in range(n):
        a, b = lc.indptr[v], lc.indptr[v + 1]
        cols, vals = lc.indices[a:b], lc.data[a:b]
        keep = cols != v
        assert np.array_equal(cols[keep], nb_idx[nb_ptr[v]:nb_ptr[v + 1]])
        off[nb_ptr[v]:nb_ptr[v + 1]] = vals[keep]
    return off, lc.diagonal().copy()


def factor(plan, off, diag):
    F = np.zeros(plan.stats["f_total"])
    for level in plan.levels:
        for s in level:
            f, c = int(plan.fn[s]), int(plan.cn[s])
            Fs = F[plan.foff[s]:plan.foff[s] + f * f].reshape(f, f)
            Fs[:] = 0.0
            a0, a1 = plan.a_ptr[s], plan.a_ptr[s + 1]
            src = plan.a_src[a0:a1]
            vals = np.where(src >= 0, -off[np.maximum(src, 0)], -diag[np.maximum(-1 - src, 0)])
            F[plan.a_dst[a0:a1]] = vals
            for ch in plan.ch_idx[plan.ch_ptr[s]:plan.ch_ptr[s + 1]]:
                fc, cc, rc = int(plan.fn[ch]), int(plan.cn[ch]), int(plan.rn[ch])
                U = F[plan.foff[ch]:plan.foff[ch] + fc * fc].reshape(fc, fc)[cc:, cc:]
                mp = plan.relmap[plan.relmap_off[ch]:plan.relmap_off[ch] + rc]
                Fs[np.ix_(mp, mp)] += np.tril(U)
            if c:
                low = np.tril(Fs)
                sym = low + np.tril(low, -1).T
                Lcc = np.linalg.cholesky(sym[:c, :c])
                Lrc = np.linalg.solve(Lcc, sym[c:, :c].T).T
                Fs[:c, :c] = Lcc
                Fs[c:, :c] = Lrc
                Fs[c:, c:] = np.tril(sym[c:, c:] - Lrc @ Lrc.T)
    return F


def solve(plan, F, off, k, ld=None, need=None):
    """Forward (tile-sparse, one f x tile [Y_C; V] block per active item) +
    backward into P rows.  `need` (bool per front) restricts the backward to
    those fronts, as a row-slab build does: the rows of the other fronts stay
    NaN, so a slab that read one of them shows it."""
    n, T = plan.n, plan.tile
    P = np.zeros((n, k))
    V = np.zeros(plan.stats["v_total"])
    touched = np.zeros((n, plan.ntiles), dtype=bool)
    for level in plan.levels:
        for s in level:
            f, c, r = int(plan.fn[s]), int(plan.cn[s]), int(plan.rn[s])
            Fs = F[plan.foff[s]:plan.foff[s] + f * f].reshape(f, f)
            Crows = plan.perm_orig[plan.c0[s]:plan.c0[s] + c]
            for it in range(plan.act_ptr[s], plan.act_ptr[s + 1]):
                t = int(plan.act_tile[it])
                j0, j1 = t * T, min(k, t * T + T)
                W = np.zeros((f, T))
                b0, b1 = plan.b_ptr[s], plan.b_ptr[s + 1]
                for e in range(b0, b1):
                    col = int(plan.b_col[e])
                    if j0 <= col < j1:
                        W[plan.b_row[e], col - j0] = off[plan.b_src[e]]
                for ch in plan.ch_idx[plan.ch_ptr[s]:plan.ch_ptr[s + 1]]:
                    ic = plan.tile_item[ch * plan.ntiles + t]
                    if ic < 0:
                        continue
                    rc, fc, cc = int(plan.rn[ch]), int(plan.fn[ch]), int(plan.cn[ch])
                    Vc = V[plan.act_voff[ic]:plan.act_voff[ic] + fc * T].reshape(fc, T)[cc:]
                    mp = plan.relmap[plan.relmap_off[ch]:plan.relmap_off[ch] + rc]
                    W[mp] += Vc
                Y = np.linalg.solve(np.tril(Fs[:c, :c]), W[:c]) if c else W[:0]
                W[c:] -= Fs[c:, :c] @ Y
                P[Crows, j0:j1] = Y[:, :j1 - j0]
                touched[Crows, t] = True
                W[:c] = Y
                V[plan.act_voff[it]:plan.act_voff[it] + f * T] = W.ravel()  # [Y_C; V]
    if need is not None:  # forget what the slab's backward does not compute
        for s in np.flatnonzero(~need):
            P[plan.perm_orig[plan.c0[s]:plan.c0[s] + plan.cn[s]]] = np.nan
    for level in reversed(plan.levels):
        for s in level:
            f, c, r = int(plan.fn[s]), int(plan.cn[s]), int(plan.rn[s])
            if not c or (need is not None and not need[s]):
                continue
            Fs = F[plan.foff[s]:plan.foff[s] + f * f].reshape(f, f)
            Crows = plan.perm_orig[plan.c0[s]:plan.c0[s] + c]
            Rrows = plan.r_orig[plan.r_ptr[s]:plan.r_ptr[s + 1]]
            Z = P[Crows] - Fs[c:, :c].T @ P[Rrows]
            P[Crows] = np.linalg.solve(np.tril(Fs[:c, :c]).T, Z)
    return P
