"""TEST SCAFFOLDING (not the product path): a dense numpy restatement of the plane-partitioned
cyclic reduction, the multi-worker orchestration of the
reference's execute_parallel_factor (proj/core/src/parallel.cpp:96-297), with
the block arithmetic abstracted behind a kernel and the mailbox replaced by a
point-to-point transport (torch.distributed: gloo on CPU in the tests, NCCL for GPU ranks).

Per level i (two phases, parallel.cpp:137-216):
  phase 1  owners invert their eliminated planes and send {E_j, Dinv_j, F_j, f_j} to
           the owner of each neighbour j-1 / j+1 that lives on another rank (one message
           per distinct destination);
  phase 2  owners of retained planes receive what they need and run eliminate_around +
           forward_rhs (acr.hpp:78-120).
Back substitution (parallel.cpp:252-292): owners of retained planes send u_j to the
owner of an eliminated neighbour; that owner recovers u_e = Dinv_e (f_e - E_e u_lo - F_e u_hi).
Every rank holds the same plan; the arithmetic per plane is unchanged, so results are
bitwise identical for every worker count (reference contract, test_parallel.cpp:75-89).
"""
from __future__ import annotations

import numpy as np

from paper_1701_00182_b200.plan import eliminated_positions, plan_schedule, retained_positions


class DenseKernel:
    """Exact dense block arithmetic (the reference's DenseKernel, acr.hpp:26-38)."""

    def invert(self, a, level, plane):
        return np.linalg.inv(a)

    def multiply(self, a, b):
        return a @ b

    def multiply_add(self, c, a, b, alpha):
        return c + alpha * (a @ b)

    def zeros_like(self, a):
        return np.zeros_like(a)

    def apply(self, a, x):
        return a @ x


def eliminate_around(k, Dj, Ej, Fj, Dlo, Elo, Flo, Dhi, Ehi, Fhi):
    D, En, Fn = Dj, None, None
    if Dlo is not None:
        T = k.multiply(Ej, Dlo)
        if Flo is not None:
            D = k.multiply_add(D, T, Flo, -1.0)
        if Elo is not None:
            En = k.multiply_add(k.zeros_like(Dj), T, Elo, -1.0)
    if Dhi is not None:
        T = k.multiply(Fj, Dhi)
        if Ehi is not None:
            D = k.multiply_add(D, T, Ehi, -1.0)
        if Fhi is not None:
            Fn = k.multiply_add(k.zeros_like(Dj), T, Fhi, -1.0)
    return D, En, Fn


def forward_rhs(k, fj, Ej, Dlo, flo, Fj, Dhi, fhi):
    out = fj.copy()
    if Dlo is not None and flo is not None:
        out = out - k.apply(Ej, k.apply(Dlo, flo))
    if Dhi is not None and fhi is not None:
        out = out - k.apply(Fj, k.apply(Dhi, fhi))
    return out


class Transport:
    """Point-to-point exchange; `send(obj, dst, tag)` / `recv(src, tag)`."""

    def __init__(self, rank, world, dist=None):
        self.rank, self.world, self.dist = rank, world, dist
        self.log = []

    def send(self, arrays, dst, tag):
        import torch
        self.log.append(("send", tag, dst, int(sum(a.nbytes for a in arrays))))
        for a in arrays:
            self.dist.send(torch.from_numpy(np.ascontiguousarray(a)), dst, tag=tag)

    def recv(self, shapes, src, tag):
        import torch
        out = []
        for shp in shapes:
            t = torch.empty(shp, dtype=torch.float64)
            self.dist.recv(t, src, tag=tag)
            out.append(t.numpy())
        self.log.append(("recv", tag, src, int(sum(a.nbytes for a in out))))
        return out


def partitioned_solve(D, E, F, f, plan, rank, transport=None, kernel=None):
    """Factor + solve the block-tridiagonal system (lists of dense numpy blocks; E[j]
    couples j->j-1 (E[0] None), F[j] couples j->j+1 (F[n-1] None)) on `rank` of the
    plan.  Returns {plane: u_plane} for the planes this rank owns at level 0, and the
    message ledger [(level, from_plane, to_plane, bytes, solve_phase)]."""
    k = kernel or DenseKernel()
    n = len(D)
    d = D[0].shape[0]
    owner = lambda lvl, j: plan.assignment[lvl][j]
    mine = {j: dict(D=D[j], E=E[j], F=F[j], f=f[j]) for j in range(n) if owner(0, j) == rank}
    ledger = []
    levels = []
    m = n
    lvl = 0
    while m > 1:
        elim = eliminated_positions(m)
        ret = retained_positions(m)
        is_elim = set(elim)
        Lv = {"m": m, "elim": elim, "ret": ret, "Dinv": {}, "E": {}, "F": {}, "f": {}}
        # phase 1: invert owned eliminated planes and post payloads
        for j, pl in mine.items():
            Lv["E"][j], Lv["F"][j] = pl["E"], pl["F"]
            if j in is_elim:
                Lv["Dinv"][j] = k.invert(pl["D"], lvl, j)
                Lv["f"][j] = pl["f"]
        for j in sorted(mine):
            if j not in is_elim:
                continue
            dests = []
            for nb in (j - 1, j + 1):
                if 0 <= nb < m and owner(lvl, nb) != rank and owner(lvl, nb) not in dests:
                    dests.append(owner(lvl, nb))
                    pl = mine[j]
                    flags = np.array([pl["E"] is not None, pl["F"] is not None], np.float64)
                    payload = [flags, Lv["Dinv"][j], pl["f"],
                               pl["E"] if pl["E"] is not None else np.zeros((d, d)),
                               pl["F"] if pl["F"] is not None else np.zeros((d, d))]
                    ledger.append((lvl, j, nb, int(sum(a.nbytes for a in payload)), False))
                    transport.send(payload, owner(lvl, nb), tag=(lvl << 20) | j)
        # phase 2: gather eliminated neighbours and update owned retained planes
        got = {}

        def neighbour(e):
            if e < 0 or e >= m or e not in is_elim:
                return None
            if e not in got:
                if owner(lvl, e) == rank:
                    got[e] = (Lv["Dinv"][e], Lv["E"].get(e), Lv["F"].get(e), Lv["f"][e])
                else:
                    flags, dinv, fe, Ee, Fe = transport.recv([(2,), (d, d), (d,), (d, d), (d, d)],
                                                             owner(lvl, e), tag=(lvl << 20) | e)
                    got[e] = (dinv, Ee if flags[0] else None, Fe if flags[1] else None, fe)
            return got[e]

        nxt = {}
        for t, j in enumerate(ret):
            if owner(lvl, j) != rank:
                continue
            pl = mine[j]
            lo, hi = neighbour(j - 1), neighbour(j + 1)
            Dn, En, Fn = eliminate_around(k, pl["D"], pl["E"], pl["F"],
                                          lo[0] if lo else None, lo[1] if lo else None, lo[2] if lo else None,
                                          hi[0] if hi else None, hi[1] if hi else None, hi[2] if hi else None)
            if En is None and t > 0 and ret[t - 1] == j - 1:
                En = pl["E"]
            if Fn is None and t + 1 < len(ret) and ret[t + 1] == j + 1:
                Fn = pl["F"]
            fn = forward_rhs(k, pl["f"], pl["E"], lo[0] if lo else None, lo[3] if lo else None,
                             pl["F"], hi[0] if hi else None, hi[3] if hi else None)
            nxt[t] = dict(D=Dn, E=En, F=Fn, f=fn)
        levels.append(Lv)
        mine = nxt
        m = len(ret)
        lvl += 1
    # apex: one plane
    u = {}
    if 0 in mine:
        apex_inv = k.invert(mine[0]["D"], lvl, 0)
        u[0] = k.apply(apex_inv, mine[0]["f"])
    # back substitution, top level down
    for li in range(len(levels) - 1, -1, -1):
        Lv = levels[li]
        m, elim, ret = Lv["m"], Lv["elim"], Lv["ret"]
        is_elim = set(elim)
        ul = {ret[t]: v for t, v in u.items()}
        for j in sorted(ul):
            for nb in (j - 1, j + 1):
                if 0 <= nb < m and nb in is_elim and owner(li, nb) != rank:
                    ledger.append((li, j, nb, int(ul[j].nbytes), True))
                    transport.send([ul[j]], owner(li, nb), tag=(1 << 30) | (li << 20) | j)
        cache = {}

        def neighbour_u(j):
            if owner(li, j) == rank:
                return ul[j]
            if j not in cache:
                cache[j] = transport.recv([(d,)], owner(li, j), tag=(1 << 30) | (li << 20) | j)[0]
            return cache[j]

        for e in elim:
            if owner(li, e) != rank:
                continue
            r = Lv["f"][e].copy()
            if e > 0 and Lv["E"].get(e) is not None:
                r = r - k.apply(Lv["E"][e], neighbour_u(e - 1))
            if e + 1 < m and Lv["F"].get(e) is not None:
                r = r - k.apply(Lv["F"][e], neighbour_u(e + 1))
            ul[e] = k.apply(Lv["Dinv"][e], r)
        u = {j: v for j, v in ul.items() if owner(li, j) == rank}
    return u, ledger
