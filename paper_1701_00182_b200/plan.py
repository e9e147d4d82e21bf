"""Plane-partition schedule for multi-GPU ACR (reference proj/core/src/parallel.cpp:383-414).

``plan_schedule(n, p)`` assigns contiguous plane ranges to p workers (GPUs) at
level 0; retained planes inherit their owner at every later level, so past the
C-level (log2(n/p)) the number of active workers halves per level.
"""
from __future__ import annotations

import dataclasses


def _pow2(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


def eliminated_positions(m: int) -> list[int]:
    """Even positions; an odd count carries the trailing plane (acr.cpp:46-51)."""
    v = list(range(0, m, 2))
    if m % 2 == 1 and v:
        v.pop()
    return v


def retained_positions(m: int) -> list[int]:
    v = list(range(1, m, 2))
    if m % 2 == 1:
        v.append(m - 1)
    return v


@dataclasses.dataclass
class ParallelPlan:
    p: int
    n_planes: int
    c_level: int
    assignment: list  # per level: plane -> worker


def plan_schedule(n_planes: int, p: int) -> ParallelPlan:
    if not _pow2(n_planes) or not _pow2(p):
        raise ValueError("plan_schedule: plane and worker counts must be powers of two")
    if p > n_planes:
        raise ValueError("plan_schedule: more workers than planes")
    per = n_planes // p
    cur = [j // per for j in range(n_planes)]
    plan = ParallelPlan(p, n_planes, (n_planes // p).bit_length() - 1, [cur])
    while len(cur) > 1:
        cur = [cur[t] for t in retained_positions(len(cur))]
        plan.assignment.append(cur)
    return plan


def critical_path_length(plan: ParallelPlan) -> int:
    total = 0
    for i in range(plan.c_level):
        planes = plan.n_planes >> (i + 1)
        total += (planes + plan.p - 1) // plan.p
    return total + (plan.p.bit_length() - 1)


def messages(plan: ParallelPlan):
    """Cross-worker payloads per level (parallel.cpp:142-161, 264-274):
    factor phase: eliminated plane j -> owner of j+-1 (one per distinct dest);
    solve phase: retained plane j -> owner of eliminated neighbour."""
    out = []
    for lvl, own in enumerate(plan.assignment[:-1]):
        m = len(own)
        elim = set(eliminated_positions(m))
        fac, sol = [], []
        for j in sorted(elim):
            dests = set()
            for nb in (j - 1, j + 1):
                if 0 <= nb < m and own[nb] != own[j] and own[nb] not in dests:
                    dests.add(own[nb])
                    fac.append((lvl, j, nb))
        for j in range(m):
            if j in elim:
                continue
            for nb in (j - 1, j + 1):
                if 0 <= nb < m and nb in elim and own[nb] != own[j]:
                    sol.append((lvl, j, nb))
        out.append((fac, sol))
    return out
