"""CPU oracle (TEST INFRASTRUCTURE ONLY): restatement of the reference Krylov drivers,
core/src/krylov.cpp:38-133 (pcg, iterative_refinement) with IterationTrace semantics
of core/include/acr/krylov.hpp:8-35, in numpy.  The operator is System.apply
(block.cpp:89-107) and the preconditioner an oracle Factorization's solve (or None for
plain CG).  Only tests/ and bench.py's CPU leg may import this module.
"""
from __future__ import annotations

import dataclasses
import time

import numpy as np


class IndefiniteError(RuntimeError):
    pass


class DivergenceError(RuntimeError):
    pass


@dataclasses.dataclass
class Trace:
    converged: bool = False
    iterations: int = 0
    residual_history: list = dataclasses.field(default_factory=list)
    apply_time: float = 0.0
    total_time: float = 0.0


def _rhs(system):
    return np.asarray(system.rhs, np.float64).reshape(-1, system.n, system.dim)[0].ravel()


def _apply(system, x):
    return system.apply(x.reshape(system.n, system.dim)).ravel()


def pcg(system, precond, tol, max_iterations):
    """krylov.cpp:38-90: returns (u (n, dim), Trace)."""
    b = _rhs(system)
    bnorm = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    tr = Trace()
    if bnorm == 0.0:
        tr.converged = True
        return x.reshape(system.n, system.dim), tr
    t0 = time.perf_counter()
    apply_s, applies = 0.0, 0

    def M(v):
        nonlocal apply_s, applies
        if precond is None:
            return v.copy()
        t = time.perf_counter()
        out = precond.solve(v.reshape(system.n, system.dim)).ravel()
        apply_s += time.perf_counter() - t
        applies += 1
        return out

    r = b.copy()
    z = M(r)
    p = z.copy()
    rz = float(r @ z)
    for k in range(1, max_iterations + 1):
        Ap = _apply(system, p)
        pAp = float(p @ Ap)
        if not pAp > 0:
            raise IndefiniteError(f"conjugate gradient: nonpositive curvature p^T A p = {pAp}")
        alpha = rz / pAp
        x += alpha * p
        r -= alpha * Ap
        true_res = float(np.linalg.norm(b - _apply(system, x))) / bnorm
        tr.residual_history.append(true_res)
        tr.iterations = k
        if true_res <= tol:
            tr.converged = True
            break
        z = M(r)
        rz_next = float(r @ z)
        p = z + (rz_next / rz) * p
        rz = rz_next
    tr.total_time = time.perf_counter() - t0
    if applies:
        tr.apply_time = apply_s / applies
    return x.reshape(system.n, system.dim), tr


def iterative_refinement(system, precond, tol, max_iterations):
    """krylov.cpp:92-131: returns (u (n, dim), Trace)."""
    b = _rhs(system)
    bnorm = float(np.linalg.norm(b))
    x = np.zeros_like(b)
    tr = Trace()
    if bnorm == 0.0:
        tr.converged = True
        return x.reshape(system.n, system.dim), tr
    t0 = time.perf_counter()
    prev, growth = 1.0, 0
    for k in range(1, max_iterations + 1):
        r = b - _apply(system, x)
        x += precond.solve(r.reshape(system.n, system.dim)).ravel()
        res = float(np.linalg.norm(b - _apply(system, x))) / bnorm
        tr.residual_history.append(res)
        tr.iterations = k
        if res <= tol:
            tr.converged = True
            break
        growth = growth + 1 if res > prev else 0
        if growth >= 3:
            raise DivergenceError(f"iterative refinement: residual grew over three consecutive corrections (last {res})")
        prev = res
    tr.total_time = time.perf_counter() - t0
    return x.reshape(system.n, system.dim), tr
