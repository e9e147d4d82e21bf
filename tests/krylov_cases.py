"""Shared cases of the reference Krylov tests (proj/tests/test_krylov.cpp), used by the
oracle (CPU) and GPU test modules."""
import dataclasses

import numpy as np

from paper_1701_00182_b200 import problems as P


def negated(sysm):
    """The operator with every entry negated (test_krylov.cpp:137-150)."""
    return dataclasses.replace(sysm, vals=-np.asarray(sysm.vals))


def zero_rhs_system():
    """identity planes with a zero right-hand side (test_krylov.cpp:41-55)."""
    return P.identity_system(4, 16, np.zeros((1, 4, 16)))


def indefinite_system():
    """Helmholtz beyond the first resonance (test_krylov.cpp:57-61): 7-point, n=8,
    omega = 12 (omega^2 h^2 = 1.78 > 3 * 4 sin^2(pi h / 2) = 0.36)."""
    return P.helmholtz7(8, 2024, omega=12.0)


def ratio_variance(h):
    ratios = [h[k] / h[k - 1] for k in range(1, len(h)) if h[k - 1] > 0]
    if not ratios:
        return 0.0
    m = sum(ratios) / len(ratios)
    return sum((r - m) ** 2 for r in ratios) / len(ratios)
