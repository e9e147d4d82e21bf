"""The CPU oracle's Krylov drivers (oracle/krylov.py) against the reference's own
test_krylov.cpp cases.  The oracle is the checker for the GPU drivers
(tests/test_gpu_krylov.py)."""
import numpy as np
import pytest

from oracle import krylov as K
from paper_1701_00182_b200 import problems as P
from krylov_cases import indefinite_system, negated, ratio_variance, zero_rhs_system


def test_pcg_exact_preconditioner_two_iterations(oracle):                        # test_krylov.cpp:20-27
    sysm = P.poisson(8)
    M = oracle.Factorization(sysm, mode="dense")
    u, tr = K.pcg(sysm, M, 1e-10, 50)
    assert tr.converged and tr.iterations <= 2
    assert sysm.relative_residual(u) <= 1e-10


def test_preconditioning_reduces_iterations(oracle):                             # test_krylov.cpp:29-39
    sysm = P.poisson(16)
    _, plain = K.pcg(sysm, None, 1e-6, 500)
    M = oracle.Factorization(sysm, eps=1e-2, threads=4)
    _, pre = K.pcg(sysm, M, 1e-6, 500)
    assert plain.converged and pre.converged
    assert pre.iterations < plain.iterations


def test_zero_rhs(oracle):                                                       # test_krylov.cpp:41-55
    sysm = zero_rhs_system()
    u, tr = K.pcg(sysm, None, 1e-8, 10)
    assert tr.converged and tr.iterations == 0 and np.linalg.norm(u) == 0.0
    M = oracle.Factorization(sysm, mode="dense")
    u, tr = K.iterative_refinement(sysm, M, 1e-8, 10)
    assert tr.converged and tr.iterations == 0 and np.linalg.norm(u) == 0.0


def test_pcg_indefinite():                                                       # test_krylov.cpp:57-61
    with pytest.raises(K.IndefiniteError):
        K.pcg(indefinite_system(), None, 1e-8, 200)


def test_history_tracks_true_residual(oracle):                                   # test_krylov.cpp:63-78
    sysm = P.poisson(8)
    M = oracle.Factorization(sysm, eps=1e-2)
    u, tr = K.pcg(sysm, M, 1e-8, 100)
    assert tr.converged and len(tr.residual_history) == tr.iterations
    assert tr.residual_history[-1] <= 1e-8
    assert sysm.relative_residual(u) == pytest.approx(tr.residual_history[-1], rel=1e-6)
    h = K.pcg(sysm, M, 1e-12, 100)[1].residual_history                          # test_krylov.cpp:80-91
    assert all(h[k] <= 1.2 * h[k - 1] for k in range(1, len(h)))


def test_refinement(oracle):                                                     # test_krylov.cpp:93-121
    sysm = P.poisson(8)
    _, tr = K.iterative_refinement(sysm, oracle.Factorization(sysm, mode="dense"), 1e-10, 10)
    assert tr.converged and tr.iterations == 1
    sysm = P.poisson(16)
    u, tr = K.iterative_refinement(sysm, oracle.Factorization(sysm, eps=1e-2, threads=4), 1e-10, 50)
    assert tr.converged and sysm.relative_residual(u) <= 1e-10
    assert ratio_variance(tr.residual_history) < 0.5


def test_refinement_nonsymmetric(oracle):                                        # test_krylov.cpp:123-133
    sysm = P.convdiff_upwind(8, 2024)
    u, tr = K.iterative_refinement(sysm, oracle.Factorization(sysm, eps=1e-3), 1e-10, 50)
    assert tr.converged
    exact = np.linalg.solve(sysm.to_dense(), sysm.rhs[0].ravel()).reshape(u.shape)
    assert np.linalg.norm(u - exact) <= 1e-8 * np.linalg.norm(exact)


def test_refinement_divergence(oracle):                                          # test_krylov.cpp:135-153
    sysm = P.poisson(4)
    bad = oracle.Factorization(negated(sysm), mode="dense")
    with pytest.raises(K.DivergenceError):
        K.iterative_refinement(sysm, bad, 1e-12, 50)


def test_nonconvergence_in_trace():                                              # test_krylov.cpp:155-160
    _, tr = K.pcg(P.poisson(16), None, 1e-14, 3)
    assert not tr.converged and tr.iterations == 3
