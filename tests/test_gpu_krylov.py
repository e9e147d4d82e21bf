"""GPU Krylov drivers (acrgpu_pcg / acrgpu_refine through the C-ABI) on the reference's
test_krylov.cpp cases, checked against the CPU oracle's restatement (oracle/krylov.py)
on the same systems: convergence flags exactly, iteration counts within +-1 (the GPU and
oracle preconditioners agree to the parity bar, not bitwise), final residuals below tol.
The reference's exact Dense-mode preconditioner is replaced on the GPU by an H-mode
factorization at eps 1e-12 (the GPU path is H-mode only)."""
import numpy as np
import pytest

from krylov_cases import indefinite_system, negated, ratio_variance, zero_rhs_system
from paper_1701_00182_b200 import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def acr():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1701_00182_b200 import acr as A
    A.lib()
    return A


@pytest.fixture(scope="module")
def K():
    from oracle import krylov
    return krylov


def near_exact(acr, sysm):
    return acr.acr_factor(sysm, acr.AcrConfig(eps=1e-12))


def test_pcg_near_exact_preconditioner(acr):                                     # test_krylov.cpp:20-27
    sysm = P.poisson(8)
    res = acr.pcg(sysm, near_exact(acr, sysm), 1e-10, 50)
    assert res.trace.converged and res.trace.iterations <= 2
    assert sysm.relative_residual(res.u) <= 1e-10


def test_preconditioning_reduces_iterations_vs_oracle(acr, oracle, K):           # test_krylov.cpp:29-39
    sysm = P.poisson(16)
    plain = acr.pcg(sysm, None, 1e-6, 500)
    pre = acr.pcg(sysm, acr.acr_factor(sysm, acr.AcrConfig(eps=1e-2)), 1e-6, 500)
    assert plain.trace.converged and pre.trace.converged
    assert pre.trace.iterations < plain.trace.iterations
    _, o_plain = K.pcg(sysm, None, 1e-6, 500)
    _, o_pre = K.pcg(sysm, oracle.Factorization(sysm, eps=1e-2, threads=8), 1e-6, 500)
    assert abs(plain.trace.iterations - o_plain.iterations) <= 1
    assert abs(pre.trace.iterations - o_pre.iterations) <= 1
    np.testing.assert_allclose(plain.trace.residual_history[:5], o_plain.residual_history[:5], rtol=1e-8)


def test_zero_rhs(acr):                                                          # test_krylov.cpp:41-55
    sysm = zero_rhs_system()
    res = acr.pcg(sysm, None, 1e-8, 10)
    assert res.trace.converged and res.trace.iterations == 0 and np.linalg.norm(res.u) == 0.0
    res = acr.iterative_refinement(sysm, near_exact(acr, sysm), 1e-8, 10)
    assert res.trace.converged and res.trace.iterations == 0 and np.linalg.norm(res.u) == 0.0


def test_pcg_indefinite(acr):                                                    # test_krylov.cpp:57-61
    with pytest.raises(acr.IndefiniteError):
        acr.pcg(indefinite_system(), None, 1e-8, 200)


def test_history_tracks_true_residual(acr):                                      # test_krylov.cpp:63-91
    sysm = P.poisson(8)
    M = acr.acr_factor(sysm, acr.AcrConfig(eps=1e-2))
    res = acr.pcg(sysm, M, 1e-8, 100)
    tr = res.trace
    assert tr.converged and len(tr.residual_history) == tr.iterations
    assert tr.residual_history[-1] <= 1e-8
    assert sysm.relative_residual(res.u) == pytest.approx(tr.residual_history[-1], rel=1e-6)
    assert tr.total_time >= 0.0 and tr.apply_time > 0.0
    h = acr.pcg(sysm, M, 1e-12, 100).trace.residual_history
    assert all(h[k] <= 1.2 * h[k - 1] for k in range(1, len(h)))


def test_refinement_vs_oracle(acr, oracle, K):                                   # test_krylov.cpp:93-121
    sysm = P.poisson(8)
    tr = acr.iterative_refinement(sysm, near_exact(acr, sysm), 1e-10, 10).trace
    assert tr.converged and tr.iterations == 1
    sysm = P.poisson(16)
    res = acr.iterative_refinement(sysm, acr.acr_factor(sysm, acr.AcrConfig(eps=1e-2)), 1e-10, 50)
    assert res.trace.converged and sysm.relative_residual(res.u) <= 1e-10
    assert ratio_variance(res.trace.residual_history) < 0.5
    _, o = K.iterative_refinement(sysm, oracle.Factorization(sysm, eps=1e-2, threads=8), 1e-10, 50)
    assert abs(res.trace.iterations - o.iterations) <= 1


def test_refinement_nonsymmetric(acr):                                           # test_krylov.cpp:123-133
    sysm = P.convdiff_upwind(8, 2024)
    res = acr.iterative_refinement(sysm, acr.acr_factor(sysm, acr.AcrConfig(eps=1e-3)), 1e-10, 50)
    assert res.trace.converged
    exact = np.linalg.solve(sysm.to_dense(), sysm.rhs[0].ravel()).reshape(res.u.shape)
    assert np.linalg.norm(res.u - exact) <= 1e-8 * np.linalg.norm(exact)


def test_refinement_divergence(acr):                                             # test_krylov.cpp:135-153
    sysm = P.poisson(4)
    bad = near_exact(acr, negated(sysm))
    with pytest.raises(acr.DivergenceError):
        acr.iterative_refinement(sysm, bad, 1e-12, 50)


def test_nonconvergence_in_trace(acr):                                           # test_krylov.cpp:155-160
    tr = acr.pcg(P.poisson(16), None, 1e-14, 3).trace
    assert not tr.converged and tr.iterations == 3


def test_config2_loose_factorization_pcg(acr):
    """The paper's time-to-solution mode at BASELINE config 2 size: a loose
    eps 1e-2 H-factorization as the preconditioner of CG to 1e-10."""
    sysm = P.config_system(2)
    M = acr.acr_factor(sysm, acr.AcrConfig(eps=1e-2))
    res = acr.pcg(sysm, M, 1e-10, 200)
    assert res.trace.converged and res.trace.iterations <= 60
    assert sysm.relative_residual(res.u) <= 1e-10
