"""Pins the CPU oracle's ACR factor/solve to the reference's own tests
(proj/tests/test_acr.cpp, test_parallel.cpp, test_acceptance.cpp)."""
import numpy as np
import pytest

from paper_1701_00182_b200 import problems as P
from paper_1701_00182_b200.plan import plan_schedule, critical_path_length


def lu_solve(sysm):
    return np.linalg.solve(sysm.to_dense(), sysm.rhs[0].ravel()).reshape(sysm.n, sysm.dim)


def rel(a, b):
    return np.linalg.norm(a.ravel() - b.ravel()) / np.linalg.norm(b.ravel())


@pytest.mark.parametrize("n", [4, 8])
def test_dense_mode_matches_lu(oracle, n):                                              # test_acr.cpp:112-124
    for sysm in (P.poisson(n), P.config_system(2, n=n), P.config_system(3, n=n), P.config_system(4, n=n)):
        u = oracle.Factorization(sysm, mode="dense").solve()
        assert sysm.relative_residual(u) <= 1e-9
        assert rel(u, lu_solve(sysm)) <= 1e-8


@pytest.mark.parametrize("n", [3, 5, 6, 7])
def test_non_power_of_two_planes(oracle, n):                                            # test_acr.cpp:204-211
    sysm = P.poisson(n)
    u = oracle.Factorization(sysm, mode="dense").solve()
    assert sysm.relative_residual(u) <= 1e-9
    assert rel(u, lu_solve(sysm)) <= 1e-8


def test_early_stop(oracle):                                                            # test_acr.cpp:213-221
    sysm = P.poisson(8)
    for stop in (1, 2, 3, 4):
        u = oracle.Factorization(sysm, mode="dense", stop_planes=stop).solve()
        assert sysm.relative_residual(u) <= 1e-9


def test_identity_system(oracle):                                                       # test_acr.cpp:138-146
    f = P.uniform_pm1(40, 1, 4 * 16).reshape(4, 16)
    sysm = P.identity_system(4, 16, f)
    u = oracle.Factorization(sysm, mode="dense").solve()
    assert np.linalg.norm(u - f) <= 1e-14


def test_multi_rhs_bitwise(oracle):                                                     # test_acr.cpp:148-163
    sysm = P.poisson(8)
    f1 = oracle.Factorization(sysm, mode="dense")
    g = P.uniform_pm1(60, 1, 8 * 64).reshape(8, 64)
    u1, u2 = f1.solve(sysm.rhs[0]), f1.solve(g)
    f2 = oracle.Factorization(sysm, mode="dense")
    assert np.array_equal(u1, f2.solve(sysm.rhs[0])) and np.array_equal(u2, f2.solve(g))
    assert np.array_equal(f1.solve(g), u2)
    both = f1.solve(np.stack([sysm.rhs[0], g]))
    assert np.array_equal(both[0], u1) and np.array_equal(both[1], u2)


def test_singular_pivot_location(oracle):                                               # test_acr.cpp:223-241
    n, d = 4, 4
    coords = np.stack([np.arange(d) % 2, np.arange(d) // 2], 1).astype(float)
    I = (np.arange(d, dtype=np.int32), np.arange(d, dtype=np.int32), np.ones(d))
    Z = (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0))
    blocks = [I, I, Z, I] + [Z] * 6
    sysm = P._assemble(n, d, coords, blocks, np.ones((1, n, d)))
    with pytest.raises(oracle.OracleError) as ei:
        oracle.Factorization(sysm, mode="dense")
    assert ei.value.code == 2 and ei.value.level == 0 and ei.value.plane == 2


def test_hmode_n16_accuracy(oracle):                                                    # test_acr.cpp:243-257
    sysm = P.poisson(16)
    f = oracle.Factorization(sysm, eps=1e-3, threads=4)
    u = f.solve()
    assert sysm.relative_residual(u) <= 1e-2
    st = f.stats()
    assert 1 <= st["largest_rank"] <= 12
    assert st["largest_rank"] >= st["average_rank"]
    assert st["factor_bytes"] > 0
    assert f.level_info()[0]["plane_count"] == 16


def test_residual_monotone_in_eps(oracle):                                              # test_acr.cpp:259-270
    sysm = P.poisson(16)
    prev = 1e9
    for eps in (1e-1, 1e-2, 1e-3, 1e-4):
        r = sysm.relative_residual(oracle.Factorization(sysm, eps=eps, threads=4).solve())
        assert r <= prev * 1.0001
        prev = r


def test_solve_shape_validation(oracle):                                                # test_acr.cpp:272-279
    f = oracle.Factorization(P.poisson(4), mode="dense")
    with pytest.raises(oracle.OracleError):
        f.solve(np.zeros((3, 16)))
    with pytest.raises(oracle.OracleError):
        f.solve(np.zeros((4, 9)))


def test_invalid_config(oracle):                                                        # test_acr.cpp:281-286
    with pytest.raises(oracle.OracleError) as ei:
        oracle.Factorization(P.poisson(4), mode="dense", stop_planes=0)
    assert ei.value.code == 4


def test_threads_bitwise(oracle):                                                       # test_parallel.cpp:75-89
    sysm = P.poisson(16)
    base = oracle.Factorization(sysm, eps=1e-3, threads=1)
    u0 = base.solve()
    for th in (2, 4, 8):
        assert np.array_equal(oracle.Factorization(sysm, eps=1e-3, threads=th).solve(), u0)


def test_plan_schedule_pins():                                                          # test_parallel.cpp:23-64
    plan = plan_schedule(16, 4)
    assert plan.c_level == 2
    assert [plan.assignment[0][j] for j in range(16)] == [j // 4 for j in range(16)]
    for lvl, exp in enumerate([4, 2, 1, 1]):
        counts = np.bincount(plan.assignment[lvl])
        assert counts.max() == exp
    for lvl in range(plan.c_level, len(plan.assignment)):
        assert len(set(plan.assignment[lvl])) == max(1, 4 >> (lvl - plan.c_level))
    for bad in ((16, 3), (16, 32), (12, 4), (16, 0)):
        with pytest.raises(ValueError):
            plan_schedule(*bad)
    assert critical_path_length(plan_schedule(16, 4)) == 5
    assert critical_path_length(plan_schedule(16, 16)) == 4
    assert critical_path_length(plan_schedule(16, 1)) == 15
    assert critical_path_length(plan_schedule(8, 1)) == 7
    assert critical_path_length(plan_schedule(8, 8)) == 3
    assert critical_path_length(plan_schedule(128, 8)) == 18


@pytest.mark.slow
def test_acceptance_criterion_2(oracle):                                                # test_acceptance.cpp:120-133
    sysm = P.poisson(32)
    f = oracle.Factorization(sysm, eps=8e-3, eta=2.0, leaf_size=32, threads=8)
    r = sysm.relative_residual(f.solve())
    assert r <= 5e-2
    assert f.stats()["largest_rank"] <= 12
