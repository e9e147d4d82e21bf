"""Full-size parity against committed oracle fixtures (tests/golden/oracle_c*_n*.json, made by
tests/golden/make_oracle_fixtures.py on the build container -- the oracle needs 25-60 min
per n=64 system, too long for a test run).

The north_star bar: relative residual within 2x of the oracle's at the same tolerance and
ranks within +-10%.  Where the GPU result is known to coincide with the oracle (C2: ranks
identical, residual equal to 7 digits) the tests pin it much tighter so that a regression
of a few percent is caught, not just a violation of the bar:
  * largest rank exact (+-1 allowed only where noted), average rank within 0.5%,
  * per-level largest rank +-1 and average within 1%,
  * stored-inverse leaf ranks leaf by leaf (same dense/low-rank layout, <= 1% of leaves
    off by more than one),
  * the solution at 1024 seeded sample positions within 1e-3 of the oracle's.

C5 (n=128, 16384-point planes, leaf 64) is too large for the oracle in this container's
62 GB of RAM (factor bytes ~73 GB).  Its leading 8-plane block sub-system is factored by
the oracle instead (fixture oracle_c5_n128_p8.json); the stored inverses of that
sub-system listed by window_entries (levels 0-2) depend only on planes 0..6 and
therefore equal the FULL system's (reduce_level, acr.cpp:70-120).  The full-system GPU
factorization is compared with them leaf by leaf, and the sub-system itself is compared
in full (residual, ranks, levels)."""
import json
import os

import numpy as np
import pytest

from paper_1701_00182_b200 import problems as P

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixture(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"fixture {name} not generated")
    with open(path) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def acr():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1701_00182_b200 import acr as A
    A.lib()
    return A


def gpu_factor(acr, sysm, fx):
    cfg = acr.AcrConfig(eps=fx["eps"], leaf_size=fx["leaf"])
    f = acr.acr_factor(sysm, cfg)
    u = f.solve(sysm.rhs)
    return f, u


def check_dinv(f, fx, max_frac=0.01, entries=None):
    tot = off = 0
    for d in fx["dinv_ranks"]:
        if entries is not None and (d["level"], d["plane"]) not in entries:
            continue
        g = f.dinv_ranks(d["level"], d["plane"])
        o = np.asarray(d["ranks"])
        assert g is not None, (d["level"], d["plane"])
        assert np.array_equal(g < 0, o < 0), "dense / low-rank leaf layout differs"
        lr = o >= 0
        tot += int(lr.sum())
        off += int((np.abs(g - o)[lr] > 1).sum())
    assert tot > 0
    assert off <= max_frac * tot, (off, tot)
    return tot, off


def check_levels(f, fx, tight=True):
    lg, lo = f.level_info(), fx["levels"]
    assert [l.plane_count for l in lg] == [l["plane_count"] for l in lo]
    assert [l.eliminated for l in lg] == [l["eliminated"] for l in lo]
    for a, b in zip(lg, lo):
        if tight:
            assert abs(a.largest_rank - b["largest_rank"]) <= 1, (a, b)
            assert abs(a.average_rank - b["average_rank"]) <= 0.01 * b["average_rank"] + 1e-9, (a, b)
        else:
            assert abs(a.largest_rank - b["largest_rank"]) <= max(1, round(0.1 * b["largest_rank"])), (a, b)


def check_solution(u, fx, rel=1e-3):
    flat = np.asarray(u).reshape(-1)
    idx = np.asarray(fx["u_sample_index"])
    us = np.asarray(fx["u_sample"])
    assert np.linalg.norm(flat[idx] - us) <= rel * np.linalg.norm(us)


@pytest.mark.parametrize("k", [2, 3])
def test_full_size_matches_oracle(acr, k):
    """C2 (variable-coefficient diffusion) and C3 (upwind convection-diffusion) at their
    BASELINE size n=64 (N=262,144; 64 planes of 4096), eps 1e-6, leaf 32."""
    fx = fixture(f"oracle_c{k}_n64.json")
    sysm = P.config_system(k, n=fx["n"], seed=fx["seed"])
    f, u = gpu_factor(acr, sysm, fx)
    rg, ro = sysm.relative_residual(u), fx["residual"]
    assert rg <= 2.0 * ro + 1e-14, (rg, ro)                  # the north_star bar
    assert abs(rg - ro) <= 0.02 * ro, (rg, ro)                # observed: equal to ~7 digits
    st, so = f.inverse_rank_stats(), fx["stats"]
    assert abs(st.largest_rank - so["largest_rank"]) <= 1, (st, so)
    assert abs(st.average_rank - so["average_rank"]) <= 0.005 * so["average_rank"], (st, so)
    assert (st.dense_leaf_count, st.lowrank_leaf_count) == (so["dense_leaf_count"], so["lowrank_leaf_count"])
    assert abs(f.factor_bytes() - so["factor_bytes"]) <= 0.02 * so["factor_bytes"]
    check_levels(f, fx)
    check_dinv(f, fx)
    check_solution(u, fx)


def test_config4_helmholtz_full_size_pinned(acr):
    """C4 (indefinite Helmholtz, eps 1e-4) at n=64.  H-arithmetic ACR at this tolerance does
    not resolve the operator (cond ~3e4, 940 negative eigenvalues): the oracle's residual is
    47.9, i.e. the reference algorithm diverges, and the pinned expectation is that the GPU
    lands in the same regime -- residual above 1 (no spurious 'solution') and within the
    north_star bar (<= 2x the oracle's) -- with ranks within +-10%.  In this regime the
    residual itself is chaotic in the rounding (GPU 2.98 vs oracle 47.9 measured), so only
    the regime and the bar are asserted, not closeness."""
    fx = fixture("oracle_c4_n64.json")
    sysm = P.config_system(4, n=fx["n"], seed=fx["seed"])
    f, u = gpu_factor(acr, sysm, fx)
    rg, ro = sysm.relative_residual(u), fx["residual"]
    assert ro > 1.0                                    # the pinned oracle behaviour: divergence
    assert rg <= 2.0 * ro + 1e-14, (rg, ro)
    assert rg > 1.0, (rg, ro)
    st, so = f.inverse_rank_stats(), fx["stats"]
    assert abs(st.largest_rank - so["largest_rank"]) <= max(1, round(0.1 * so["largest_rank"])), (st, so)
    assert abs(st.average_rank - so["average_rank"]) <= 0.1 * so["average_rank"], (st, so)
    # the first two levels precede the amplification of rounding differences (measured: level 5
    # largest rank 28 on the GPU vs 20 in the oracle), so they are compared leaf by leaf
    lg, lo = f.level_info(), fx["levels"]
    assert [l.plane_count for l in lg] == [l["plane_count"] for l in lo]
    for a, b in zip(lg[:2], lo[:2]):
        assert abs(a.largest_rank - b["largest_rank"]) <= max(1, round(0.1 * b["largest_rank"])), (a, b)
        assert abs(a.average_rank - b["average_rank"]) <= 0.05 * b["average_rank"], (a, b)
    check_dinv(f, fx, entries={(d["level"], d["plane"]) for d in fx["dinv_ranks"] if d["level"] <= 1})


def test_config5_leading_subsystem_matches_oracle(acr):
    """C5's first 8 planes (16384-point planes, leaf 64, eps 1e-6, 16 right-hand sides):
    the whole sub-system against the oracle."""
    fx = fixture("oracle_c5_n128_p8.json")
    sysm = P.first_planes(P.config_system(5, seed=fx["seed"]), fx["planes"])
    f, u = gpu_factor(acr, sysm, fx)
    rg, ro = sysm.relative_residual(u), fx["residual"]
    assert rg <= 2.0 * ro + 1e-14, (rg, ro)
    st, so = f.inverse_rank_stats(), fx["stats"]
    assert abs(st.largest_rank - so["largest_rank"]) <= 1, (st, so)
    assert abs(st.average_rank - so["average_rank"]) <= 0.01 * so["average_rank"], (st, so)
    check_levels(f, fx)
    check_dinv(f, fx)
    check_solution(u, fx)


def window_entries(fx):
    """(level, position) of stored inverses that the leading sub-system shares with the full
    system.  Position j of level l is original plane (j + 1) 2^l - 1; its inverse depends on
    the original planes [j 2^l, (j + 2) 2^l - 2] (every retained plane inside that range is
    updated from neighbours inside it).  The sub-system differs from the full system only
    in the update of its last plane p - 1, so the inverse is shared when the whole range
    lies below p - 1 ... or ends at p - 1 itself only at level 0 (no update involved)."""
    out = set()
    p = fx["planes"]
    for d in fx["dinv_ranks"]:
        l, j = d["level"], d["plane"]
        hi = (j + 2) * (1 << l) - 2
        if hi < p - 1 or (l == 0 and hi <= p - 1):
            out.add((l, j))
    return out


def test_config5_full_system_ranks_match_oracle(acr):
    """The n=128 C5 system itself (N=2,097,152, the north_star target), factored on the GPU:
    every stored inverse the oracle can reach in this container (levels 0-2, see
    window_entries) matches the oracle leaf by leaf, and the solve's residual is small."""
    fx = fixture("oracle_c5_n128_p8.json")
    entries = window_entries(fx)
    assert {(0, 0), (0, 2), (0, 4), (0, 6), (1, 0), (1, 2), (2, 0)} <= entries
    sysm = P.config_system(5, seed=fx["seed"])
    f, u = gpu_factor(acr, sysm, fx)
    tot, off = check_dinv(f, fx, entries=entries)
    assert tot > 1000
    assert sysm.relative_residual(u) <= 1e-6
