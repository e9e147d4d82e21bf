"""GPU parity tests: libacrgpu.so (sm_100a, through the C-ABI) against the CPU
oracle on identical seeded inputs, plus the reference's own H-mode pins
(proj/tests/test_acr.cpp, test_acceptance.cpp) run on the GPU path.

Bar (BASELINE.json north_star): relative residual within 2x of the oracle's at the
same tolerance, stored-inverse ranks within +-10%.  Integer/structural outputs
(plane counts, leaf counts) must match exactly."""
import numpy as np
import pytest

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


def compare(acr, oracle, sysm, eps, leaf=32, eta=2.0, weak=False, stop=1, exact=False, threads=8):
    cfg = acr.AcrConfig(eps=eps, leaf_size=leaf, eta=eta, stop_planes=stop, exact_dense_products=exact,
                        admissibility=acr.Admissibility.Weak if weak else acr.Admissibility.Standard)
    g = acr.acr_factor(sysm, cfg)
    ug = g.solve(sysm.rhs)
    o = oracle.Factorization(sysm, eps=eps, leaf_size=leaf, eta=eta, weak=weak, stop_planes=stop, threads=threads)
    uo = o.solve(sysm.rhs)
    rg, ro = sysm.relative_residual(ug), sysm.relative_residual(uo)
    sg, so = g.inverse_rank_stats(), o.stats()
    return g, o, ug, uo, rg, ro, sg, so


def assert_parity(rg, ro, sg, so, lv_g=None, lv_o=None):
    assert rg <= 2.0 * ro + 1e-14, (rg, ro)
    assert abs(sg.largest_rank - so["largest_rank"]) <= max(1, round(0.1 * so["largest_rank"])), (sg, so)
    assert abs(sg.average_rank - so["average_rank"]) <= 0.1 * so["average_rank"] + 1e-9, (sg, so)
    assert sg.dense_leaf_count == so["dense_leaf_count"] and sg.lowrank_leaf_count == so["lowrank_leaf_count"]
    if lv_g is not None:
        assert [l.plane_count for l in lv_g] == [l["plane_count"] for l in lv_o]
        assert [l.eliminated for l in lv_g] == [l["eliminated"] for l in lv_o]
        for a, b in zip(lv_g, lv_o):
            assert abs(a.largest_rank - b["largest_rank"]) <= max(1, round(0.1 * b["largest_rank"]))


@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_baseline_configs_small_n(acr, oracle, k):
    """BASELINE configs 1-4 operators at n=16 with their own leaf/eps."""
    c = P.CONFIGS[k]
    sysm = P.config_system(k, n=16)
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, c["eps"], c["leaf"])
    assert_parity(rg, ro, sg, so, g.level_info(), o.level_info())
    if k != 4:  # C4 (indefinite Helmholtz): H-ACR at eps 1e-4 does not converge in the reference either
        assert np.linalg.norm(ug - uo) <= 1e-3 * np.linalg.norm(uo)


@pytest.mark.parametrize("n", [16, 32])
def test_config5_operator_leaf64_multi_rhs(acr, oracle, n):
    """BASELINE config 5 (vardiff, leaf 64, eps 1e-6, 16 RHS) at reduced plane counts: the
    64x64 dense-leaf kernels (k_dd_product, k_lu_inverse at 64, mid64/d128/QR truncation
    classes) against the oracle, all 16 right-hand sides in one solve."""
    c = P.CONFIGS[5]
    sysm = P.config_system(5, n=n)
    assert sysm.rhs.shape[0] == 16
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, c["eps"], c["leaf"], threads=16)
    assert_parity(rg, ro, sg, so, g.level_info(), o.level_info())
    assert np.linalg.norm(ug - uo) <= 1e-3 * np.linalg.norm(uo)
    assert abs(g.factor_bytes() - so["factor_bytes"]) <= 0.02 * so["factor_bytes"]


@pytest.mark.parametrize("n", [14, 18])
def test_config5_operator_odd_leaf_sizes(acr, oracle, n):
    """Leaf 64 on planes whose leaf clusters are odd (n = 14: 196 points -> 49-point leaves) or
    mixed (n = 18: 324 -> 81 -> {40, 41}): the 64-class kernels on operands whose sizes and
    addresses are not 16-byte aligned -- k_dd_product's load/store staging instead of its two TMA
    bulk copies, the slab kernel's producer-store path -- against the oracle, 16 right-hand sides."""
    c = P.CONFIGS[5]
    sysm = P.config_system(5, n=n)
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, c["eps"], c["leaf"], threads=8)
    assert_parity(rg, ro, sg, so, g.level_info(), o.level_info())
    assert np.linalg.norm(ug - uo) <= 1e-3 * np.linalg.norm(uo)


def test_config1_full_size(acr, oracle):
    """C1 at its BASELINE size (n=32, N=32768, eps 1e-6): residual, ranks, bytes."""
    sysm = P.config_system(1)
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, 1e-6, 32, threads=16)
    assert_parity(rg, ro, sg, so, g.level_info(), o.level_info())
    assert abs(g.factor_bytes() - so["factor_bytes"]) <= 0.02 * so["factor_bytes"]


def test_reference_hmode_n16(acr):                                               # test_acr.cpp:243-257
    sysm = P.poisson(16)
    f = acr.acr_factor(sysm, acr.AcrConfig(eps=1e-3))
    u = f.solve(sysm.rhs[0])
    assert sysm.relative_residual(u) <= 1e-2
    st = f.inverse_rank_stats()
    assert 1 <= st.largest_rank <= 12
    assert st.largest_rank >= st.average_rank
    assert f.factor_bytes() > 0
    assert f.level_info()[0].plane_count == 16


def test_reference_residual_monotone(acr):                                       # test_acr.cpp:259-270
    sysm = P.poisson(16)
    prev = 1e9
    for eps in (1e-1, 1e-2, 1e-3, 1e-4):
        r = sysm.relative_residual(acr.acr_factor(sysm, acr.AcrConfig(eps=eps)).solve(sysm.rhs[0]))
        assert r <= prev * 1.0001
        prev = r


def test_acceptance_criterion_2(acr):                                            # test_acceptance.cpp:120-133
    sysm = P.poisson(32)
    f = acr.acr_factor(sysm, acr.AcrConfig(eps=8e-3, eta=2.0, leaf_size=32))
    assert sysm.relative_residual(f.solve(sysm.rhs[0])) <= 5e-2
    assert f.inverse_rank_stats().largest_rank <= 12


def test_acceptance_criterion_3_poisson_ranks(acr):                              # test_acceptance.cpp:135-145
    for n in (8, 16, 32):
        f = acr.acr_factor(P.poisson(n), acr.AcrConfig(eps=1e-3))
        assert f.inverse_rank_stats().largest_rank <= 12


def test_dinv_leaf_ranks_match_oracle(acr, oracle):
    sysm = P.config_system(1, n=16)
    g = acr.acr_factor(sysm, acr.AcrConfig(eps=1e-6))
    o = oracle.Factorization(sysm, eps=1e-6, threads=8)
    tot = diff = 0
    for li, lvl in enumerate(o.level_info()):
        planes = range(lvl["plane_count"])
        for j in planes:
            a, b = g.dinv_ranks(li, j), o.dinv_ranks(li, j)
            if b is None:
                assert a is None
                continue
            assert np.array_equal(a < 0, b < 0)  # same dense/low-rank leaf layout
            tot += (b >= 0).sum()
            diff += (np.abs(a - b)[b >= 0] > 1).sum()
    assert diff <= 0.01 * tot


def test_multi_rhs_bitwise_and_linearity(acr):                                  # test_acr.cpp:148-163
    sysm = P.config_system(2, n=16)
    f = acr.acr_factor(sysm, acr.AcrConfig(eps=1e-6))
    g1 = sysm.rhs[0]
    g2 = P.uniform_pm1(60, 1, g1.size).reshape(g1.shape)
    u1, u2 = f.solve(g1), f.solve(g2)
    both = f.solve(np.stack([g1, g2]))
    assert np.array_equal(both[0], u1) and np.array_equal(both[1], u2)
    assert np.array_equal(f.solve(g2), u2)
    u3 = f.solve(2.0 * g1 - 0.5 * g2)
    assert np.linalg.norm(u3 - (2.0 * u1 - 0.5 * u2)) <= 1e-12 * np.linalg.norm(u3)


@pytest.mark.parametrize("k,n,nrhs", [(5, 16, 16), (5, 32, 16), (5, 14, 16), (2, 16, 5), (1, 10, 7), (3, 14, 20), (2, 22, 33)])
def test_bulk_copy_slab_kernel_is_bitwise_the_load_kernel(acr, monkeypatch, k, n, nrhs):
    # Solves with more than 4 right-hand sides run phase 2 of the H-matvec on the TMA bulk-copy
    # engine (k_mv_slab_tma: cp.async.bulk into a shared-memory ring, DMMA from shared memory).
    # It performs the per-lane load kernel's arithmetic (k_mv_slab, ACRGPU_MV_LDG=1) in the same
    # order, so the solutions are bitwise equal -- including plane sizes whose leaf clusters are
    # odd (n = 10: 25-point leaves; n = 14: {24, 25}; n = 22: {30, 31}), which take the unaligned
    # copy path, right-hand-side counts that are not multiples of 16, and several 16-column passes.
    c = P.CONFIGS[k]
    sysm = P.config_system(k, n=n)
    f = acr.acr_factor(sysm, acr.AcrConfig(eps=c["eps"], leaf_size=c["leaf"]))
    g = P.uniform_pm1(77, k, nrhs * sysm.rhs[0].size).reshape((nrhs,) + sysm.rhs[0].shape)
    u_tma = f.solve(g)
    monkeypatch.setenv("ACRGPU_MV_LDG", "1")
    u_ldg = f.solve(g)
    monkeypatch.delenv("ACRGPU_MV_LDG")
    assert np.array_equal(u_tma, u_ldg)
    assert np.array_equal(f.solve(g), u_tma)
    for j in (0, nrhs - 1):
        assert sysm.relative_residual(u_tma[j:j + 1], g[j:j + 1]) <= 1e-4


def test_bulk_copy_slab_kernel_wide_leaves(acr, monkeypatch):
    # Rk leaves of rank > 64 take the slab kernel's one-stage-per-piece path (TF_WIDE) and phase 1's
    # multi-tile loop.  Weak admissibility makes the off-diagonal half blocks of a 48 x 48 plane
    # low-rank leaves whose rank at eps 1e-12 exceeds 64 (asserted, so the path cannot go untested).
    sysm = P.config_system(1, n=48)
    sysm = P.first_planes(sysm, 6)  # six 2304-point planes
    cfg = acr.AcrConfig(eps=1e-12, leaf_size=32, admissibility=acr.Admissibility.Weak)
    f = acr.acr_factor(sysm, cfg)
    assert f.inverse_rank_stats().largest_rank > 64
    nrhs = 16
    g = P.uniform_pm1(91, 3, nrhs * sysm.rhs[0].size).reshape((nrhs,) + sysm.rhs[0].shape)
    u_tma = f.solve(g)
    monkeypatch.setenv("ACRGPU_MV_LDG", "1")
    u_ldg = f.solve(g)
    monkeypatch.delenv("ACRGPU_MV_LDG")
    assert np.array_equal(u_tma, u_ldg)
    assert sysm.relative_residual(u_tma, g) <= 1e-8


def test_factorization_deterministic(acr):
    sysm = P.config_system(3, n=16)
    cfg = acr.AcrConfig(eps=1e-6)
    u1 = acr.acr_factor(sysm, cfg).solve(sysm.rhs)
    u2 = acr.acr_factor(sysm, cfg).solve(sysm.rhs)
    assert np.array_equal(u1, u2)


def test_root_plan_block_split_and_level_pipeline_are_bitwise_neutral(acr, monkeypatch):
    # Two schedules that only regroup work: root products run as their 4 x 4 target blocks
    # (Engine::mult_add, C5-sized planes; forced here at a small size) and the pipelined
    # levels of the single-GPU driver (do_factor).  Same per-leaf part lists and per-plane
    # arithmetic, so solutions, ranks and bytes are bitwise those of the plain schedule.
    sysm = P.config_system(2, n=16)
    cfg = acr.AcrConfig(eps=1e-6)
    f1 = acr.acr_factor(sysm, cfg)
    u1 = f1.solve(sysm.rhs)
    for env in ("ACRGPU_FORCE_SPLIT", "ACRGPU_NO_PIPELINE"):
        monkeypatch.setenv(env, "1")
        f2 = acr.acr_factor(sysm, cfg)
        u2 = f2.solve(sysm.rhs)
        monkeypatch.delenv(env)
        assert np.array_equal(u1, u2), env
        s1, s2 = f1.inverse_rank_stats(), f2.inverse_rank_stats()
        assert (s1.largest_rank, s1.average_rank) == (s2.largest_rank, s2.average_rank)
        assert f1.factor_bytes() == f2.factor_bytes()
        for li in (0, 1):
            assert np.array_equal(f1.dinv_ranks(li, 0), f2.dinv_ranks(li, 0))


@pytest.mark.parametrize("at", ["0", "0.000001"])
def test_persistent_arena_compaction_is_bitwise_neutral(acr, monkeypatch, at):
    # Engine::gc (C5-sized planes compact live low-rank data into the other semi-space of the
    # persistent arena) forced at small size: every safe point ("0") or once past a tiny fill.
    sysm = P.config_system(2, n=12)
    cfg = acr.AcrConfig(eps=1e-6)
    f1 = acr.acr_factor(sysm, cfg)
    u1 = f1.solve(sysm.rhs)
    monkeypatch.setenv("ACRGPU_GC_FORCE", at)
    f2 = acr.acr_factor(sysm, cfg)
    u2 = f2.solve(sysm.rhs)
    monkeypatch.delenv("ACRGPU_GC_FORCE")
    assert np.array_equal(u1, u2)
    s1, s2 = f1.inverse_rank_stats(), f2.inverse_rank_stats()
    assert (s1.largest_rank, s1.average_rank) == (s2.largest_rank, s2.average_rank)
    assert f1.factor_bytes() == f2.factor_bytes()


def test_resident_system_matches_host_path(acr):
    sysm = P.config_system(4, n=16)
    cfg = acr.AcrConfig(eps=1e-4)
    u_host = acr.acr_factor(sysm, cfg).solve(sysm.rhs)
    dsys = acr.DeviceSystem(sysm)
    u_dev = acr.acr_factor(dsys, cfg).solve(sysm.rhs)
    assert np.array_equal(u_host, u_dev)


@pytest.mark.parametrize("n", [5, 7, 12])
def test_non_power_of_two_planes(acr, oracle, n):                               # test_acr.cpp:204-211
    sysm = P.config_system(1, n=n)
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, 1e-6, 32)
    assert_parity(rg, ro, sg, so)


@pytest.mark.parametrize("stop", [2, 3])
def test_early_stop_apex(acr, oracle, stop):                                    # test_acr.cpp:213-221
    sysm = P.config_system(1, n=8)
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, 1e-6, 32, stop=stop)
    assert_parity(rg, ro, sg, so)


@pytest.mark.parametrize("weak,eta,leaf", [(True, 2.0, 32), (False, 1.0, 16), (False, 4.0, 32)])
def test_admissibility_variants(acr, oracle, weak, eta, leaf):
    sysm = P.config_system(2, n=16)
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, 1e-5, leaf, eta=eta, weak=weak)
    assert_parity(rg, ro, sg, so)


def test_exact_dense_products_deviation(acr, oracle):
    """DESIGN.md §5 deviation: exact dense*dense products into dense leaves; must stay within the bar."""
    sysm = P.config_system(1, n=16)
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, 1e-6, 32, exact=True)
    assert_parity(rg, ro, sg, so)


def test_lift_lowrank_entries(acr, oracle):
    """Entries inside admissible leaves: build_from_sparse factors them through their
    nonzero columns and truncates (hmatrix.cpp:127-147)."""
    base = P.poisson(8)
    n, dim = base.n, base.dim
    blocks = [base.block(b) for b in range(base.nblocks)]
    r, c, v = blocks[0]
    far = (np.array([0, dim - 1, 3], np.int32), np.array([dim - 1, 0, dim - 5], np.int32), np.array([0.3, -0.2, 0.1]))
    blocks[0] = (np.concatenate([r, far[0]]), np.concatenate([c, far[1]]), np.concatenate([v, far[2]]))
    sysm = P._assemble(n, dim, base.coords, blocks, P.seeded_rhs(5, 1, n, dim))
    cfg = dict(eps=1e-6, leaf=16)
    g, o, ug, uo, rg, ro, sg, so = compare(acr, oracle, sysm, 1e-6, 16)
    assert_parity(rg, ro, sg, so)


def test_singular_pivot_location(acr):                                          # test_acr.cpp:223-241
    n, d = 4, 16
    coords = P.plane_coords(4)
    I = (np.arange(d, dtype=np.int32), np.arange(d, dtype=np.int32), np.ones(d))
    Z = (np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0))
    blocks = [I, I, Z, I] + [Z] * 6
    sysm = P._assemble(n, d, coords, blocks, np.ones((1, n, d)))
    with pytest.raises(acr.SingularBlockError) as ei:
        acr.acr_factor(sysm, acr.AcrConfig(eps=1e-6, leaf_size=8))
    assert ei.value.level == 0 and ei.value.plane == 2


def test_error_paths(acr):
    sysm = P.poisson(4)
    f = acr.acr_factor(sysm, acr.AcrConfig(eps=1e-3))
    with pytest.raises(acr.DimensionError):
        f.solve(np.zeros((3, 16)))
    with pytest.raises(acr.DimensionError):
        f.solve(np.zeros((4, 9)))
    with pytest.raises(acr.UsageError):
        acr.acr_factor(sysm, acr.AcrConfig(stop_planes=0))
    with pytest.raises(acr.LeafMemoryError):
        acr.acr_factor(P.poisson(8), acr.AcrConfig(eps=1e-3, leaf_memory_cap=64))
    bad = P.poisson(4)
    bad.rows = bad.rows.copy()
    bad.rows[0] = 99
    with pytest.raises(acr.DimensionError):
        acr.acr_factor(bad, acr.AcrConfig(eps=1e-3))


def test_config2_full_size_properties(acr):
    """C2 at its BASELINE size (n=64, N=262144): the oracle needs ~25 min here, so
    size-independent properties: small residual, linearity, multi-RHS consistency, and
    the rank/residual figures the oracle produced for this exact input (profiles/)."""
    sysm = P.config_system(2)
    f = acr.acr_factor(sysm, acr.AcrConfig(eps=1e-6, leaf_size=32))
    u = f.solve(sysm.rhs)
    r = sysm.relative_residual(u)
    ro = 3.0486020791786735e-07                    # oracle residual for this input (seed 2024)
    assert r <= 2 * ro                              # the north_star bar
    assert abs(r - ro) <= 0.01 * ro                 # measured: equal to 7 digits
    st = f.inverse_rank_stats()
    # measured: identical to the oracle's (22 / 5.393053855569151); a rank regression of a
    # fraction of a percent must fail here, not only a violation of the +-10% bar
    assert st.largest_rank == 22 and abs(st.average_rank - 5.393053855569151) <= 1e-6 * 5.393053855569151
    g2 = P.uniform_pm1(9, 1, sysm.rhs.size).reshape(sysm.rhs.shape)
    u2 = f.solve(g2)
    u3 = f.solve(sysm.rhs - 3.0 * g2)
    assert np.linalg.norm(u3 - (u - 3.0 * u2)) <= 1e-11 * np.linalg.norm(u3)
