"""run / sweep / report schema on the GPU path (reference tests/test_report.cpp), the
partitioned run's message ledger (tests/test_parallel.cpp:91-183), and GPU-vs-oracle
parity on the reference's own generators (assemble_convdiff, assemble_helmholtz)."""
import dataclasses

import numpy as np
import pytest

from paper_1701_00182_b200 import problems as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1701_00182_b200 import acr, report
    acr.lib()
    return report


def small_config(R, mode):                                   # test_report.cpp:18-25
    return R.RunConfig(problem="poisson", n=8, mode=mode, eps=1e-2)


def strip_timing(r):                                         # test_report.cpp:10-16
    return dataclasses.replace(r, t_factor=0.0, t_solve=0.0, peak_bytes=0, peak_is_estimate=False)


def test_acr_run_populates_rank_statistics(R):               # test_report.cpp:38-47
    cfg = dataclasses.replace(small_config(R, "acr"), n=16, eps=1e-3)
    rep = R.run(cfg)
    assert rep.relative_residual <= 1e-1
    assert rep.largest_rank >= 1
    assert rep.factor_bytes > 0 and rep.t_factor > 0
    assert rep.largest_rank >= rep.average_rank


def test_json_round_trips_exactly(R):                        # test_report.cpp:49-66
    rep = R.run(small_config(R, "acr"))
    assert R.parse_json(R.emit_json(rep)) == rep
    pcg = R.run(dataclasses.replace(small_config(R, "pcg"), tol=1e-8))
    assert pcg.residual_history
    assert R.parse_json(R.emit_json(pcg)) == pcg
    par = R.run(dataclasses.replace(small_config(R, "acr"), workers=2))
    assert par.factor_ledger
    assert R.parse_json(R.emit_json(par)) == par
    assert R.parse_json_list(R.emit_json([rep, par])) == [rep, par]


def test_csv_round_trips_exactly(R):                         # test_report.cpp:77-91
    reports = [R.run(dataclasses.replace(small_config(R, "pcg"), format="csv")),
               R.run(dataclasses.replace(small_config(R, "acr"), workers=2))]
    text = R.emit_csv(reports)
    assert text.startswith("schema")
    assert R.parse_csv(text) == reports


def test_identical_configs_identical_reports(R):             # test_report.cpp:93-98
    cfg = small_config(R, "acr")
    assert strip_timing(R.run(cfg)) == strip_timing(R.run(cfg))


def test_sweep_eps_monotone(R):                              # test_report.cpp:100-108
    reps = R.sweep(small_config(R, "acr"), "eps", [1e-1, 1e-2, 1e-3])
    assert [r.config.eps for r in reps] == [1e-1, 1e-2, 1e-3]
    assert reps[1].relative_residual <= reps[0].relative_residual * 1.0001
    assert reps[2].relative_residual <= reps[1].relative_residual * 1.0001


def test_sweep_records_failures(R):                          # test_report.cpp:110-117
    reps = R.sweep(small_config(R, "acr"), "n", [8, 0, 4])
    assert [bool(r.error) for r in reps] == [False, True, False]
    assert not reps[1].converged


def test_invalid_configs_rejected(R):                        # test_report.cpp:125-136
    from paper_1701_00182_b200.acr import UsageError
    for cfg in (dataclasses.replace(small_config(R, "acr"), eps=-1.0),
                dataclasses.replace(small_config(R, "acr"), n=1),
                dataclasses.replace(small_config(R, "pcg"), problem="convdiff", alpha=10.0),
                dataclasses.replace(small_config(R, "acr"), workers=3)):
        with pytest.raises(UsageError):
            R.run(cfg)


def test_refine_reaches_tolerance(R):                        # test_report.cpp:147-154
    rep = R.run(dataclasses.replace(small_config(R, "refine"), tol=1e-10))
    assert rep.converged and rep.relative_residual <= 1e-10 and rep.iterations >= 1


def test_peak_memory_reported(R, tmp_path):                  # test_report.cpp:156-163
    out = tmp_path / "rep.json"
    rep = R.run(dataclasses.replace(small_config(R, "acr"), output=str(out)))
    assert not rep.peak_is_estimate and rep.peak_bytes >= rep.factor_bytes
    assert R.parse_json(out.read_text()) == rep


# ------------------------------------------------------------------ ledger (test_parallel.cpp)
def test_ledger_nearest_neighbour_messages(R):               # test_parallel.cpp:91-101
    from paper_1701_00182_b200 import acr
    from paper_1701_00182_b200.plan import plan_schedule
    sysm = P.poisson(16)
    for p in (2, 4, 8):
        f = acr.acr_factor_partitioned(sysm, acr.Comm.local_ranks(p), acr.AcrConfig(eps=1e-3))
        led = acr.message_ledger(f, plan_schedule(16, p))
        assert led.records
        for m in led.records:
            assert abs(m.from_plane - m.to_plane) == 1 and m.bytes > 0
        # contiguous partitions: one elimination payload per internal boundary per level
        # while every worker still holds two or more planes
        for l in led.factor:
            if l.active_workers == p and 16 >> l.level >= 2 * p:
                assert l.messages == p - 1


def test_ledger_active_workers_halve(R):                     # test_parallel.cpp:113-123
    rep = R.run(R.RunConfig(problem="poisson", n=16, eps=1e-3, workers=4))
    lv = rep.factor_ledger
    assert len(lv) == 4
    assert [l.active_workers for l in lv] == [4, 4, 4, 2]
    assert all(l.active_workers + l.idle_workers == 4 for l in lv)
    assert sum(l.messages for l in rep.solve_ledger) > 0     # test_parallel.cpp:175-183


def test_ledger_bytes_are_hmatrix_footprints(R):             # test_parallel.cpp:125-136
    from paper_1701_00182_b200 import acr
    from paper_1701_00182_b200.plan import plan_schedule
    sysm = P.poisson(8)
    f = acr.acr_factor_partitioned(sysm, acr.Comm.local_ranks(4), acr.AcrConfig(eps=1e-3))
    led = acr.message_ledger(f, plan_schedule(8, 4))
    assert sysm.relative_residual(f.solve(sysm.rhs)) <= 1e-2
    assert led.total_bytes() > 0
    for m in led.records:
        assert m.bytes < 4 * 64 * 64 * 8


def test_ledger_volume_envelope(R):                          # test_parallel.cpp:138-158
    b = {p: sum(l.bytes for l in R.run(R.RunConfig(problem="poisson", n=16, eps=1e-2, workers=p)).factor_ledger)
         for p in (2, 4, 8)}
    assert b[2] < b[4] < b[8]
    for p in (4, 8):
        assert b[2] / 2 / 2 <= b[p] / p <= 2 * b[2] / 2


def test_single_rank_has_no_messages(R):                     # test_parallel.cpp:66-73
    rep = R.run(R.RunConfig(problem="poisson", n=8, eps=1e-3, workers=1))
    assert rep.factor_ledger == [] and rep.solve_ledger == []


# ------------------------------------------------------------------ oracle parity, reference generators
@pytest.mark.parametrize("kind,n,kw,eps", [
    ("convdiff", 16, dict(alpha=20.0, a=1.0), 1e-6),
    ("convdiff", 16, dict(alpha=100.0, a=2.0), 1e-4),
    ("helmholtz", 16, dict(), 1e-6),
    ("helmholtz", 16, dict(kappa=4.0), 1e-4),
])
def test_reference_generators_match_oracle(R, kind, n, kw, eps):
    from oracle import oracle as O
    from paper_1701_00182_b200 import acr
    sysm = P.assemble(kind, n, **kw)
    f = acr.acr_factor(sysm, acr.AcrConfig(eps=eps, leaf_size=32))
    u = f.solve(sysm.rhs)
    ref = O.Factorization(sysm, eps=eps, leaf_size=32, threads=4)
    u_ref = ref.solve(sysm.rhs)
    res, res_ref = sysm.relative_residual(u), sysm.relative_residual(u_ref)
    assert res <= 2.0 * res_ref + 1e-14, (res, res_ref)
    st, st_ref = f.inverse_rank_stats(), ref.stats()
    assert abs(st.largest_rank - st_ref["largest_rank"]) <= max(1, 0.1 * st_ref["largest_rank"])
    assert abs(st.average_rank - st_ref["average_rank"]) <= 0.1 * st_ref["average_rank"] + 1e-12
    if kind == "convdiff":  # the discrete solution is known exactly (discretize.cpp:145-156)
        err = np.linalg.norm(u.reshape(-1) - sysm.exact.reshape(-1)) / np.linalg.norm(sysm.exact)
        assert err <= 1e-2


# ------------------------------------------------------------------ CLI (test_cli.cpp)
def _cli(args, env=None):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    return subprocess.run([sys.executable, "-m", "paper_1701_00182_b200.cli"] + args, cwd=root,
                          env=dict(os.environ, **(env or {})), capture_output=True, text=True, timeout=600)


def test_cli_factor_reports_statistics(R):                   # test_cli.cpp:106-112
    r = _cli(["factor", "--problem", "poisson", "--n", "16", "--eps", "1e-3"])
    assert r.returncode == 0, r.stderr
    rep = R.parse_json(r.stdout)
    assert rep.factor_bytes > 0 and rep.largest_rank >= 1


def test_cli_bench_sweep_csv(R):                             # test_cli.cpp:114-122
    r = _cli(["bench", "--problem", "poisson", "--n", "8", "--axis", "eps", "--values", "1e-1,1e-2,1e-3",
              "--format", "csv"])
    assert r.returncode == 0, r.stderr
    reps = R.parse_csv(r.stdout)
    assert len(reps) == 3
    assert reps[1].relative_residual <= reps[0].relative_residual * 1.0001
    assert reps[2].relative_residual <= reps[1].relative_residual * 1.0001


def test_cli_workers_from_environment(R):                    # test_cli.cpp:124-137
    r = _cli(["solve", "--problem", "poisson", "--n", "8", "--mode", "acr", "--eps", "1e-2"], env={"ACR_WORKERS": "2"})
    assert r.returncode == 0, r.stderr
    rep = R.parse_json(r.stdout)
    assert rep.config.workers == 2 and rep.factor_ledger


def test_cli_solver_failure_exit_3(R):                       # test_cli.cpp:86-91
    r = _cli(["pcg", "--problem", "helmholtz", "--n", "8", "--kappa", "12", "--eps", "1e-2", "--tol", "1e-12"])
    assert r.returncode == 3, (r.stdout, r.stderr)
    assert "{" in r.stderr


def test_cli_solve_writes_output_file(R, tmp_path):          # test_cli.cpp:56-67
    out = tmp_path / "rep.csv"
    r = _cli(["solve", "--problem", "convdiff", "--alpha", "10", "--n", "8", "--eps", "1e-4", "--format", "csv",
              "-o", str(out)])
    assert r.returncode == 0, r.stderr
    assert r.stdout == ""
    (rep,) = R.parse_csv(out.read_text())
    assert rep.config.problem == "convdiff" and rep.relative_residual < 1e-2
