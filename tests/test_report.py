"""Report schema (reference report.cpp) and the reference's problem generators
(discretize.cpp), CPU only.  Cases follow the reference's test_report.cpp / test_discretize.cpp:
JSON and CSV round trips, header/schema rejection, quoting, validation messages."""
import dataclasses
import json

import numpy as np
import pytest

from paper_1701_00182_b200 import problems as P
from paper_1701_00182_b200 import report as R
from paper_1701_00182_b200.acr import LevelTraffic, UsageError


def _sample():
    c = R.RunConfig(problem="convdiff", n=16, alpha=20.0, a=2.0, kappa=0.0, mode="refine", eps=1e-4, eta=1.5,
                    leaf=16, workers=4, seed=7, tol=1e-9, max_iterations=50, output="out, \"q\".csv", format="csv")
    return R.SolveReport(config=c, relative_residual=3.0486017332135285e-07, average_rank=5.393053855569155,
                         largest_rank=22, factor_bytes=5117018624, peak_bytes=123456789, peak_is_estimate=False,
                         t_factor=4.72, t_solve=0.024, iterations=3, converged=True,
                         residual_history=[1e-2, 1e-5, 1.5e-10],
                         factor_ledger=[LevelTraffic(0, 3, 1000, 4, 0), LevelTraffic(1, 3, 2000, 4, 0)],
                         solve_ledger=[LevelTraffic(0, 6, 96, 4, 0), LevelTraffic(1, 6, 96, 4, 0)],
                         error="")


def test_json_round_trip():
    r = _sample()
    assert R.parse_json(R.emit_json(r)) == r
    many = [r, dataclasses.replace(r, error="SingularBlockError: level 2, plane 3", converged=False)]
    assert R.parse_json_list(R.emit_json(many)) == many


def test_json_layout_matches_reference_schema():
    j = json.loads(R.emit_json(_sample()))
    assert j["schema"] == 1
    assert set(j) == {"schema", "config", "relative_residual", "average_rank", "largest_rank", "factor_bytes",
                      "peak_bytes", "peak_is_estimate", "t_factor", "t_solve", "iterations", "converged",
                      "residual_history", "ledger", "error"}
    assert set(j["config"]) == {f.name for f in dataclasses.fields(R.RunConfig)}
    assert set(j["ledger"]) == {"factor", "solve"}
    assert set(j["ledger"]["factor"][0]) == {"level", "messages", "bytes", "active_workers", "idle_workers"}
    # nlohmann's std::map objects print keys sorted; dump(2) indents by two
    text = R.emit_json(_sample())
    assert text.startswith('{\n  "average_rank"')


def test_json_missing_key_rejected():
    j = json.loads(R.emit_json(_sample()))
    del j["t_solve"]
    with pytest.raises(UsageError):
        R.parse_json(json.dumps(j))


def test_csv_round_trip_and_quoting():
    r = _sample()
    text = R.emit_csv([r, r])
    lines = text.split("\n")
    assert lines[0] == R.CSV_HEADER and len(R.CSV_HEADER.split(",")) == 30
    assert text.endswith("\n")
    assert '"out, ""q"".csv"' in lines[1]
    back = R.parse_csv(text)
    assert back == [r, r]


def test_csv_number_format_is_precision_17():
    """std::ostream << double at precision(17) is printf("%.17g") (report.cpp:20-25)."""
    import ctypes
    libc = ctypes.CDLL(None)
    buf = ctypes.create_string_buffer(64)
    for v in (0.001, 0.0, 1e-6, 2.0, -3.5e300, 5e-324, 3.0486017332135285e-07, 4.72, 123456789.0):
        libc.snprintf(buf, 64, b"%.17g", ctypes.c_double(v))
        assert R.fmt_double(v) == buf.value.decode(), v
    assert R.fmt_double(1e-6) == "9.9999999999999995e-07"


def test_csv_rejections():
    with pytest.raises(UsageError, match="empty"):
        R.parse_csv("")
    with pytest.raises(UsageError, match="header"):
        R.parse_csv("schema,problem\n1,poisson\n")
    row = R.emit_csv([_sample()]).split("\n")[1]
    with pytest.raises(UsageError, match="column count"):
        R.parse_csv(R.CSV_HEADER + "\n" + row + ",extra\n")
    with pytest.raises(UsageError, match="schema version 2"):
        R.parse_csv(R.CSV_HEADER + "\n2" + row[1:] + "\n")
    assert R.parse_csv(R.CSV_HEADER + "\n\n" + row + "\n\n") == [_sample()]


def test_parse_names():
    assert [R.parse_run_mode(m) for m in R.RUN_MODES] == list(R.RUN_MODES)
    for bad, fn in (("lu", R.parse_run_mode), ("xml", R.parse_report_format), ("wave", R.parse_problem_kind)):
        with pytest.raises(UsageError):
            fn(bad)


@pytest.mark.parametrize("field,value,msg", [
    ("n", 1, "n must be >= 2"), ("eps", 0.0, "eps must be positive"), ("eta", -1.0, "eta must be positive"),
    ("leaf", 0, "leaf must be >= 1"), ("workers", 0, "workers must be >= 1"), ("tol", 0.0, "tol must be positive"),
    ("max_iterations", 0, "max_iterations must be >= 1"), ("alpha", -1.0, "alpha must be nonnegative"),
])
def test_validate(field, value, msg):
    with pytest.raises(UsageError, match=msg):
        R.validate(dataclasses.replace(R.RunConfig(), **{field: value}))


def test_validate_pcg_needs_symmetric():
    with pytest.raises(UsageError, match="symmetric"):
        R.validate(R.RunConfig(problem="convdiff", alpha=1.0, mode="pcg"))
    R.validate(R.RunConfig(problem="convdiff", alpha=0.0, mode="pcg"))


def test_cr_dense_is_not_a_gpu_mode():
    with pytest.raises(UsageError, match="cr-dense"):
        R.to_acr_config(R.RunConfig(mode="cr-dense"))


def test_sweep_argument_errors():
    with pytest.raises(UsageError, match="empty axis"):
        R.sweep(R.RunConfig(), "eps", [])
    with pytest.raises(UsageError, match="unknown axis"):
        R.sweep(R.RunConfig(), "leaf", [16])


def test_peak_rss():
    v = R.peak_rss_bytes()
    assert v is None or v > 0


# ------------------------------------------------------------------ generators
def test_convdiff_alpha0_is_poisson_operator():
    s, p = P.convdiff_vortex(6, 0.0), P.poisson(6)
    assert np.array_equal(s.blk_off, p.blk_off) and np.array_equal(s.cols, p.cols)
    assert np.array_equal(s.vals, p.vals)


def test_convdiff_rhs_is_operator_times_exact():
    """assemble_convdiff defines f = A u_exact (discretize.cpp:152-156)."""
    s = P.convdiff_vortex(7, 25.0, 1.0)
    A = s.to_dense()
    assert np.abs(A - A.T).max() > 0.1  # nonsymmetric once alpha > 0
    np.testing.assert_allclose(A @ s.exact.ravel(), s.rhs.ravel(), rtol=0, atol=1e-12)
    # first-order upwind keeps the operator an M-matrix: nonpositive off-diagonals
    off = A - np.diag(np.diag(A))
    assert off.max() <= 0.0
    assert np.all(np.diag(A) + off.sum(axis=1) >= -1e-12)


def test_helmholtz_fem_stencil():
    """27-point trilinear FEM (discretize.cpp:176-214): symmetric 9-point plane blocks,
    f = h^3, kappa = n/2 by default."""
    n = 5
    s = P.assemble("helmholtz", n)
    h = 1.0 / (n + 1)
    A = s.to_dense()
    assert np.abs(A - A.T).max() < 1e-15
    assert s.rhs.shape == (1, n, n * n) and np.all(s.rhs == h ** 3)
    r, c, v = s.E(1)
    assert len(r) == (3 * n - 2) ** 2  # 9-point pattern on an n x n plane
    # interior row sum of K is 0, so the row sum is -kappa^2 * (sum of M) = -kappa^2 h^3
    kappa = P.helmholtz_kappa_for(n)
    mid = (n // 2) * n * n + (n // 2) * n + n // 2
    assert A[mid].sum() == pytest.approx(-kappa * kappa * h ** 3, rel=1e-12)
    k2 = P.assemble("helmholtz", n, kappa=1.0).to_dense()
    assert k2[mid].sum() == pytest.approx(-h ** 3, rel=1e-12)


def test_assemble_dispatch():
    assert np.array_equal(P.assemble("poisson", 4).vals, P.poisson(4).vals)
    with pytest.raises(ValueError):
        P.assemble("wave", 4)
    with pytest.raises(ValueError):
        P.convdiff_vortex(4, -1.0)


# ------------------------------------------------------------------ Matrix Market + CLI (CPU paths)
def test_matrix_market_round_trip(tmp_path):                 # test_core.cpp:130-151
    from paper_1701_00182_b200 import mmio
    for sysm in (P.poisson(4), P.convdiff_vortex(4, 30.0, 1.5), P.assemble("helmholtz", 4)):
        d = tmp_path / sysm.name
        mmio.write_system(sysm, str(d))
        for f in ("D_0.mtx", "D_3.mtx", "E_1.mtx", "F_0.mtx", "F_2.mtx", "f_0.txt"):
            assert (d / f).exists()
        assert not (d / "E_0.mtx").exists() and not (d / "F_3.mtx").exists()
        back = mmio.read_system(str(d), 4)
        assert back.n == 4 and back.dim == 16
        assert np.array_equal(back.blk_off, sysm.blk_off)
        assert np.array_equal(back.rows, sysm.rows) and np.array_equal(back.cols, sysm.cols)
        assert np.array_equal(back.vals, sysm.vals)          # %.17g round-trips exactly
        assert np.array_equal(back.rhs, sysm.rhs)
        np.testing.assert_array_equal(back.coords, sysm.coords)


def test_matrix_market_errors(tmp_path):
    from paper_1701_00182_b200 import mmio
    from paper_1701_00182_b200.acr import Error
    p = tmp_path / "x.mtx"
    p.write_text("not a header\n")
    with pytest.raises(Error, match="not a Matrix Market"):
        mmio.read_matrix_market(str(p))
    p.write_text("%%MatrixMarket matrix coordinate real general\n% comment\n3 4 0\n")
    with pytest.raises(Error, match="square"):
        mmio.read_matrix_market(str(p))
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 2.0\n")
    with pytest.raises(Error, match="truncated entries"):
        mmio.read_matrix_market(str(p))
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n1 1 2.0\n2 1 -1\n")
    dim, (r, c, v) = mmio.read_matrix_market(str(p))   # duplicates summed (block.cpp:19-27)
    assert dim == 2 and list(r) == [0, 1] and list(c) == [0, 0] and list(v) == [3.0, -1.0]
    with pytest.raises(Error, match="cannot open"):
        mmio.read_plane_vector(str(tmp_path / "missing.txt"))


def _cli(args, env=None):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **(env or {}))
    return subprocess.run([sys.executable, "-m", "paper_1701_00182_b200.cli"] + args, cwd=root, env=e,
                          capture_output=True, text=True, timeout=300)


def test_cli_usage_errors_exit_2():                          # test_cli.cpp:77-84
    for args in (["solve", "--problem", "poisson", "--n", "1"], ["solve", "--problem", "bogus", "--n", "8"],
                 ["frobnicate"], ["solve", "--problem", "poisson", "--n", "8", "--eps", "-3"],
                 ["solve", "--mode", "cr-dense"]):
        r = _cli(args)
        assert r.returncode == 2, (args, r.stderr)
        assert r.stderr
    r = _cli(["solve", "--n", "8"], env={"ACR_WORKERS": "0"})
    assert r.returncode == 2 and json.loads(r.stderr.strip().splitlines()[-1])["kind"] == "usage"


def test_cli_generate(tmp_path):                             # test_cli.cpp:93-104
    d = tmp_path / "gen"
    r = _cli(["generate", "--problem", "poisson", "--n", "4", "--out", str(d)])
    assert r.returncode == 0, r.stderr
    for f in ("D_0.mtx", "D_3.mtx", "E_1.mtx", "F_2.mtx", "f_0.txt"):
        assert (d / f).exists()
