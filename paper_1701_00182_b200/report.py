"""Run reports and parameter sweeps over the GPU path (reference report.hpp / report.cpp).

Mirrors ``acr::RunConfig`` / ``acr::SolveReport`` / ``run`` / ``sweep`` and the
schema-1 JSON and CSV emitters and parsers (/root/reference/proj/core/include/acr/
report.hpp:11-80, core/src/report.cpp:59-527), so reports written by this package
are read by the reference's own tooling and vice versa:

    RunConfig, SolveReport               report.hpp:21-58
    run(config)                          report.cpp:326-397  (factor + solve / pcg / refine)
    sweep(base, axis, values)            report.cpp:399-436
    emit_json / parse_json / parse_json_list   report.cpp:438-455, 59-137
    emit_csv / parse_csv                 report.cpp:140-312, 457-476  (fixed 30 columns)
    peak_rss_bytes                       report.cpp:311-324

The factorization is the GPU one (``acr.acr_factor``; ``workers > 1`` runs the plane
partition ``acr.acr_factor_partitioned`` with in-process ranks and fills the ledger).
The reference's ``cr-dense`` mode is its exact dense CPU kernel (DenseKernel), which is
not part of the GPU path: ``run`` raises UsageError for it.

JSON follows nlohmann's ``dump(2)`` (keys sorted, two-space indent); CSV numbers use the
reference's ``precision(17)`` stream format (``%.17g``).
"""
from __future__ import annotations

import dataclasses
import json
import math
import time

from . import acr, problems
from .acr import LevelTraffic, UsageError

RUN_MODES = ("acr", "cr-dense", "pcg", "refine")
FORMATS = ("json", "csv")


def parse_run_mode(name: str) -> str:
    """report.cpp:254-260."""
    if name not in RUN_MODES:
        raise UsageError(f"unknown run mode: {name}")
    return name


def parse_report_format(name: str) -> str:
    """report.cpp:273-277."""
    if name not in FORMATS:
        raise UsageError(f"unknown report format: {name}")
    return name


def parse_problem_kind(name: str) -> str:
    """discretize.cpp:25-30."""
    if name not in problems.PROBLEM_KINDS:
        raise UsageError(f"unknown problem kind: {name}")
    return name


@dataclasses.dataclass
class RunConfig:
    """report.hpp:21-37 (same fields, same defaults)."""
    problem: str = "poisson"
    n: int = 8
    alpha: float = 0.0
    a: float = 1.0
    kappa: float = 0.0
    mode: str = "acr"
    eps: float = 1e-3
    eta: float = 2.0
    leaf: int = 32
    workers: int = 1
    seed: int = 0
    tol: float = 1e-6
    max_iterations: int = 200
    output: str = ""
    format: str = "json"


@dataclasses.dataclass
class SolveReport:
    """report.hpp:42-58."""
    config: RunConfig = dataclasses.field(default_factory=RunConfig)
    relative_residual: float = 0.0
    average_rank: float = 0.0
    largest_rank: int = 0
    factor_bytes: int = 0
    peak_bytes: int = 0
    peak_is_estimate: bool = False
    t_factor: float = 0.0
    t_solve: float = 0.0
    iterations: int = 0
    converged: bool = True
    residual_history: list = dataclasses.field(default_factory=list)
    factor_ledger: list = dataclasses.field(default_factory=list)
    solve_ledger: list = dataclasses.field(default_factory=list)
    error: str = ""


def validate(c: RunConfig) -> None:
    """report.cpp:29-41 (same checks, same messages)."""
    if c.n < 2:
        raise UsageError("run: n must be >= 2")
    if not c.eps > 0:
        raise UsageError("run: eps must be positive")
    if not c.eta > 0:
        raise UsageError("run: eta must be positive")
    if c.leaf < 1:
        raise UsageError("run: leaf must be >= 1")
    if c.workers < 1:
        raise UsageError("run: workers must be >= 1")
    if not c.tol > 0:
        raise UsageError("run: tol must be positive")
    if c.max_iterations < 1:
        raise UsageError("run: max_iterations must be >= 1")
    if c.alpha < 0:
        raise UsageError("run: alpha must be nonnegative")
    if c.mode == "pcg" and c.problem == "convdiff" and c.alpha > 0:
        raise UsageError("run: pcg requires a symmetric operator; use refine for convection-diffusion")


def to_acr_config(c: RunConfig) -> acr.AcrConfig:
    """report.cpp:43-50 (H-matrix mode only on the GPU path)."""
    if c.mode == "cr-dense":
        raise UsageError("run: cr-dense is the reference's exact dense CPU kernel; the GPU path is H-matrix only")
    return acr.AcrConfig(eps=c.eps, eta=c.eta, leaf_size=c.leaf)


def peak_rss_bytes():
    """VmHWM of this process (report.cpp:311-324), or None."""
    try:
        with open("/proc/self/status") as fh:
            for line in fh:
                if line.startswith("VmHWM:"):
                    kb = int(line.split()[1])
                    return kb * 1024 if kb > 0 else None
    except OSError:
        return None
    return None


def run(config: RunConfig) -> SolveReport:
    """acr::run (report.cpp:326-397): assemble, factor on the GPU (plane partition when
    workers > 1), then direct solve / PCG / refinement.  Like the reference, a
    partitioned run solves inside the factor timing (report.cpp:347-353)."""
    validate(config)
    rep = SolveReport(config=dataclasses.replace(config))
    try:
        system = problems.assemble(config.problem, config.n, config.alpha, config.a, config.kappa)
    except ValueError as e:
        raise UsageError(str(e)) from None
    ac = to_acr_config(config)
    t0 = time.perf_counter()
    u = None
    if config.workers > 1:
        from .plan import plan_schedule
        try:
            plan = plan_schedule(config.n, config.workers)
        except ValueError as e:
            raise UsageError(str(e)) from None
        comm = acr.Comm.local_ranks(config.workers)
        fact = acr.acr_factor_partitioned(system, comm, ac)
        u = fact.solve(system.rhs)[0]
        ledger = acr.message_ledger(fact, plan)
        rep.factor_ledger, rep.solve_ledger = ledger.factor, ledger.solve
    else:
        fact = acr.acr_factor(system, ac)
    rep.t_factor = time.perf_counter() - t0

    t1 = time.perf_counter()
    if config.mode == "acr":
        if u is None:
            u = fact.solve(system.rhs)[0]
    else:
        fn = acr.pcg if config.mode == "pcg" else acr.iterative_refinement
        res = fn(system, fact, config.tol, config.max_iterations)
        u = res.u
        rep.iterations = res.trace.iterations
        rep.converged = res.trace.converged
        rep.residual_history = list(res.trace.residual_history)
    rep.t_solve = time.perf_counter() - t1

    rep.relative_residual = system.relative_residual(u)
    st = fact.inverse_rank_stats()
    rep.average_rank = st.average_rank
    rep.largest_rank = st.largest_rank
    rep.factor_bytes = fact.factor_bytes()
    peak = peak_rss_bytes()
    if peak is not None:
        rep.peak_bytes = peak
    else:
        rep.peak_bytes = rep.factor_bytes
        rep.peak_is_estimate = True
    _write_output(rep)
    return rep


def sweep(base: RunConfig, axis: str, values) -> list:
    """acr::sweep (report.cpp:399-436): one run per value; acr errors are captured in
    the report's error field, the combined file is written once."""
    values = list(values)
    if not values:
        raise UsageError("sweep: empty axis")
    if axis not in ("eps", "n", "alpha"):
        raise UsageError(f"sweep: unknown axis {axis} (expected eps, n or alpha)")
    reports = []
    for v in values:
        c = dataclasses.replace(base, output="")
        if axis == "eps":
            c.eps = v
        elif axis == "n":
            c.n = int(v)
        else:
            c.alpha = v
        try:
            reports.append(run(c))
        except acr.Error as e:
            reports.append(SolveReport(config=c, converged=False, error=str(e)))
        reports[-1].config.output = base.output
    if base.output:
        text = emit_json(reports) + "\n" if base.format == "json" else emit_csv(reports)
        _write_file(base.output, text)
    return reports


# ------------------------------------------------------------------ JSON (schema 1)
def _ledger_json(lv):
    return [{"level": l.level, "messages": l.messages, "bytes": l.bytes, "active_workers": l.active_workers,
             "idle_workers": l.idle_workers} for l in lv]


def _ledger_from_json(arr):
    return [LevelTraffic(int(l["level"]), int(l["messages"]), int(l["bytes"]), int(l["active_workers"]),
                         int(l["idle_workers"])) for l in arr]


def _f(v) -> float:
    return float(v)


def report_json(r: SolveReport) -> dict:
    """report.cpp:72-103."""
    c = r.config
    return {
        "schema": 1,
        "config": {"problem": c.problem, "n": int(c.n), "alpha": _f(c.alpha), "a": _f(c.a), "kappa": _f(c.kappa),
                   "mode": c.mode, "eps": _f(c.eps), "eta": _f(c.eta), "leaf": int(c.leaf),
                   "workers": int(c.workers), "seed": int(c.seed), "tol": _f(c.tol),
                   "max_iterations": int(c.max_iterations), "output": c.output, "format": c.format},
        "relative_residual": _f(r.relative_residual),
        "average_rank": _f(r.average_rank),
        "largest_rank": int(r.largest_rank),
        "factor_bytes": int(r.factor_bytes),
        "peak_bytes": int(r.peak_bytes),
        "peak_is_estimate": bool(r.peak_is_estimate),
        "t_factor": _f(r.t_factor),
        "t_solve": _f(r.t_solve),
        "iterations": int(r.iterations),
        "converged": bool(r.converged),
        "residual_history": [_f(x) for x in r.residual_history],
        "ledger": {"factor": _ledger_json(r.factor_ledger), "solve": _ledger_json(r.solve_ledger)},
        "error": r.error,
    }


def report_from_json(j: dict) -> SolveReport:
    """report.cpp:105-137 (missing keys raise, as json::at does)."""
    try:
        c = j["config"]
        cfg = RunConfig(problem=parse_problem_kind(c["problem"]), n=int(c["n"]), alpha=_f(c["alpha"]),
                        a=_f(c["a"]), kappa=_f(c["kappa"]), mode=parse_run_mode(c["mode"]), eps=_f(c["eps"]),
                        eta=_f(c["eta"]), leaf=int(c["leaf"]), workers=int(c["workers"]), seed=int(c["seed"]),
                        tol=_f(c["tol"]), max_iterations=int(c["max_iterations"]), output=c["output"],
                        format=parse_report_format(c["format"]))
        return SolveReport(
            config=cfg, relative_residual=_f(j["relative_residual"]), average_rank=_f(j["average_rank"]),
            largest_rank=int(j["largest_rank"]), factor_bytes=int(j["factor_bytes"]),
            peak_bytes=int(j["peak_bytes"]), peak_is_estimate=bool(j["peak_is_estimate"]),
            t_factor=_f(j["t_factor"]), t_solve=_f(j["t_solve"]), iterations=int(j["iterations"]),
            converged=bool(j["converged"]), residual_history=[_f(x) for x in j["residual_history"]],
            factor_ledger=_ledger_from_json(j["ledger"]["factor"]),
            solve_ledger=_ledger_from_json(j["ledger"]["solve"]), error=j["error"])
    except KeyError as e:
        raise UsageError(f"report json: missing key {e}") from None


def _dump(obj) -> str:
    return json.dumps(obj, indent=2, sort_keys=True)


def emit_json(report) -> str:
    """emit_json(SolveReport) / emit_json(vector<SolveReport>) (report.cpp:438-445)."""
    if isinstance(report, SolveReport):
        return _dump(report_json(report))
    return _dump([report_json(r) for r in report])


def parse_json(text: str) -> SolveReport:
    return report_from_json(json.loads(text))


def parse_json_list(text: str) -> list:
    return [report_from_json(j) for j in json.loads(text)]


# ------------------------------------------------------------------ CSV (schema 1)
CSV_HEADER = ("schema,problem,n,alpha,a,kappa,mode,eps,eta,leaf,workers,seed,tol,max_iterations,"
              "output,format,relative_residual,average_rank,largest_rank,factor_bytes,peak_bytes,"
              "peak_is_estimate,t_factor,t_solve,iterations,converged,residual_history,"
              "factor_ledger,solve_ledger,error")


def fmt_double(v: float) -> str:
    """std::ostream with precision(17), default float format (report.cpp:20-25)."""
    v = float(v)
    if math.isnan(v):
        return "nan" if math.copysign(1.0, v) > 0 else "-nan"
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return format(v, ".17g")


def _csv_quote(s: str) -> str:
    if not any(ch in s for ch in ',"\n'):
        return s
    return '"' + s.replace('"', '""') + '"'


def _csv_split(line: str) -> list:
    """report.cpp:157-182."""
    out, cur, quoted, i = [], [], False, 0
    while i < len(line):
        ch = line[i]
        if quoted:
            if ch == '"' and i + 1 < len(line) and line[i + 1] == '"':
                cur.append('"')
                i += 1
            elif ch == '"':
                quoted = False
            else:
                cur.append(ch)
        elif ch == '"':
            quoted = True
        elif ch == ",":
            out.append("".join(cur))
            cur = []
        else:
            cur.append(ch)
        i += 1
    out.append("".join(cur))
    return out


def _join_ledger(lv) -> str:
    return "|".join(f"{l.level}:{l.messages}:{l.bytes}:{l.active_workers}:{l.idle_workers}" for l in lv)


def _split_ledger(s: str) -> list:
    out = []
    for tok in s.split("|"):
        if not tok:
            continue
        f = tok.split(":")
        out.append(LevelTraffic(int(f[0]), int(f[1]), int(f[2]), int(f[3]), int(f[4])))
    return out


def _csv_row(r: SolveReport) -> str:
    """report.cpp:233-270."""
    c = r.config
    cols = ["1", c.problem, str(int(c.n)), fmt_double(c.alpha), fmt_double(c.a), fmt_double(c.kappa), c.mode,
            fmt_double(c.eps), fmt_double(c.eta), str(int(c.leaf)), str(int(c.workers)), str(int(c.seed)),
            fmt_double(c.tol), str(int(c.max_iterations)), c.output, c.format,
            fmt_double(r.relative_residual), fmt_double(r.average_rank), str(int(r.largest_rank)),
            str(int(r.factor_bytes)), str(int(r.peak_bytes)), "1" if r.peak_is_estimate else "0",
            fmt_double(r.t_factor), fmt_double(r.t_solve), str(int(r.iterations)), "1" if r.converged else "0",
            ";".join(fmt_double(x) for x in r.residual_history), _join_ledger(r.factor_ledger),
            _join_ledger(r.solve_ledger), r.error]
    return ",".join(_csv_quote(x) for x in cols)


def _report_from_row(f: list) -> SolveReport:
    """report.cpp:272-305."""
    if len(f) != 30:
        raise UsageError("csv row has wrong column count")
    if f[0] != "1":
        raise UsageError(f"unsupported csv schema version {f[0]}")
    try:
        cfg = RunConfig(problem=parse_problem_kind(f[1]), n=int(f[2]), alpha=float(f[3]), a=float(f[4]),
                        kappa=float(f[5]), mode=parse_run_mode(f[6]), eps=float(f[7]), eta=float(f[8]),
                        leaf=int(f[9]), workers=int(f[10]), seed=int(f[11]), tol=float(f[12]),
                        max_iterations=int(f[13]), output=f[14], format=parse_report_format(f[15]))
        return SolveReport(
            config=cfg, relative_residual=float(f[16]), average_rank=float(f[17]), largest_rank=int(f[18]),
            factor_bytes=int(f[19]), peak_bytes=int(f[20]), peak_is_estimate=f[21] == "1",
            t_factor=float(f[22]), t_solve=float(f[23]), iterations=int(f[24]), converged=f[25] == "1",
            residual_history=[float(t) for t in f[26].split(";") if t], factor_ledger=_split_ledger(f[27]),
            solve_ledger=_split_ledger(f[28]), error=f[29])
    except ValueError as e:
        raise UsageError(f"csv row: {e}") from None


def emit_csv(reports) -> str:
    """Header line, then one row per report, each newline-terminated (report.cpp:457-465)."""
    return CSV_HEADER + "\n" + "".join(_csv_row(r) + "\n" for r in reports)


def parse_csv(text: str) -> list:
    """report.cpp:467-476: the header must match schema 1 exactly; empty lines are skipped."""
    lines = text.split("\n")
    if not text:
        raise UsageError("csv input is empty")
    if lines[0] != CSV_HEADER:
        raise UsageError("csv header does not match schema version 1")
    return [_report_from_row(_csv_split(line)) for line in lines[1:] if line]


def _write_file(path: str, text: str) -> None:
    try:
        with open(path, "w") as fh:
            fh.write(text)
    except OSError:
        raise UsageError(f"cannot open output file: {path}") from None


def _write_output(r: SolveReport) -> None:
    """report.cpp:307-315."""
    if not r.config.output:
        return
    _write_file(r.config.output, emit_json(r) + "\n" if r.config.format == "json" else emit_csv([r]))
