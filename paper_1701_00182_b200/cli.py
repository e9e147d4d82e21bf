"""Command-line harness over the GPU path (reference tools/acr_cli.cpp).

    python -m paper_1701_00182_b200.cli generate --problem poisson --n 16 --out DIR
    python -m paper_1701_00182_b200.cli factor|solve [--mode acr] [problem/solver flags]
    python -m paper_1701_00182_b200.cli pcg [--refine] [flags]
    python -m paper_1701_00182_b200.cli bench --axis eps --values 1e-1,1e-2,1e-3 [flags]

Same subcommands, flags, ACR_WORKERS override, report printing and exit codes as the
reference: 0 ok, 2 usage error, 3 solver failure / nonconvergence; errors go to stderr
as one JSON object with "kind" usage | solver | internal (acr_cli.cpp:12-167).
"""
from __future__ import annotations

import argparse
import json
import os
import sys

EXIT_USAGE = 2
EXIT_SOLVER_FAILURE = 3


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        sys.exit(EXIT_USAGE)


def _positive_int(s):
    v = int(s)
    if v <= 0:
        raise argparse.ArgumentTypeError("must be positive")
    return v


def _problem_flags(p):
    p.add_argument("--problem", default="poisson", choices=["poisson", "convdiff", "helmholtz"])
    p.add_argument("--n", type=_positive_int, default=8)
    p.add_argument("--alpha", type=float, default=0.0)
    p.add_argument("--a", type=float, default=1.0)
    p.add_argument("--kappa", type=float, default=0.0)


def _solver_flags(p):
    p.add_argument("--eps", type=float, default=1e-3)
    p.add_argument("--eta", type=float, default=2.0)
    p.add_argument("--leaf", type=int, default=32)
    p.add_argument("--workers", type=int, default=1)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--tol", type=float, default=1e-6)
    p.add_argument("--max-iterations", type=int, default=200)
    p.add_argument("--output", "-o", default="")
    p.add_argument("--format", default="json", choices=["json", "csv"])


def _config(a, mode):
    from .report import RunConfig, parse_problem_kind, parse_report_format, parse_run_mode
    from .acr import UsageError
    workers = a.workers
    env = os.environ.get("ACR_WORKERS")
    if env is not None:
        try:
            workers = int(env)
        except ValueError:
            workers = 0
        if workers < 1:
            raise UsageError("ACR_WORKERS must be a positive integer")
    return RunConfig(problem=parse_problem_kind(a.problem), n=a.n, alpha=a.alpha, a=a.a, kappa=a.kappa,
                     mode=parse_run_mode(mode), eps=a.eps, eta=a.eta, leaf=a.leaf, workers=workers, seed=a.seed,
                     tol=a.tol, max_iterations=a.max_iterations, output=a.output,
                     format=parse_report_format(a.format))


def _print_report(rep):
    from .report import emit_csv, emit_json
    if rep.config.output:
        return
    sys.stdout.write(emit_json(rep) + "\n" if rep.config.format == "json" else emit_csv([rep]))


def main(argv=None) -> int:
    ap = _Parser(prog="acr", description="Tolerance-controlled block tridiagonal solver (B200)")
    sub = ap.add_subparsers(dest="cmd", parser_class=_Parser)
    sub.required = True
    g = sub.add_parser("generate", help="write a problem as Matrix Market files")
    _problem_flags(g)
    g.add_argument("--out", default="system")
    for name in ("factor", "solve"):
        s = sub.add_parser(name)
        _problem_flags(s)
        _solver_flags(s)
        s.add_argument("--mode", default="acr", choices=["acr", "cr-dense"])
    pc = sub.add_parser("pcg", help="iterate with the factorization as preconditioner")
    _problem_flags(pc)
    _solver_flags(pc)
    pc.add_argument("--refine", action="store_true")
    b = sub.add_parser("bench", help="sweep one parameter, one report per point")
    _problem_flags(b)
    _solver_flags(b)
    b.add_argument("--mode", default="acr")
    b.add_argument("--axis", default="eps")
    b.add_argument("--values", default="1e-1,1e-2,1e-3")
    a = ap.parse_args(argv)

    from .acr import Error, UsageError

    def fail(msg, kind, code):
        sys.stderr.write(json.dumps({"error": msg, "kind": kind}) + "\n")
        return code

    try:
        from . import report as R
        if a.cmd == "generate":
            from . import mmio, problems
            try:
                sysm = problems.assemble(R.parse_problem_kind(a.problem), a.n, a.alpha, a.a, a.kappa)
            except ValueError as e:
                raise UsageError(str(e)) from None
            mmio.write_system(sysm, a.out)
            print(f"wrote {a.n}-plane system to {a.out}")
        elif a.cmd in ("factor", "solve"):
            _print_report(R.run(_config(a, a.mode)))
        elif a.cmd == "pcg":
            rep = R.run(_config(a, "refine" if a.refine else "pcg"))
            _print_report(rep)
            if not rep.converged:
                sys.stderr.write(json.dumps({"error": f"did not converge in {rep.iterations} iterations"}) + "\n")
                return EXIT_SOLVER_FAILURE
        else:
            cfg = _config(a, a.mode)
            values = [float(t) for t in a.values.split(",") if t]
            reps = R.sweep(cfg, a.axis, values)
            if not cfg.output:
                sys.stdout.write(R.emit_json(reps) + "\n" if cfg.format == "json" else R.emit_csv(reps))
    except UsageError as e:
        return fail(str(e), "usage", EXIT_USAGE)
    except Error as e:
        return fail(str(e), "solver", EXIT_SOLVER_FAILURE)
    except Exception as e:  # noqa: BLE001 -- mirrors the reference's catch of std::exception
        return fail(str(e), "internal", EXIT_SOLVER_FAILURE)
    return 0


if __name__ == "__main__":
    sys.exit(main())
