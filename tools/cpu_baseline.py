"""Measured CPU baseline on the GPU box's host (SURVEY §8(d) "CPU baseline timing"): the oracle
(restatement of the reference path; the reference itself needs Eigen, absent here) timed
on a BASELINE config at full size.

    python tools/cpu_baseline.py CONFIG THREADS [N] [--sample-n S]

Modes (parallel.cpp:383-405 is the reference's only parallelism -- planes per worker):
  THREADS = p  plane-parallel level loop with p workers (factor and solve timed separately,
               not folded together as report.cpp:395-411 does)
  THREADS = 1  sequential acr_factor + solve (one core)
With --sample-n S it also times the bench's extrapolation sample (the same operator at
n = S) and reports the ratio measured / extrapolated, which calibrates bench.py's
--impl reference arm.  Writes one JSON line with the host CPU model and core count."""
import argparse
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1701_00182_b200 import problems as P  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def timed(cfgk, n, threads):
    c = P.CONFIGS[cfgk]
    sysm = P.config_system(cfgk, n=n)
    O.flops_reset()
    t0 = time.perf_counter()
    f = O.Factorization(sysm, eps=c["eps"], leaf_size=c["leaf"], threads=threads)
    tf = time.perf_counter() - t0
    t0 = time.perf_counter()
    u = f.solve(sysm.rhs)
    ts = time.perf_counter() - t0
    fl = O.flops_read()
    st = f.stats()
    return dict(n=sysm.n, N=sysm.total_dim, nrhs=int(sysm.rhs.shape[0]), t_factor_s=tf, t_solve_s=ts,
                flops=sum(fl[k] for k in ("gemm", "geqrf", "orgqr", "svd", "lu")),
                residual=float(sysm.relative_residual(u)), largest_rank=st["largest_rank"],
                average_rank=st["average_rank"],
                dof_per_s=sysm.total_dim * sysm.rhs.shape[0] / (tf + ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("threads", type=int)
    ap.add_argument("n", type=int, nargs="?", default=None)
    ap.add_argument("--sample-n", type=int, default=None)
    a = ap.parse_args()
    out = dict(config=a.config, threads=a.threads, cpu=cpu_model(), nproc=os.cpu_count(),
               kind="port (oracle/acr_oracle.cpp, -O3)")
    out["full"] = timed(a.config, a.n, a.threads)
    if a.sample_n:
        s = timed(a.config, a.sample_n, a.threads)
        out["sample"] = s
        t_extrap = (s["t_factor_s"] + s["t_solve_s"]) * out["full"]["flops"] / s["flops"]
        out["extrapolated_full_s"] = t_extrap
        out["measured_full_s"] = out["full"]["t_factor_s"] + out["full"]["t_solve_s"]
        out["calibration_measured_over_extrapolated"] = out["measured_full_s"] / t_extrap
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
