"""Generate the full-size oracle fixtures the GPU parity tests compare against.

TEST INFRASTRUCTURE ONLY: runs the CPU oracle (oracle/acr_oracle.cpp, the restatement of
/root/reference/proj/core/src/acr.cpp:146-229 + hmatrix.cpp) on a BASELINE config at its
stated size and records what the north_star bar is stated on:

  * relative residual ||f - A u|| / ||f|| of the solve (block.cpp:109-123),
  * inverse rank statistics and factor bytes (acr.cpp:231-258),
  * per-level largest / average rank (level_info, acr.cpp:260-300),
  * leaf-by-leaf ranks of the stored inverses of planes {0, 1, last} at every level
    (rank_stats walk, hmatrix.cpp:538-554),
  * u at 1024 seeded sample positions (solution comparison without shipping 2 MB).

Usage:  python tests/golden/make_oracle_fixtures.py --config 3 --threads 3
Writes tests/golden/oracle_c<k>_n<n>.json.  Run once on the build container (C2-C4 at n=64
take 25-60 min each); the GPU tests read the JSON only (no oracle at run time).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_1701_00182_b200 import problems as P  # noqa: E402

SAMPLE_SEED = 77


def sample_index(n_total: int, count: int = 1024) -> np.ndarray:
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n_total, size=min(count, n_total), replace=False))


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--threads", type=int, default=4)
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--planes", type=int, default=None,
                    help="factor only the leading k x k block sub-system (first_planes); its stored "
                         "inverses at eliminated positions < 2^(l+1)-1 of level l equal the full system's")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    c = P.CONFIGS[a.config]
    n = c["n"] if a.n is None else a.n
    sysm = P.config_system(a.config, n=n, seed=a.seed)
    if a.planes:
        sysm = P.first_planes(sysm, a.planes)
    t0 = time.time()
    fac = O.Factorization(sysm, eps=c["eps"], leaf_size=c["leaf"], threads=a.threads)
    tf = time.time() - t0
    t0 = time.time()
    u = fac.solve(sysm.rhs)
    ts = time.time() - t0
    res = float(sysm.relative_residual(u))
    levels = fac.level_info()
    dinv = []
    for li, lv in enumerate(levels):
        m = lv["plane_count"]
        for j in (range(m) if a.planes else sorted({0, 1, m - 1})):
            r = fac.dinv_ranks(li, j)
            if r is not None:
                dinv.append(dict(level=li, plane=j, ranks=[int(x) for x in r]))
    flat = np.asarray(u).reshape(-1)
    idx = sample_index(flat.size)
    out = dict(
        config=a.config, n=n, planes=a.planes, seed=a.seed, eps=c["eps"], leaf=c["leaf"], kind=c["kind"],
        residual=res, stats=fac.stats(), levels=levels, dinv_ranks=dinv,
        u_norm=float(np.linalg.norm(flat)), u_sample_index=[int(i) for i in idx],
        u_sample=[float(x) for x in flat[idx]],
        t_factor_s=tf, t_solve_s=ts, threads=a.threads, cpu=cpu_model(), nproc=os.cpu_count(),
        generator="tests/golden/make_oracle_fixtures.py",
    )
    tag = f"_p{a.planes}" if a.planes else ""
    path = a.out or os.path.join(HERE, f"oracle_c{a.config}_n{n}{tag}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {path}: residual {res:.6e} largest {out['stats']['largest_rank']} "
          f"avg {out['stats']['average_rank']:.6f} factor {tf:.1f} s solve {ts:.2f} s")


if __name__ == "__main__":
    main()
