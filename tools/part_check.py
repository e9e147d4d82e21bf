"""Partitioned (multi-rank) factor/solve on one GPU via in-process ranks: bitwise
comparison with the single-rank path (test_parallel.cpp:75-89 contract)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1701_00182_b200 import acr, problems as P

cases = [("poisson16", P.poisson(16), 1e-3), ("C1", P.config_system(1), 1e-6)]
if len(sys.argv) > 1:
    cases = [c for c in cases if c[0] in sys.argv[1:]] or cases
for name, s, eps in cases:
    cfg = acr.AcrConfig(eps=eps)
    f1 = acr.acr_factor(s, cfg)
    u1 = f1.solve(s.rhs)
    st1 = f1.inverse_rank_stats()
    for p in (1, 2, 4, 8):
        if p > s.n:
            continue
        comm = acr.Comm.local_ranks(p)
        t = time.time()
        fp = acr.acr_factor_partitioned(s, comm, cfg)
        tf = time.time() - t
        up = fp.solve(s.rhs)
        stp = fp.inverse_rank_stats()
        print(json.dumps(dict(case=name, p=p, bitwise=bool(np.array_equal(u1, up)),
                              maxdiff=float(np.max(np.abs(u1 - up))), res=s.relative_residual(up),
                              res1=s.relative_residual(u1), avg=stp.average_rank, avg1=st1.average_rank,
                              largest=stp.largest_rank, bytes=fp.factor_bytes(), bytes1=f1.factor_bytes(),
                              levels=[(l.largest_rank, round(l.average_rank, 3)) for l in fp.level_info()] ==
                              [(l.largest_rank, round(l.average_rank, 3)) for l in f1.level_info()],
                              tf=tf)), flush=True)
        del fp
