import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1701_00182_b200 import acr, problems as P
cfgk = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
exact = len(sys.argv) > 3 and sys.argv[3] == "exact"
planes = int(os.environ.get("PLANES", "0"))
sysm = P.config_system(cfgk, n=n)
if planes:
    sysm = P.first_planes(sysm, planes)
c = P.CONFIGS[cfgk]
cfg = acr.AcrConfig(eps=c["eps"], leaf_size=c["leaf"], exact_dense_products=exact)
acr.default_context()
t = time.time(); f = acr.acr_factor(sysm, cfg); tf = time.time() - t
t = time.time(); u = f.solve(sysm.rhs); ts = time.time() - t
st = f.inverse_rank_stats()
print(json.dumps(dict(cfg=cfgk, n=sysm.n, exact=exact, res=sysm.relative_residual(u), tf=tf, ts=ts, largest=st.largest_rank,
                      avg=st.average_rank, fbytes=f.factor_bytes(), timing=f.timing())))
rep = acr.profile_report()
rows = [l.split() for l in rep.strip().splitlines() if not l.startswith('#')]
top = [l for l in rep.strip().splitlines() if l.startswith('#')]
tot = sum(float(r[1]) for r in rows)
for r in sorted(rows, key=lambda r: -float(r[1])):
    fl = float(r[4]) if len(r) > 4 else 0.0
    print("%-18s %10.2f ms %5.1f%%  launches %7s  ctas %10s  %7.2f TF/s" % (r[0], float(r[1]), 100 * float(r[1]) / tot, r[2], r[3],
                                                                      fl / float(r[1]) / 1e9 if float(r[1]) > 0 else 0))
print("total kernel ms", tot)
print("\n".join(top[:25]))
