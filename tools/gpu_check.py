import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1701_00182_b200 import acr, problems as P
from oracle import oracle as O

def run(sysm, eps, leaf=32, **kw):
    cfg = acr.AcrConfig(eps=eps, leaf_size=leaf, **kw)
    t = time.time(); f = acr.acr_factor(sysm, cfg); tf = time.time() - t
    t = time.time(); u = f.solve(sysm.rhs); ts = time.time() - t
    st = f.inverse_rank_stats()
    return dict(res=sysm.relative_residual(u), tf=tf, ts=ts, largest=st.largest_rank, avg=st.average_rank,
                fbytes=f.factor_bytes(), timing=f.timing()), f, u

cases = [("poisson8", P.poisson(8), 1e-3), ("poisson16", P.poisson(16), 1e-3), ("poisson16_1e-6", P.config_system(1, n=16), 1e-6)]
if len(sys.argv) > 1 and sys.argv[1] == "c1":
    cases.append(("C1", P.config_system(1), 1e-6))
for name, sysm, eps in cases:
    try:
        g, f, u = run(sysm, eps)
    except Exception as e:
        print(name, "GPU ERROR", type(e).__name__, e, flush=True); continue
    t = time.time(); of = O.Factorization(sysm, eps=eps, threads=16); uo = of.solve(sysm.rhs); to = time.time() - t
    os_ = of.stats()
    print(json.dumps(dict(case=name, gpu=g, oracle=dict(res=sysm.relative_residual(uo), largest=os_["largest_rank"], avg=os_["average_rank"], fbytes=os_["factor_bytes"], t=to),
                          udiff=float(np.linalg.norm(u - uo) / np.linalg.norm(uo)))), flush=True)
    print("levels gpu", [(l.largest_rank, round(l.average_rank, 2)) for l in f.level_info()])
    print("levels orc", [(l["largest_rank"], round(l["average_rank"], 2)) for l in of.level_info()], flush=True)
