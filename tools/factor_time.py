"""Factor (+ solve) wall/device time of one BASELINE config, for A/B runs of kernel variants.
    python tools/factor_time.py CONFIG [N] [REPS]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1701_00182_b200 import acr, problems as P  # noqa: E402

cfgk = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c = P.CONFIGS[cfgk]
sysm = P.config_system(cfgk, n=n)
ctx = acr.Context(0)
dsys = acr.DeviceSystem(sysm, ctx)
cfg = acr.AcrConfig(eps=c["eps"], leaf_size=c["leaf"])
for r in range(reps):
    f = acr.acr_factor(dsys, cfg)
    u = f.solve(sysm.rhs)
    t = f.timing()
    st = f.inverse_rank_stats()
    print(json.dumps(dict(config=cfgk, n=sysm.n, rep=r, factor_ms=t["factor_ms"], solve_ms=t["solve_ms"],
                          residual=sysm.relative_residual(u), largest=st.largest_rank, avg=st.average_rank,
                          launches=t["factor_launches"], variant=os.environ.get("ACRGPU_QR_VARIANT", "0"))), flush=True)
    del f
