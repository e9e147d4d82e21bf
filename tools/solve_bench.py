"""Solve throughput against the HBM roofline: factor one BASELINE config once, then time
repeated solves (device events of the library stream) and the two matvec kernels.

    python tools/solve_bench.py CONFIG [N] [REPS]

Algorithmic bytes of a solve = every stored entry of every H-matrix the solve applies,
read once (k_mv_t reads V, k_mv_slab reads U and the dense leaves); each entry takes part in
2*nrhs flops, so bytes = 8 * apply_flops / (2 * nrhs)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1701_00182_b200 import acr, problems as P  # noqa: E402

cfgk = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
c = P.CONFIGS[cfgk]
sysm = P.config_system(cfgk, n=n)
nrhs = sysm.rhs.shape[0]
ctx = acr.Context(0)
dsys = acr.DeviceSystem(sysm, ctx)
f = acr.acr_factor(dsys, acr.AcrConfig(eps=c["eps"], leaf_size=c["leaf"]))
f_dev = torch.from_numpy(np.ascontiguousarray(sysm.rhs)).cuda()
u_dev = torch.empty_like(f_dev)
f.solve_device(f_dev.data_ptr(), u_dev.data_ptr(), nrhs)
res = sysm.relative_residual(u_dev.cpu().numpy())
acr.profile_report(reset=True)
acr.profile_select("k_mv_t,k_mv_slab,k_mv_resolve")
ms = []
for _ in range(reps):
    f.solve_device(f_dev.data_ptr(), u_dev.data_ptr(), nrhs)
    ms.append(f.timing()["solve_ms"])
torch.cuda.synchronize()
rows = {}
for line in acr.profile_report(reset=True).splitlines():
    p = line.split()
    if line.startswith("#phase mv") or line.startswith("#top"):
        print(line, file=sys.stderr)
    if line.startswith("#") or len(p) < 5:
        continue
    rows[p[0]] = dict(ms=float(p[1]) / reps, launches=int(p[2]) // reps, flops=float(p[4]) / reps)
acr.profile_select(None)
fl = sum(r["flops"] for r in rows.values())
kms = sum(r["ms"] for r in rows.values())  # k_mv_t + k_mv_resolve (records, packed x) + k_mv_slab
bytes_h = 8.0 * fl / (2.0 * nrhs)
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
out = dict(config=cfgk, n=sysm.n, nrhs=nrhs, residual=res, solve_ms=sorted(ms)[len(ms) // 2], solve_ms_all=ms,
           kernels=rows, h_bytes=bytes_h, matvec_kernel_ms=kms,
           achieved_gbs_kernels=bytes_h / (kms / 1e3) / 1e9 if kms > 0 else None,
           achieved_gbs_solve=bytes_h / (sorted(ms)[len(ms) // 2] / 1e3) / 1e9, hbm_peak_gbs=peak)
out["frac_kernels"] = out["achieved_gbs_kernels"] / peak if out["achieved_gbs_kernels"] else None
out["frac_solve"] = out["achieved_gbs_solve"] / peak
print(json.dumps(out), flush=True)
