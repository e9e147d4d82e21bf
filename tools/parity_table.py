"""GPU vs oracle at full size, from the committed oracle fixtures (tests/golden/): residual,
largest / average inverse rank, factor bytes, per-level ranks and the stored-inverse leaf
ranks leaf by leaf.  Writes one JSON object (DESIGN.md §3's table).
    python tools/parity_table.py > profiles/r02_parity_table.json"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from paper_1701_00182_b200 import acr, problems as P  # noqa: E402
from test_gpu_fullsize import window_entries  # noqa: E402

rows = []
for path in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "oracle_c*.json"))):
    fx = json.load(open(path))
    sysm = P.config_system(fx["config"], n=fx["n"], seed=fx["seed"])
    full_c5 = fx.get("planes")
    cases = [("sub-system", P.first_planes(sysm, fx["planes"]), None)] if full_c5 else [("full", sysm, None)]
    if full_c5:
        cases.append(("full system, shared inverses", sysm, window_entries(fx)))
    for what, s, entries in cases:
        f = acr.acr_factor(s, acr.AcrConfig(eps=fx["eps"], leaf_size=fx["leaf"]))
        u = f.solve(s.rhs)
        st = f.inverse_rank_stats()
        tot = eq = off = 0
        for d in fx["dinv_ranks"]:
            if entries is not None and (d["level"], d["plane"]) not in entries:
                continue
            g = f.dinv_ranks(d["level"], d["plane"])
            o = np.asarray(d["ranks"])
            lr = o >= 0
            tot += int(lr.sum())
            eq += int((g == o)[lr].sum())
            off += int((np.abs(g - o)[lr] > 1).sum())
        row = dict(fixture=os.path.basename(path), case=what, N=s.total_dim, nrhs=int(s.rhs.shape[0]),
                   residual_gpu=float(s.relative_residual(u)),
                   leaf_ranks_compared=tot, leaf_ranks_equal=eq, leaf_ranks_off_by_more_than_1=off)
        if entries is None:
            row.update(residual_oracle=fx["residual"], largest_gpu=st.largest_rank, largest_oracle=fx["stats"]["largest_rank"],
                       average_gpu=st.average_rank, average_oracle=fx["stats"]["average_rank"],
                       factor_bytes_gpu=f.factor_bytes(), factor_bytes_oracle=fx["stats"]["factor_bytes"],
                       levels_gpu=[(l.largest_rank, round(l.average_rank, 4)) for l in f.level_info()],
                       levels_oracle=[(l["largest_rank"], round(l["average_rank"], 4)) for l in fx["levels"]],
                       oracle_threads=fx["threads"], oracle_factor_s=fx["t_factor_s"])
            flat = np.asarray(u).reshape(-1)
            idx = np.asarray(fx["u_sample_index"])
            us = np.asarray(fx["u_sample"])
            row["u_sample_rel_diff"] = float(np.linalg.norm(flat[idx] - us) / np.linalg.norm(us))
        rows.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
        del f
print(json.dumps(dict(rows=rows), indent=1))
