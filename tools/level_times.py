"""Per-level device times of one factorization (ACRGPU_VERBOSE level events), optionally of a
leading k-plane sub-system -- input of the multi-GPU projection in DESIGN.md §7: with the
contiguous plan_schedule partition, rank 0's share of levels 0 .. log2(n/p) - 1 is the
factorization of the first n/p planes.
    ACRGPU_VERBOSE=1 python tools/level_times.py CONFIG [PLANES] [REPS]"""
import json
import os
import re
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__" and os.environ.get("_LT_CHILD") != "1":
    env = dict(os.environ, _LT_CHILD="1", ACRGPU_VERBOSE="1")
    p = subprocess.run([sys.executable, __file__] + sys.argv[1:], env=env, capture_output=True, text=True)
    lv = {}
    for line in p.stderr.splitlines():
        m = re.search(r"level (\d+): ([0-9.]+) ms", line)
        if m:
            lv.setdefault(int(m.group(1)), []).append(float(m.group(2)))
    out = json.loads(p.stdout.strip().splitlines()[-1]) if p.stdout.strip() else {"error": p.stderr[-2000:]}
    out["level_ms"] = {k: v for k, v in sorted(lv.items())}
    print(json.dumps(out))
    sys.exit(p.returncode)

from paper_1701_00182_b200 import acr, problems as P  # noqa: E402

cfgk = int(sys.argv[1])
planes = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c = P.CONFIGS[cfgk]
sysm = P.config_system(cfgk)
if planes:
    sysm = P.first_planes(sysm, planes)
ctx = acr.Context(0)
dsys = acr.DeviceSystem(sysm, ctx)
cfg = acr.AcrConfig(eps=c["eps"], leaf_size=c["leaf"])
res = []
for r in range(reps):
    f = acr.acr_factor(dsys, cfg)
    res.append(f.timing()["factor_ms"])
    del f
print(json.dumps(dict(config=cfgk, planes=planes or sysm.n, factor_ms=res)))
