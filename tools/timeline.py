"""Pipeline timeline of repeated factorizations (ACRGPU_VERBOSE): python tools/timeline.py CONFIG [REPS]"""
import os, sys, json
os.environ["ACRGPU_VERBOSE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1701_00182_b200 import acr, problems as P
cfgk = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = P.CONFIGS[cfgk]
sysm = P.config_system(cfgk)
ctx = acr.Context(0)
dsys = acr.DeviceSystem(sysm, ctx)
cfg = acr.AcrConfig(eps=c["eps"], leaf_size=c["leaf"])
for r in range(reps):
    f = acr.acr_factor(dsys, cfg)
    print(json.dumps(f.timing()), file=sys.stderr)
    del f
