"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
total time, launches and share of the summed kernel time.  These times are cold-cache
and serialised (ncu), so only the SHARES are comparable with bench.py's live
per-kernel CUDA-event breakdown.  Usage: python tools/launch_shares.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict

NAMES = {  # template instantiations -> the launch names bench.py reports
    r"k_small32<0>": "k_trunc_small32", r"k_small32<1>": "k_dd_small32",
    r"k_truncate<64, 64, 256": "k_trunc_mid64", r"k_truncate<128, 56, 512": "k_trunc_d128|k_trunc_qr",
}


def short(name):
    for pat, s in NAMES.items():
        if pat in name:
            return s
    return re.sub(r"\(.*", "", name).replace("void ", "")


acc = defaultdict(lambda: [0.0, 0])
with open(sys.argv[1]) as fh:
    lines = [l for l in fh if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    ns = float(r["Metric Value"].replace(",", ""))
    a = acc[short(r["Kernel Name"])]
    a[0] += ns / 1e6
    a[1] += 1
tot = sum(a[0] for a in acc.values())
print(f"# {sum(a[1] for a in acc.values())} launches, {tot:.1f} ms summed kernel time (serialised, cold cache)")
for k, (ms, n) in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:28s} {ms:10.2f} ms {100 * ms / tot:6.1f}%  launches {n:6d}")
