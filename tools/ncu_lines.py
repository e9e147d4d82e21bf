"""Aggregate an `ncu --page source --csv --print-source cuda,sass` dump by CUDA
source line: warp-stall samples and executed instructions per line, plus the
dominant stall reasons.  Usage: python tools/ncu_lines.py dump.csv [top]"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = None
cur_file = None
cur_line = None
agg = defaultdict(lambda: [0, 0, defaultdict(int), ""])
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 1:
        continue
    if r[0]:
        cur_line = (cur_file, int(r[0]), r[1][:90])
        continue
    if cur_line is None:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ex = int(d.get("Instructions Executed", "0") or 0)
    except ValueError:
        continue
    a = agg[cur_line]
    a[0] += s
    a[1] += ex
    for k, v in d.items():
        if k.startswith("stall_"):
            try:
                a[2][k] += int(v or 0)
            except ValueError:
                pass
tot = sum(a[0] for a in agg.values()) or 1
print("total samples", tot)
for key, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    reasons = sorted(a[2].items(), key=lambda kv: -kv[1])[:3]
    print("%5.1f%% %10d inst  %s:%d  %s | %s" % (100.0 * a[0] / tot, a[1], key[0], key[1], key[2].strip(),
                                                 " ".join("%s=%d" % (k[6:], v) for k, v in reasons)))
