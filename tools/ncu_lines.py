"""Aggregate ncu warp-stall samples per CUDA source line (from --page source --print-source cuda,sass CSV)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
agg = collections.Counter(); tot = 0; fname = None; cur = None; hdr = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; iS = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None or len(r) < 5: continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:100])
        continue
    try: v = float(r[iS])
    except ValueError: continue
    agg[cur] += v; tot += v
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print("%5.1f%%  %s:%d  %s" % (100 * v / tot, k[0], k[1], k[2]))
