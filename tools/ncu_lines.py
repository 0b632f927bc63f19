"""Per (file, line) instruction / sample totals from an ncu source-page CSV (cuda,sass)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur = "?"
hdr = None
agg_i = defaultdict(float)
agg_s = defaultdict(float)
src = {}
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ii = hdr.index("Instructions Executed")
        continue
    if hdr is None:
        continue
    if r[0].isdigit():
        line = (cur, int(r[0]))
        src[line] = r[1]
    if len(r) > ii and r[2]:
        try:
            agg_i[line] += float(r[ii] or 0)
            agg_s[line] += float(r[si] or 0)
        except ValueError:
            pass
ti = sum(agg_i.values()) or 1
ts = sum(agg_s.values()) or 1
byfile = defaultdict(float)
for k, v in agg_i.items():
    byfile[k[0]] += v
print("instructions by file:", {k: f"{100 * v / ti:.1f}%" for k, v in byfile.items()})
for k, v in sorted(agg_i.items(), key=lambda x: -x[1])[:topn]:
    print(f"{k[0]:22s}:{k[1]:4d} {100 * v / ti:5.1f}% inst {100 * agg_s[k] / ts:5.1f}% smp | {src.get(k, '')[:80]}")
