"""Summarise an ncu source page (--print-source=cuda,sass --csv): per CUDA source line, the warp-stall
samples and executed instructions, top-N lines, plus per-line top stall reasons."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hdr_i]
src_line = {}
samples = defaultdict(float)
insts = defaultdict(float)
stalls = defaultdict(lambda: defaultdict(float))
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
si = hdr.index("Warp Stall Sampling (All Samples)")
ii = hdr.index("Instructions Executed")
line = None
for r in rows[hdr_i + 1:]:
    if not r:
        continue
    if r[0] and r[0].isdigit():
        line = int(r[0])
        src_line[line] = r[1]
    if len(r) > ii and r[2]:
        try:
            samples[line] += float(r[si] or 0)
            insts[line] += float(r[ii] or 0)
            for c in stall_cols:
                stalls[line][hdr[c]] += float(r[c] or 0)
        except ValueError:
            pass
tot = sum(samples.values()) or 1
tot_i = sum(insts.values()) or 1
print(f"total samples {tot:.0f}, warp instructions {tot_i:.0f}")
for l, s in sorted(samples.items(), key=lambda x: -x[1])[:topn]:
    top = sorted(stalls[l].items(), key=lambda x: -x[1])[:3]
    ts = " ".join(f"{k[6:]}={v / max(s, 1):.0%}" for k, v in top)
    print(f"{l:5d} {100 * s / tot:5.1f}% smp {100 * insts[l] / tot_i:5.1f}% inst | {src_line.get(l, '')[:70]:70s} | {ts}")
