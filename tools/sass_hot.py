"""Top stall-sampled SASS lines of an ncu source-page CSV: python tools/sass_hot.py file.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr, data = rows[hi], rows[hi + 1:]
si, ai = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Address")
srci = hdr.index("Source")
tot = sum(float(r[si] or 0) for r in data if len(r) > si)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
idx = {r[ai]: k for k, r in enumerate(data)}
top = sorted(data, key=lambda r: -float(r[si] or 0))[:n]
for r in top:
    k = idx[r[ai]]
    prev = data[k - 1][srci] if k else ""
    print(f"{100 * float(r[si]) / tot:5.1f}%  {r[ai]}  {r[srci][:70]:70s} | prev: {prev[:50]}")
