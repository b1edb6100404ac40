"""Hot instructions of an ncu --page source CSV (gzip ok): top PCs by stall
samples with their dominant stall reasons and the preceding instructions.

    python scripts/ncu_hot.py prof_source.csv.gz [N]
"""
import csv
import gzip
import sys

f = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
op = gzip.open if f.endswith(".gz") else open
r = csv.reader(op(f, "rt"))
next(r)
h = next(r)
rows = [x for x in r if len(x) == len(h)]
ia, sa, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(x[sa]) for x in rows)
print(f"samples {tot}, warp instructions {sum(int(x[ia]) for x in rows)}")
agg = {c: sum(int(x[h.index(c)]) for x in rows) for c in reasons}
print("by reason:", sorted(((v, c) for c, v in agg.items() if v), reverse=True)[:8])
order = sorted(range(len(rows)), key=lambda i: -int(rows[i][sa]))[:n]
for i in order:
    x = rows[i]
    rs = sorted(((int(x[h.index(c)]), c[6:]) for c in reasons if int(x[h.index(c)])), reverse=True)[:3]
    print(f"{int(x[sa]):6d} {int(x[ia]):9d}  {x[src].strip()[:60]:60s} {rs}")
    for j in range(max(0, i - 2), i):
        print(f"{'':17s}  prev: {rows[j][src].strip()[:60]}")
