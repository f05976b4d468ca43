"""Summarise ncu --page source --csv output: top source lines by warp-stall samples."""
import csv, sys
r = list(csv.reader(open(sys.argv[1])))
# find header line containing 'Warp Stall Sampling'
hi = next(i for i, x in enumerate(r) if any('Warp Stall Sampling (All' in c for c in x))
hdr = r[hi]
si = next(i for i, h in enumerate(hdr) if h.startswith('Warp Stall Sampling (All'))
li = hdr.index('# Line') if '# Line' in hdr else 0
srci = hdr.index('Source')
rows = []
for x in r[hi + 1:]:
    if len(x) <= si:
        continue
    try:
        v = float(x[si] or 0)
    except ValueError:
        continue
    rows.append((v, x[li], x[srci][:100]))
tot = sum(v for v, _, _ in rows) or 1
for v, l, s in sorted(rows, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{100*v/tot:5.1f}% {l:>5} {s}")
