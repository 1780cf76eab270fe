"""Dev aid: top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
h = r[1]
ci = h.index("Warp Stall Sampling (All Samples)")
si = h.index("Source")
rows = []
for x in r[2:]:
    if len(x) > ci:
        try:
            rows.append((float(x[ci] or 0), x[0], x[si]))
        except ValueError:
            pass
tot = sum(a for a, _, _ in rows) or 1
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for a, ad, s in sorted(rows, reverse=True)[:n]:
    print(f"{100 * a / tot:5.1f}% {ad} {s}")
