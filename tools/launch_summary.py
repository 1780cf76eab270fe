"""Summarize an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launches, total time and share (the same numbers DESIGN.md and
profiles/*.md quote)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if r[0] == "ID")
head = rows[h]
ki, mi, vi, ui = (head.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[h + 1:]:
    if len(r) != len(head) or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[ui], 1e-6)
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += v * scale
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"| kernel | launches | total ms | share |\n|---|---:|---:|---:|")
for k in sorted(tot, key=tot.get, reverse=True):
    print(f"| `{k}` | {cnt[k]} | {tot[k]:.3f} | {100 * tot[k] / all_ms:.1f} % |")
print(f"| all | {sum(cnt.values())} | {all_ms:.3f} | 100 % |")
