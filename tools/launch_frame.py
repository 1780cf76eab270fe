"""Dev aid: the kernel sequence (name:us) of the last full frame in an ncu
`gpu__time_duration.sum` launch list (frames run k_raygen .. k_accumulate)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
head = rows[h]
ki, vi, ui = head.index("Kernel Name"), head.index("Metric Value"), head.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
seq = []
for r in rows[h + 1:]:
    if len(r) != len(head):
        continue
    n = r[ki].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
    seq.append((n, float(r[vi].replace(",", "")) * scale[r[ui]]))
frames, cur = [], None
for n, v in seq:
    if n == "k_raygen":
        cur = []
    if cur is not None:
        cur.append((n, v))
    if n == "k_accumulate" and cur is not None:
        frames.append(cur)
        cur = None
f = frames[-1]
print(f"{len(f)} launches, {sum(v for _, v in f):.0f} us of kernels")
print(" ".join(f"{n.replace('k_', '')}:{v:.0f}" for n, v in f))
