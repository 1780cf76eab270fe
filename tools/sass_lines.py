"""Dev aid: warp-stall samples of an ncu capture aggregated per CUDA source
line (the ncu CUDA-source page of these reports carries no metrics, so the
SASS page is mapped through nvdisasm's line table of the same library).

  ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
  python tools/sass_lines.py sass.csv path/to/libhrt.so <mangled kernel name> [top]
(per line: share of stall samples, instructions executed, top two stall reasons)
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

sass_csv, lib, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30

rows = list(csv.reader(open(sass_csv)))
h = rows[1]
ai, ci = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
si = [k for k, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
samples = []
for r in rows[2:]:
    if len(r) > ci and r[ai].startswith("0x"):
        samples.append((int(r[ai], 16), float(r[ci] or 0), float(r[ei] or 0),
                        [float(r[k] or 0) for k in si]))
base = samples[0][0]

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True,
               stdout=subprocess.DEVNULL)
cubin = next(os.path.join(tmp, f) for f in os.listdir(tmp) if f.startswith("hrt.") and f.endswith(".cubin"))
dis = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
sec = dis.split(f".text.{kern}:", 1)[1].split("//---------------------", 1)[0]
line_of = {}
cur = None
for ln in sec.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg, inst = defaultdict(float), defaultdict(float)
why = defaultdict(lambda: [0.0] * len(si))
for addr, s, e, st in samples:
    k = line_of.get(addr - base, "?")
    agg[k] += s
    inst[k] += e
    why[k] = [a + b for a, b in zip(why[k], st)]
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    w = why[k]
    tw = sum(w) or 1
    top2 = sorted(range(len(si)), key=lambda x: -w[x])[:2]
    reasons = " ".join(f"{h[si[x]][6:]} {100 * w[x] / tw:.0f}%" for x in top2)
    print(f"{100 * v / tot:5.1f}%  {k:28s} inst {inst[k]:.3g}  [{reasons}]")
