"""Dev aid: per-sample L2->L1 traffic of the field engine over one cfg1 frame,
from an ncu metrics capture of every k_field_ws launch of the frame:

  ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,\
lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:k_field_ws --launch-skip 1 --csv \
      --log-file field.csv python tools/quick_bench.py 1 800x800 1 1

python tools/field_traffic.py field.csv <evaluated samples of that frame> out.json"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
head = rows[h]
ii, mi, vi = head.index("ID"), head.index("Metric Name"), head.index("Metric Value")
per = defaultdict(dict)
for r in rows[h + 1:]:
    if len(r) == len(head):
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
tot = defaultdict(float)
for d in per.values():
    for k, v in d.items():
        tot[k] += v
samples = float(sys.argv[2])
n = len(per)
out = {
    "kernel": "fws::k_field_ws<32,2>",
    "capture": "ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,"
               "lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum "
               "--clock-control none -k regex:k_field_ws --launch-skip 1 python tools/quick_bench.py 1 800x800 1 1 "
               "(every field-engine launch of one cfg1 frame)",
    "launches": n,
    "samples": int(samples),
    "dram_read_bytes": tot["dram__bytes_read.sum"],
    "dram_write_bytes": tot["dram__bytes_write.sum"],
    "dram_bytes_per_launch": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / max(1, n),
    "l2_to_l1_sectors": tot["lts__t_sectors_srcunit_tex_op_read.sum"],
    "l2_sectors_per_sample": tot["lts__t_sectors_srcunit_tex_op_read.sum"] / samples,
    "l2_requests_per_sample": tot["lts__t_requests_srcunit_tex_op_read.sum"] / samples,
    "note": "The 46.5 MiB hash table is L2-resident; DRAM traffic is mostly the sample batch in/out. "
            "The L1 miss path is bound by requests (~1 per clk per SM, hrt_gather_peak and "
            "tools/gather_paths_probe.cu); per sample the encode issues the requests above.",
}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out, indent=1))
