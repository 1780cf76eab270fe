"""Per-sample L2->L1 traffic of the field engine over one frame, from an ncu
metrics capture of every k_field_ws launch of that frame (bench.py reads the
JSON this writes as the source of `roofline_gather.requests_per_sample`):

  ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,\
lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct \
      --clock-control none -k regex:k_field_ws --csv --log-file field.csv \
      python tools/quick_bench.py 3 1920x1080 8 1

  python tools/field_traffic.py field.csv <evaluated samples of that frame> \
      profiles/rNN_field_traffic_cfg3.json cfg3 <commit> [kernel label]

The first k_field_ws launch of a renderer is the occupancy-grid build
(density only), not a march round: it is listed but excluded from the
per-sample totals."""
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
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
ids = sorted(per)
march = ids[1:]                                  # ids[0] = occupancy build
tot = defaultdict(float)
for k in march:
    for m, v in per[k].items():
        tot[m] += v
samples = float(sys.argv[2])
config = sys.argv[4] if len(sys.argv) > 4 else "cfg3"
commit = sys.argv[5] if len(sys.argv) > 5 else None
n = len(march)
SM_CLK, SMS = 1.965e9, 148


def req_per_clk(d):
    dur = d.get("gpu__time_duration.sum", 0.0) * 1e-9
    return d.get("lts__t_requests_srcunit_tex_op_read.sum", 0.0) / (dur * SM_CLK * SMS) if dur > 0 else 0.0


out = {
    "kernel": sys.argv[6] if len(sys.argv) > 6 else "fws::k_field_ws<32,2,T> (T = 2: encode teams, first 3 march rounds of a chunk)",
    "config": config,
    "commit": commit,
    "capture": "ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,"
               "lts__t_requests_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
               "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct "
               "--clock-control none -k regex:k_field_ws (every field-engine launch of one frame; "
               "launch 0 = occupancy build, excluded)",
    "launches": n,
    "samples": int(samples),
    "engine_ms": tot["gpu__time_duration.sum"] * 1e-6,
    "dram_read_bytes": tot["dram__bytes_read.sum"],
    "dram_write_bytes": tot["dram__bytes_write.sum"],
    "dram_bytes_per_launch": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / max(1, n),
    "l2_bytes_per_launch": tot["lts__t_sectors_srcunit_tex_op_read.sum"] * 32.0 / max(1, n),
    "l2_to_l1_sectors": tot["lts__t_sectors_srcunit_tex_op_read.sum"],
    "l2_sectors_per_sample": tot["lts__t_sectors_srcunit_tex_op_read.sum"] / samples,
    "l2_requests_per_sample": tot["lts__t_requests_srcunit_tex_op_read.sum"] / samples,
    "l2_requests_per_sm_clk_frame": tot["lts__t_requests_srcunit_tex_op_read.sum"] /
                                    (tot["gpu__time_duration.sum"] * 1e-9 * SM_CLK * SMS),
    "per_launch": [{"id": k, "ms": round(per[k].get("gpu__time_duration.sum", 0.0) * 1e-6, 4),
                    "l2_requests_per_sm_clk": round(req_per_clk(per[k]), 3),
                    "l1_sector_hit_pct": round(per[k].get("l1tex__t_sector_hit_rate.pct", 0.0), 1)}
                   for k in ids],
    "dram_bytes_per_sample": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / samples,
    "note": ("The 46.5 MiB hash table is L2-resident; DRAM traffic is mostly the sample batch in/out. "
             "The L1 miss path takes ~1 request per clk per SM (hrt_gather_peak); the first, coherent "
             "march rounds (primary rays, 77 % L1 hits) run far below it, the later incoherent rounds "
             "(secondary bounces) at 0.8+ requests/clk/SM.") if config != "cfg4" else
            ("The 344 MiB cfg4 hash table does not fit L2: the finest levels stream from HBM "
             "(dram_bytes_per_sample), the coarse ones stay in L2 / L1."),
}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "per_launch"}, indent=1))
