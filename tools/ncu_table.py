"""Dev aid: key ncu `--set full` metrics of several reports side by side
(markdown), as quoted in profiles/r02_summary.md.
usage: python tools/ncu_table.py label1=rep1.ncu-rep label2=rep2.ncu-rep ..."""
import csv
import io
import subprocess
import sys

WANT = [("duration (ms)", "gpu__time_duration.sum"), ("SM issue active %", "sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
        ("L1TEX throughput %", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L1->L2 request path busy %", "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("LSU data pipe %", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        ("TEX data pipe %", "l1tex__data_pipe_tex_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        ("L1 sector hit %", "l1tex__t_sector_hit_rate.pct"), ("L2 sector hit %", "lts__t_sector_hit_rate.pct"),
        ("DRAM throughput %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("tensor pipe active %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("registers / thread", "launch__registers_per_thread"),
        ("L2 read requests (M)", "lts__t_requests_srcunit_tex_op_read.sum")]
UNIT = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}

cols = []
for arg in sys.argv[1:]:
    label, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {}
    for name, k in WANT:
        i = h.index(k)
        x = float(v[i].replace(",", ""))
        if k == "gpu__time_duration.sum":
            x *= UNIT.get(u[i], 1.0)
        if k.startswith("lts__t_requests"):
            x *= 1e-6
        d[name] = x
    d["L2 requests / clk / SM"] = d["L2 read requests (M)"] * 1e6 / (d["duration (ms)"] * 1e-3 * 1.965e9 * 148)
    cols.append((label, d))
names = [w[0] for w in WANT] + ["L2 requests / clk / SM"]
print("| metric | " + " | ".join(lbl for lbl, _ in cols) + " |")
print("|---|" + "---:|" * len(cols))
for n in names:
    print(f"| {n} | " + " | ".join(f"{d[n]:.3g}" for _, d in cols) + " |")
