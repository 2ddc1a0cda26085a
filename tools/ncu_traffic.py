"""Per-launch DRAM traffic of the kernels in an ncu --set full report, as JSON
(the `traffic` field of bench.py's roofline object).

usage: python tools/ncu_traffic.py REPORT.ncu-rep --workload c2:sweep:30000000 > profiles/rNN_traffic.json
"""
import argparse
import csv
import json
import subprocess

p = argparse.ArgumentParser()
p.add_argument("report")
p.add_argument("--workload", required=True, help="config:path the capture ran (bench.py's key)")
a = p.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
tscale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def val(r, key, table):
    i = hdr.index(key)
    return float(r[i].replace(",", "")) * table[units[i]]


kernels = {}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
    rd = val(r, "dram__bytes_read.sum", scale)
    wr = val(r, "dram__bytes_write.sum", scale)
    ms = val(r, "gpu__time_duration.sum", tscale)
    ent = {"dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes": rd + wr, "ms": ms}
    for key, col in (("pipe_alu_pct", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                     ("pipe_fma_pct", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                     ("issue_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     ("warp_inst", "smsp__inst_executed.sum")):
        if col in hdr:
            ent[key] = float(r[hdr.index(col)].replace(",", ""))
    kernels.setdefault(name, []).append(ent)
res = {"workload": a.workload, "source": a.report.split("/")[-1],
       "method": "ncu --set full --clock-control none, one capture per launch",
       "kernels": {k: {"launches": len(v),
                       "traffic_bytes_per_launch": sum(x["traffic_bytes"] for x in v) / len(v),
                       "dram_read_bytes_per_launch": sum(x["dram_read_bytes"] for x in v) / len(v),
                       "dram_write_bytes_per_launch": sum(x["dram_write_bytes"] for x in v) / len(v),
                       "ms_per_launch_under_ncu": sum(x["ms"] for x in v) / len(v),
                       **{k: sum(x[k] for x in v) / len(v) for k in
                          ("pipe_alu_pct", "pipe_fma_pct", "issue_pct", "warp_inst") if k in v[0]}}
                   for k, v in kernels.items()}}
print(json.dumps(res, indent=1))
