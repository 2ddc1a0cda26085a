"""Instruction mix (executed warp instructions per opcode) and stall samples of one
kernel from an ncu report's SASS source page.

usage: python tools/ncu_sass_mix.py REPORT.ncu-rep [--top 25]
"""
import argparse
import csv
import subprocess
from collections import defaultdict

p = argparse.ArgumentParser()
p.add_argument("report")
p.add_argument("--top", type=int, default=25)
a = p.parse_args()
out = subprocess.run(["ncu", "-i", a.report, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ops = defaultdict(lambda: [0, 0])
stalls = defaultdict(int)
total = 0
for r in rows[2:]:
    if len(r) <= iex or not r[iex].isdigit():
        continue
    op = r[isrc].strip().split()[0] if r[isrc].strip() else "?"
    if op.startswith("@"):
        op = r[isrc].strip().split()[1]
    op = op.split(".")[0]
    n = int(r[iex])
    ops[op][0] += n
    ops[op][1] += int(r[isamp] or 0)
    total += n
    for i in stall_cols:
        stalls[hdr[i]] += int(r[i] or 0)
print(f"{'opcode':12s} {'warp_inst':>14s} {'share':>7s} {'stall_samples':>13s}")
for op, (n, s) in sorted(ops.items(), key=lambda x: -x[1][0])[:a.top]:
    print(f"{op:12s} {n:14d} {n / total:7.3f} {s:13d}")
print("total", total)
tot_s = sum(stalls.values())
print("stall reasons (share of samples):",
      ", ".join(f"{k[6:]} {v / tot_s:.2f}" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]))
