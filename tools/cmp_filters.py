"""Time the filter kernels against each other per (L, e) on device-generated pairs.

usage: python tools/cmp_filters.py --L 250 --n 30000000 --e 5 12 25 --flags 0 4
Prints one JSON line per (L, e, flags): ms (median of reps, CUDA events), Gpairs/s,
ALU fraction against the DESIGN.md algorithmic op count, and an accept-bit checksum
(identical across flags or the kernels disagree).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import pairgen  # noqa: E402
import paper_2103_14978_b200 as gk  # noqa: E402

ALU_PEAK = 148 * 64 * 1.965e9


def ops_per_pair(L, e):
    return (5 * (L * (2 * e + 1) - e * (e + 1)) + 8 * L) / 32.0


p = argparse.ArgumentParser()
p.add_argument("--L", type=int, default=250)
p.add_argument("--n", type=int, default=30_000_000)
p.add_argument("--e", type=int, nargs="+", default=[12, 25])
p.add_argument("--flags", type=int, nargs="+", default=[0, 4])
p.add_argument("--reps", type=int, default=5)
a = p.parse_args()
r, f = pairgen.gen_pairs_cuda(a.n, a.L)
q, uq = gk.encode(r, a.L)
s, us = gk.encode(f, a.L)
del r, f
torch.cuda.synchronize()
acc = torch.empty(gk.result_words(a.n), dtype=torch.int32, device="cuda")
err = torch.empty(a.n, dtype=torch.uint8, device="cuda")
for e in a.e:
    if e >= a.L:
        continue
    sums = {}
    for fl in a.flags:
        gk.filter(q, s, uq, us, a.n, a.L, e, accept=acc, errcount=err, flags=fl)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            gk.filter(q, s, uq, us, a.n, a.L, e, accept=acc, errcount=err, flags=fl)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        chk = int(acc.to(torch.int64).sum().item()) ^ (int(err.to(torch.int64).sum().item()) << 20)
        sums[fl] = chk
        gps = a.n / ms / 1e6
        print(json.dumps({"L": a.L, "e": e, "flags": fl, "ms": round(ms, 4),
                          "Gpairs_s": round(gps, 3),
                          "alu_frac": round(gps * 1e9 * ops_per_pair(a.L, e) / ALU_PEAK, 4),
                          "checksum": chk}), flush=True)
    if len(set(sums.values())) != 1:
        print(json.dumps({"L": a.L, "e": e, "MISMATCH": sums}), flush=True)
