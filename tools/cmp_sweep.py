"""Time gk_filter_sweep (one pass, e = 0..e_max) against e_max+1 gk_filter launches
on device-generated pairs, and check that every row agrees.

usage: python tools/cmp_sweep.py --L 100 --emax 10 [--n 30000000]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import pairgen  # noqa: E402
import paper_2103_14978_b200 as gk  # noqa: E402


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


p = argparse.ArgumentParser()
p.add_argument("--L", type=int, default=100)
p.add_argument("--n", type=int, default=30_000_000)
p.add_argument("--emax", type=int, nargs="+", default=[10])
p.add_argument("--reps", type=int, default=5)
a = p.parse_args()
r, f = pairgen.gen_pairs_cuda(a.n, a.L)
q, uq = gk.encode(r, a.L)
s, us = gk.encode(f, a.L)
del r, f
for emax in a.emax:
    acc, err = gk.filter_sweep(q, s, uq, us, a.n, a.L, emax)
    ms_sweep = timed(lambda: gk.filter_sweep(q, s, uq, us, a.n, a.L, emax, accept=acc, errcount=err), a.reps)
    a1 = torch.empty(gk.result_words(a.n), dtype=torch.int32, device="cuda")
    c1 = torch.empty(a.n, dtype=torch.uint8, device="cuda")
    ms_each, same = 0.0, True
    for e in range(emax + 1):
        ms_each += timed(lambda: gk.filter(q, s, uq, us, a.n, a.L, e, accept=a1, errcount=c1), max(1, a.reps // 2))
        same = same and torch.equal(acc[e], a1) and torch.equal(err[e], c1)
    print(json.dumps({"L": a.L, "emax": emax, "n": a.n, "ms_sweep": round(ms_sweep, 4),
                      "ms_per_e_sum": round(ms_each, 4),
                      "Gfiltrations_s_sweep": round(a.n * (emax + 1) / ms_sweep / 1e6, 2),
                      "Gfiltrations_s_per_e": round(a.n * (emax + 1) / ms_each / 1e6, 2),
                      "rows_identical": bool(same)}), flush=True)
