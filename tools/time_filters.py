#!/usr/bin/env python
"""A/B timing of the filter kernels on resident packed pairs (CUDA events, median of
reps).  Variant libraries are built with tools/ab_build.py (GK_LIB selects one).

    GK_LIB=... python tools/time_filters.py --L 250 --e 12 --sweep 25 --n 30000000
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import pairgen  # noqa: E402
import paper_2103_14978_b200 as gk  # noqa: E402


def timed(fn, reps=7, warm=2):
    for _ in range(warm):
        fn()
    out = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, nargs="+", default=[100, 150, 250])
    ap.add_argument("--n", type=int, default=30_000_000)
    ap.add_argument("--tag", default=os.environ.get("GK_LIB", "default"))
    a = ap.parse_args()
    gk.load_library()
    res = {"lib": a.tag}
    for L in a.L:
        r, f = pairgen.gen_pairs_cuda(a.n, L)
        e5 = L // 20
        emax = (L + 9) // 10
        q, uq = gk.encode(r, L)
        s, us = gk.encode(f, L)
        res[f"{L}bp_encode_x2_ms"] = round(timed(lambda: (gk.encode(r, L, out=(q, uq)),
                                                          gk.encode(f, L, out=(s, us)))), 4)
        accf, errf = gk.filter_ascii(r, f, e5)
        res[f"{L}bp_fused_e{e5}_ms"] = round(timed(lambda: gk.filter_ascii(
            r, f, e5, accept=accf, errcount=errf)), 4)
        try:
            accs, errs = gk.filter_ascii_sweep(r, f, emax)
            res[f"{L}bp_fused_sweep_e0-{emax}_ms"] = round(timed(lambda: gk.filter_ascii_sweep(
                r, f, emax, accept=accs, errcount=errs)), 4)
            del accs, errs
        except gk.GateKeeperError as ex:
            res[f"{L}bp_fused_sweep_e0-{emax}_ms"] = str(ex)
        del r, f, accf, errf
        acc, err = gk.filter(q, s, uq, us, a.n, L, e5)
        res[f"{L}bp_filter_e{e5}_ms"] = round(timed(lambda: gk.filter(q, s, uq, us, a.n, L, e5,
                                                                       accept=acc, errcount=err)), 4)
        acc2, err2 = gk.filter_sweep(q, s, uq, us, a.n, L, emax)
        res[f"{L}bp_sweep_e0-{emax}_ms"] = round(timed(lambda: gk.filter_sweep(
            q, s, uq, us, a.n, L, emax, accept=acc2, errcount=err2)), 4)
        del q, s, uq, us, acc, err, acc2, err2
        torch.cuda.empty_cache()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
