#!/usr/bin/env python
"""A/B timing of the packed filter kernels (gk_filter at one e, gk_filter_sweep) on
resident pairs, with a checksum of the outputs so that variant libraries (tools/ab_build.py,
GK_LIB=...) can be checked for identical results across processes.

    GK_LIB=... python tools/time_filters2.py --per-e 250:12 150:7 --sweep 100:10
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


def checksum(*ts):
    h = 0
    for t in ts:
        v = t.contiguous().reshape(-1).view(torch.uint8).to(torch.int64)
        w = torch.arange(v.numel(), device=v.device, dtype=torch.int64) % 1000003 + 1
        h = (h * 1000033 + int((v * w).sum().item())) % (1 << 61)
    return h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--per-e", nargs="*", default=["250:12"])
    ap.add_argument("--sweep", nargs="*", default=[])
    ap.add_argument("--encode", nargs="*", type=int, default=[], help="read lengths: time gk_encode x2")
    ap.add_argument("--n", type=int, default=30_000_000)
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("GK_LIB", "default")))
    a = ap.parse_args()
    gk.load_library()
    res = {"lib": a.tag, "n": a.n}
    cache = {}

    def packed(L):
        if L not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            r, f = pairgen.gen_pairs_cuda(a.n, L)
            q, uq = gk.encode(r, L)
            s, us = gk.encode(f, L)
            del r, f
            cache[L] = (q, s, uq, us)
        return cache[L]

    for L in a.encode:
        cache.clear()
        torch.cuda.empty_cache()
        r, f = pairgen.gen_pairs_cuda(a.n, L)
        q, uq = gk.encode(r, L)
        s, us = gk.encode(f, L)
        res[f"{L}bp_encode_x2_ms"] = round(timed(lambda: (gk.encode(r, L, out=(q, uq)),
                                                          gk.encode(f, L, out=(s, us)))), 4)
        res[f"{L}bp_encode_GB_s"] = round(a.n * 2 * (L + L / 4) / (res[f"{L}bp_encode_x2_ms"] / 1e3) / 1e9, 1)
        res[f"{L}bp_encode_sum"] = checksum(q, s, uq, us)
        del r, f, q, s, uq, us
    for spec in a.per_e:
        L, e = map(int, spec.split(":"))
        q, s, uq, us = packed(L)
        acc, err = gk.filter(q, s, uq, us, a.n, L, e)
        res[f"{L}bp_e{e}_ms"] = round(timed(lambda: gk.filter(q, s, uq, us, a.n, L, e,
                                                               accept=acc, errcount=err)), 4)
        res[f"{L}bp_e{e}_sum"] = checksum(acc, err)
        del acc, err
    for spec in a.sweep:
        L, emax = map(int, spec.split(":"))
        q, s, uq, us = packed(L)
        acc, err = gk.filter_sweep(q, s, uq, us, a.n, L, emax)
        res[f"{L}bp_sweep{emax}_ms"] = round(timed(lambda: gk.filter_sweep(
            q, s, uq, us, a.n, L, emax, accept=acc, errcount=err)), 4)
        res[f"{L}bp_sweep{emax}_sum"] = checksum(acc, err)
        del acc, err
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
