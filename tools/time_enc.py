"""CUDA-event time of gk_encode on device-generated ASCII (median of reps).
usage: python tools/time_enc.py --n 30000000 --L 100 150 250"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import pairgen  # noqa: E402
import paper_2103_14978_b200 as gk  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=30_000_000)
p.add_argument("--L", type=int, nargs="+", default=[100])
p.add_argument("--reps", type=int, default=7)
a = p.parse_args()
for L in a.L:
    r, _ = pairgen.gen_pairs_cuda(a.n, L)
    out = gk.encode(r, L)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        gk.encode(r, L, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    byts = a.n * L + a.n * L / 4 + a.n / 8
    print(json.dumps({"L": L, "n": a.n, "ms": round(ms, 4), "GB_s": round(byts / ms / 1e6, 1),
                      "hbm_frac": round(byts / ms / 1e6 / 6544, 4)}), flush=True)
    del r, out
    torch.cuda.empty_cache()
