"""A/B: the L2-staged fused kernel (gk_filter_ascii_ws) vs the packed path (gk_encode x2 +
gk_filter) on the C5 buckets' pairs; results must be identical.
usage: python tools/time_l2.py [--n 30000000] [--reps 5]   (one JSON line per bucket)"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import pairgen  # noqa: E402
import paper_2103_14978_b200 as gk  # noqa: E402
from pairgen.workloads import WORKLOADS  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=30_000_000)
p.add_argument("--reps", type=int, default=5)
p.add_argument("--tag", default="")
p.add_argument("--buckets", default="0,1,2")
a = p.parse_args()
s = torch.cuda.current_stream()


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps


for bi in [int(x) for x in a.buckets.split(",")]:
    bk = WORKLOADS["c5"].buckets[bi]
    L, e, idx0 = bk.L, bk.es[0], bk.idx0
    n = a.n
    reads, refs = pairgen.gen_pairs_cuda(n, L, idx0=idx0)
    pq = torch.empty(gk.packed_words(n, L), dtype=torch.int32, device="cuda")
    pr = torch.empty_like(pq)
    uq = torch.empty(gk.undef_words(n), dtype=torch.int32, device="cuda")
    ur = torch.empty_like(uq)
    acc0 = torch.empty(gk.result_words(n), dtype=torch.int32, device="cuda")
    err0 = torch.empty(n, dtype=torch.uint8, device="cuda")
    acc1 = torch.empty_like(acc0)
    err1 = torch.empty_like(err0)
    ws = torch.empty(gk.filter_ascii_workspace_bytes(L), dtype=torch.uint8, device="cuda")

    def packed():
        gk.encode(reads, L, out=(pq, uq), stream=s)
        gk.encode(refs, L, out=(pr, ur), stream=s)
        gk.filter(pq, pr, uq, ur, n, L, e, accept=acc0, errcount=err0, stream=s)

    def l2():
        gk.filter_ascii_ws(reads, refs, e, L, accept=acc1, errcount=err1, workspace=ws, stream=s)

    t_p = timed(packed)
    t_l = timed(l2)
    same = bool(torch.equal(acc0, acc1) and torch.equal(err0, err1))
    print(json.dumps({"tag": a.tag, "L": L, "e": e, "n": n, "packed_ms": round(t_p, 4),
                      "l2_ms": round(t_l, 4), "speedup": round(t_p / t_l, 3), "identical": same,
                      "ws_MB": round(ws.numel() / 1e6, 1),
                      "l2_hbm_frac_ascii": round(2 * L * n / (t_l / 1e3) / 6465.8e9, 3)}),
          flush=True)
    del reads, refs, pq, pr, uq, ur, acc0, acc1, err0, err1, ws
    torch.cuda.empty_cache()
