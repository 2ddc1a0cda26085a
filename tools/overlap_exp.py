"""Experiment: does encoding chunk c+1 (stream B) overlap with the sweep of chunk c
(stream A)?  Times the C2 step (encode x2 + sweep, no compaction) serial vs chunked.
usage: GK_ENC_PER_SM=k python tools/overlap_exp.py --chunks 4"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import pairgen  # noqa: E402
import paper_2103_14978_b200 as gk  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=30_000_000)
p.add_argument("--L", type=int, default=100)
p.add_argument("--emax", type=int, default=10)
p.add_argument("--chunks", type=int, nargs="+", default=[1, 2, 4, 8])
a = p.parse_args()
n, L, E = a.n, a.L, a.emax
r, f = pairgen.gen_pairs_cuda(n, L)
sA = torch.cuda.current_stream()
sB = torch.cuda.Stream()
for K in a.chunks:
    m = (n // K) // 1024 * 1024
    bufs = []
    for j in range(2):
        q = torch.empty(gk.packed_words(m, L), dtype=torch.int32, device="cuda")
        s = torch.empty_like(q)
        uq = torch.empty(gk.undef_words(m), dtype=torch.int32, device="cuda")
        us = torch.empty_like(uq)
        acc = torch.empty((E + 1, gk.result_words(m)), dtype=torch.int32, device="cuda")
        err = torch.empty((E + 1, m), dtype=torch.uint8, device="cuda")
        bufs.append((q, s, uq, us, acc, err))
    enc_done = [torch.cuda.Event() for _ in range(2)]
    sw_done = [torch.cuda.Event() for _ in range(2)]

    def step():
        for c in range(K):
            j = c % 2
            q, s, uq, us, acc, err = bufs[j]
            rr, ff = r[c * m:(c + 1) * m], f[c * m:(c + 1) * m]
            es = sB if K > 1 else sA
            if c >= 2:
                es.wait_event(sw_done[j])
            gk.encode(rr, L, out=(q, uq), stream=es)
            gk.encode(ff, L, out=(s, us), stream=es)
            enc_done[j].record(es)
            sA.wait_event(enc_done[j])
            gk.filter_sweep(q, s, uq, us, m, L, E, accept=acc, errcount=err, stream=sA)
            sw_done[j].record(sA)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sA)
    for _ in range(5):
        step()
    e1.record(sA)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5 * n / (m * K)
    print(f"chunks={K} per_sm={os.environ.get('GK_ENC_PER_SM', 'max')} ms/step(30M-equiv)={ms:.3f}", flush=True)
