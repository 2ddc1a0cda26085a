"""Run each kernel of the hot path a few times on one synthetic batch (for ncu).

usage: python tools/prof_run.py --n 4000000 --L 100 --e 5 [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import pairgen  # noqa: E402
import paper_2103_14978_b200 as gk  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=4_000_000)
p.add_argument("--L", type=int, default=100)
p.add_argument("--e", type=int, nargs="+", default=[5])
p.add_argument("--reps", type=int, default=2)
a = p.parse_args()
r, f = pairgen.gen_pairs_cuda(a.n, a.L)
torch.cuda.synchronize()
for _ in range(a.reps):
    q, uq = gk.encode(r, a.L)
    s, us = gk.encode(f, a.L)
    for e in a.e:
        acc, err = gk.filter(q, s, uq, us, a.n, a.L, e)
        acc2, err2 = gk.filter_ascii(r, f, e, a.L)
        idx, n_acc = gk.compact(acc, a.n)
torch.cuda.synchronize()
print("done")
