"""Run the sweep kernel and the block-transposed / register filters once each on
one synthetic batch (for ncu).  usage: python tools/prof_sweep.py --n 4000000 --L 100 --emax 10"""
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
p.add_argument("--emax", type=int, default=10)
a = p.parse_args()
r, f = pairgen.gen_pairs_cuda(a.n, a.L)
q, uq = gk.encode(r, a.L)
s, us = gk.encode(f, a.L)
gk.filter_sweep(q, s, uq, us, a.n, a.L, a.emax)
gk.filter(q, s, uq, us, a.n, a.L, a.emax, flags=gk.GK_FLAG_BLOCKED)
gk.filter(q, s, uq, us, a.n, a.L, a.emax)
torch.cuda.synchronize()
print("done")
