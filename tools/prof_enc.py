"""Encode one synthetic batch twice (for ncu).  usage: python tools/prof_enc.py --n 4000000 --L 100"""
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
a = p.parse_args()
r, f = pairgen.gen_pairs_cuda(a.n, a.L)
for _ in range(2):
    gk.encode(r, a.L)
    gk.encode(f, a.L)
torch.cuda.synchronize()
print("done")
