"""Small invocation of every kernel of libgk.so, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck): TMA encoder + tail paths, the
register filter, the block-transposed filter and its e sweep, the mask-major fallback, the fused
ASCII filter, compaction (single and batched), the reference-index packing / gathering, the accuracy harness and the host
pipelines."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import pairgen  # noqa: E402
import paper_2103_14978_b200 as gk  # noqa: E402

for L, n in [(100, 3000), (150, 2200), (37, 1500)]:
    hr, hf = pairgen.gen_pairs(n, L, profile=pairgen.PROFILE_BALANCED, emax=5)
    r = torch.from_numpy(hr).cuda()
    f = torch.from_numpy(hf).cuda()
    q, uq = gk.encode(r, L)
    s, us = gk.encode(f, L)
    for e in (0, 3, 13, L - 1 if L < 40 else 30):
        acc, err = gk.filter(q, s, uq, us, n, L, e)
        gk.filter(q, s, uq, us, n, L, e, flags=gk.GK_FLAG_NO_EDGE_FIX)
        gk.filter(q, s, uq, us, n, L, e, flags=gk.GK_FLAG_GENERIC)
        gk.filter_sweep(q, s, uq, us, n, L, e)
        gk.filter_ascii(r, f, e, L)
        gk.compact(acc, n)
    gp = gk.pack_planes(f)
    offs = torch.arange(n, device="cuda", dtype=torch.int64) * L
    gk.gather_windows(gp, n * L, offs, L)
    d = gk.edit_distance(r, f, L)
    a2, e2 = gk.filter_sweep(q, s, uq, us, n, L, 4)
    gk.accuracy(a2, e2, d, n, range(5))
    gk.compact_rows(a2, n)
    torch.cuda.synchronize()
    acc, _, _ = gk.filter_host(torch.from_numpy(hr).pin_memory(),
                               torch.from_numpy(hf).pin_memory(), 4, indices=True,
                               chunk_pairs=1024)
    gk.filter_host_sweep(torch.from_numpy(hr), torch.from_numpy(hf), [0, 5], chunk_pairs=1024)
torch.cuda.synchronize()
print("sanitize_run ok")
