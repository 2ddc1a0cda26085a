"""Reference-index mode timing: a synthetic genome packed
once, reads packed once, n candidate (read, position) pairs gathered into the packed
layout and filtered for every e <= e_max in one sweep pass.  CUDA-event times,
median of reps; compare with the ASCII path (gk_encode of both sides per pair).

usage: python tools/time_index.py --G 250000000 --reads 3000000 --cands 30000000 --L 100 --emax 10
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2103_14978_b200 as gk  # noqa: E402


def timed(fn, reps=5):
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
p.add_argument("--G", type=int, default=250_000_000)
p.add_argument("--reads", type=int, default=3_000_000)
p.add_argument("--cands", type=int, default=30_000_000)
p.add_argument("--L", type=int, default=100)
p.add_argument("--emax", type=int, default=10)
a = p.parse_args()
g = torch.Generator(device="cuda").manual_seed(2103149780)
lut = torch.tensor(list(b"ACGT"), dtype=torch.uint8, device="cuda")
genome = lut[torch.randint(0, 4, (1, a.G), device="cuda", generator=g)]
true_pos = torch.randint(0, a.G - a.L, (a.reads,), device="cuda", generator=g)
idx = true_pos[:, None] + torch.arange(a.L, device="cuda")[None, :]
reads = genome[0][idx].contiguous()
sub = torch.rand(reads.shape, device="cuda", generator=g) < 0.03
reads = torch.where(sub, lut[torch.randint(0, 4, reads.shape, device="cuda", generator=g)], reads)
# a mapper lists the candidates of a read together: read_id = candidate // (cands / reads)
read_id = torch.arange(a.cands, device="cuda") * a.reads // a.cands
near = torch.rand(a.cands, device="cuda", generator=g) < 0.5
pos = torch.where(near, true_pos[read_id], torch.randint(0, a.G - a.L, (a.cands,), device="cuda",
                                                          generator=g)).to(torch.int64)
roff = (read_id * a.L).to(torch.int64)
del idx, sub, true_pos
torch.cuda.synchronize()

ms_pack_genome = timed(lambda: gk.pack_planes(genome), 3)
gp = gk.pack_planes(genome)
rp = gk.pack_planes(reads)
ms_pack_reads = timed(lambda: gk.pack_planes(reads), 3)
q, uq = gk.gather_windows(rp, a.reads * a.L, roff, a.L)
r, ur = gk.gather_windows(gp, a.G, pos, a.L)
ms_gather_q = timed(lambda: gk.gather_windows(rp, a.reads * a.L, roff, a.L, out=(q, uq)))
ms_gather_r = timed(lambda: gk.gather_windows(gp, a.G, pos, a.L, out=(r, ur)))
acc, err = gk.filter_sweep(q, r, uq, ur, a.cands, a.L, a.emax)
ms_sweep = timed(lambda: gk.filter_sweep(q, r, uq, ur, a.cands, a.L, a.emax, accept=acc, errcount=err))
# the ASCII path for the same candidates: materialised windows, encoded per pair
ref_rows = genome[0][pos[:, None] + torch.arange(a.L, device="cuda")[None, :]]
read_rows = reads[read_id]
q2, uq2 = gk.encode(read_rows, a.L)
r2, ur2 = gk.encode(ref_rows, a.L)
ms_encode = timed(lambda: (gk.encode(read_rows, a.L, out=(q2, uq2)), gk.encode(ref_rows, a.L, out=(r2, ur2))))
torch.cuda.synchronize()
same = torch.equal(uq, uq2) and torch.equal(ur, ur2)
acc2, err2 = gk.filter_sweep(q2, r2, uq2, ur2, a.cands, a.L, a.emax)
torch.cuda.synchronize()
same = same and torch.equal(acc, acc2) and torch.equal(err, err2)
# end to end from host candidate lists (offsets in pinned host memory, results back to host)
import time  # noqa: E402
ro_h = roff.cpu().pin_memory()
fo_h = pos.cpu().pin_memory()
acc_h = torch.empty((a.emax + 1, gk.result_words(a.cands)), dtype=torch.int32, pin_memory=True)
err_h = torch.empty((a.emax + 1, a.cands), dtype=torch.uint8, pin_memory=True)
chunk = 1 << 21
ws = torch.empty(gk.load_library().gk_host_index_workspace_bytes(chunk, a.L, a.emax),
                 dtype=torch.uint8, device="cuda")
gk.filter_host_index(rp, a.reads * a.L, gp, a.G, ro_h, fo_h, a.L, a.emax, accept=acc_h,
                     errcount=err_h, workspace=ws, chunk_pairs=chunk)
t0 = time.perf_counter()
for _ in range(3):
    gk.filter_host_index(rp, a.reads * a.L, gp, a.G, ro_h, fo_h, a.L, a.emax, accept=acc_h,
                         errcount=err_h, workspace=ws, chunk_pairs=chunk)
dt_e2e = (time.perf_counter() - t0) / 3
same = same and torch.equal(acc_h.cuda(), acc) and torch.equal(err_h.cuda(), err)
gbytes = a.cands * (3 * a.L / 8 + a.L / 4 + 1 / 8)  # planes of the window + packed words out
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
except OSError:
    peak = 6650.0
print(json.dumps({
    "G": a.G, "reads": a.reads, "cands": a.cands, "L": a.L, "emax": a.emax,
    "ms_pack_genome_once": round(ms_pack_genome, 3), "ms_pack_reads_once": round(ms_pack_reads, 3),
    "ms_gather_reads": round(ms_gather_q, 4), "ms_gather_refs": round(ms_gather_r, 4),
    "gather_GB_s": round(gbytes / (ms_gather_r / 1e3) / 1e9, 1),
    "gather_hbm_frac": round(gbytes / (ms_gather_r / 1e3) / 1e9 / peak, 4),
    "gather_reads_GB_s": round(gbytes / (ms_gather_q / 1e3) / 1e9, 1),
    "ms_sweep": round(ms_sweep, 4),
    "index_path_Gfiltrations_s": round(a.cands * (a.emax + 1) / (ms_gather_q + ms_gather_r + ms_sweep) / 1e6, 2),
    "ms_encode_ascii_path": round(ms_encode, 4),
    "ascii_path_Gfiltrations_s": round(a.cands * (a.emax + 1) / (ms_encode + ms_sweep) / 1e6, 2),
    "ascii_input_bytes_per_pair": 2 * a.L, "index_input_bytes_per_pair": 16,
    "e2e_host_index_s": round(dt_e2e, 4),
    "e2e_host_index_Gfiltrations_s": round(a.cands * (a.emax + 1) / dt_e2e / 1e9, 2),
    "e2e_h2d_bytes": a.cands * 16, "e2e_d2h_bytes": (a.emax + 1) * (a.cands // 8 + a.cands),
    "results_identical_to_ascii_path": bool(same)}), flush=True)
