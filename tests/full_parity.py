"""Full-size parity of the bench path against the oracle's golden chunk hashes.

TEST INFRASTRUCTURE.  For every pair of a workload (BASELINE configs[1..4] =
C2-C5; pairgen.workloads) the CUDA path -- the same step bench.py times
(paper_2103_14978_b200.pipeline) -- computes (accept, errcount) for every
threshold of the workload; tests/native/parity_hash.cu hashes them per chunk
of 2^20 pairs; the hashes are compared with tests/golden/full_parity.json,
written by tools/oracle_hashes.py from the CPU oracle alone.  A chunk whose
hash differs is recomputed by the oracle on the host and diffed pair by pair.
"""
from __future__ import annotations

import json
import os
import time

import numpy as np

import parity_hash

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "full_parity.json")


def load_golden():
    if not os.path.exists(GOLDEN):
        return None
    with open(GOLDEN) as f:
        return json.load(f)


def _bits_to_u8(words: np.ndarray, n: int) -> np.ndarray:
    return np.unpackbits(words.view(np.uint8), bitorder="little")[:n]


def diff_chunk(L, es, p0, m, acc_dev, err_dev, limit=5):
    """Oracle on the host for pairs [p0, p0+m) vs the device rows -> list of mismatches."""
    import oracle
    import pairgen
    reads, refs = pairgen.gen_pairs(m, L, idx0=p0)
    oa, oc = oracle.sweep_prefix(reads, refs, max(es))
    out = []
    for j, e in enumerate(es):
        da = _bits_to_u8(acc_dev[j], m)
        dc = err_dev[j][:m]
        bad = np.nonzero((da != oa[e]) | (dc != oc[e]))[0]
        for i in bad[:limit]:
            out.append({"pair": int(p0 + i), "e": int(e), "oracle": [int(oa[e][i]), int(oc[e][i])],
                        "cuda": [int(da[i]), int(dc[i])],
                        "read": bytes(reads[i]).decode(errors="replace"),
                        "ref": bytes(refs[i]).decode(errors="replace")})
        if bad.size:
            out.append({"e": int(e), "mismatching_pairs": int(bad.size)})
    return out


def run_workload(name: str, path: str | None = None, mem_gb: float = 60.0, max_pairs=None,
                 device=None, log=print):
    """Hash the CUDA path's outputs for every pair of `name` and compare with the golden.
    Returns a record dict (chunks compared / mismatching, details of any mismatch)."""
    import torch

    import pairgen
    from pairgen.workloads import HASH_CHUNK, WORKLOADS
    from paper_2103_14978_b200.pipeline import BucketStep, SweepStep

    golden = load_golden()
    if golden is None or name not in golden.get("workloads", {}):
        raise FileNotFoundError(f"no golden hashes for {name} in {GOLDEN}")
    gw = golden["workloads"][name]
    wl = WORKLOADS[name]
    dev = torch.device("cuda", 0) if device is None else torch.device(device)
    stream = torch.cuda.current_stream(dev)
    rec = {"workload": name, "buckets": [], "chunks_compared": 0, "chunks_mismatching": 0,
           "pairs_compared": 0}
    t0 = time.time()
    for bi, b in enumerate(wl.buckets):
        gb = gw["buckets"][bi]
        nch_golden = len(gb["hashes"][str(b.es[0])])
        n = b.n if max_pairs is None else min(
            b.n, max(HASH_CHUNK, max_pairs // HASH_CHUNK * HASH_CHUNK))
        nch = (n + HASH_CHUNK - 1) // HASH_CHUNK
        if nch > nch_golden:
            raise FileNotFoundError(f"golden for {name} bucket {bi} has {nch_golden} of {nch} chunks")
        rows = len(b.es)
        out = torch.zeros((rows, nch), dtype=torch.int64, device=dev)
        per_pair = 2 * b.L + b.L // 2 + 16 + rows * 2
        batch = max(HASH_CHUNK, int(mem_gb * 1e9 / per_pair) // HASH_CHUNK * HASH_CHUNK)
        from paper_2103_14978_b200.pipeline import auto_path
        bpath = path or auto_path(b.L)
        sweep = name != "c5"
        for s0 in range(0, n, batch):
            m = min(batch, n - s0)
            p_first = b.idx0 + s0
            reads, refs = pairgen.gen_pairs_cuda(m, b.L, idx0=p_first, device=dev)
            if sweep:
                st = SweepStep(torch, m, b.L, b.emax, dev, compact_indices=False, path=bpath)
                st.run(reads, refs, stream)
                acc, err = st.accept[list(b.es)], st.errc[list(b.es)]
            else:
                st = BucketStep(torch, m, b.L, b.es[0], dev, path=bpath, compact_indices=False)
                st.run(reads, refs, stream)
                acc, err = st.accept, st.errc
            parity_hash.hash_rows_cuda(acc, err, m, b.es, p_first, b.idx0, out, HASH_CHUNK)
            del st, reads, refs, acc, err
            torch.cuda.empty_cache()
        got = out.cpu().numpy().astype(np.uint64)
        bad = []
        for j, e in enumerate(b.es):
            ref = [int(h, 16) for h in gb["hashes"][str(e)][:nch]]
            for c in range(nch):
                if int(got[j, c]) != ref[c]:
                    bad.append((c, e))
        bad_chunks = sorted({c for c, _ in bad})
        detail = []
        for c in bad_chunks[:3]:
            p0 = b.idx0 + c * HASH_CHUNK
            m = min(HASH_CHUNK, b.idx0 + n - p0)
            reads, refs = pairgen.gen_pairs_cuda(m, b.L, idx0=p0, device=dev)
            if sweep:
                st = SweepStep(torch, m, b.L, b.emax, dev, compact_indices=False, path=bpath)
                st.run(reads, refs, stream)
                acc, err = st.accept[list(b.es)], st.errc[list(b.es)]
            else:
                st = BucketStep(torch, m, b.L, b.es[0], dev, path=bpath, compact_indices=False)
                st.run(reads, refs, stream)
                acc, err = st.accept, st.errc
            torch.cuda.synchronize(dev)
            detail.append({"chunk": c, "diff": diff_chunk(b.L, b.es, p0, m,
                                                          acc.cpu().numpy(), err.cpu().numpy())})
        rec["buckets"].append({"read_len": b.L, "es": list(b.es), "pairs": n, "chunks": nch,
                               "path": bpath, "mismatching_chunks": bad_chunks,
                               "mismatch_detail": detail})
        rec["chunks_compared"] += nch * rows
        rec["chunks_mismatching"] += len(bad)
        rec["pairs_compared"] += n
        log(f"{name} bucket {bi} ({b.L} bp, e {b.es[0]}..{b.es[-1]}): {n} pairs, {nch} chunks x "
            f"{rows} rows, {len(bad)} mismatching")
    rec["seconds"] = round(time.time() - t0, 1)
    return rec
