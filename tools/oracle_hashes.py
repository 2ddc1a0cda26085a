#!/usr/bin/env python
"""Write tests/golden/full_parity.json: per-chunk hashes of the ORACLE's
(accept, errcount) for every pair of BASELINE configs[1..4] (C2-C5).

Calls only pairgen (host generator) and oracle/ (oracle.sweep_prefix, pinned
row for row against independent filtrations in tests/test_oracle_sweep.py);
no value comes from the CUDA path.  The GPU side
(tests/test_full_parity_gpu.py, tools/full_parity.py) hashes the bench path's
outputs for the same pairs and compares chunk by chunk.

Long-running (about an hour of CPU for C5 on 8 cores); resumable: finished
chunks are kept in tests/golden/full_parity.partial.json.

    python tools/oracle_hashes.py [--only c2,c3] [--threads N]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import pairgen  # noqa: E402
import parity_hash  # noqa: E402
from pairgen.workloads import HASH_CHUNK, SEED, WORKLOADS, chunks  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden", "full_parity.json")
PARTIAL = os.path.join(ROOT, "tests", "golden", "full_parity.partial.json")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c2,c3,c4,c5")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    state = {}
    if os.path.exists(PARTIAL):
        with open(PARTIAL) as f:
            state = json.load(f)
    state.setdefault("meta", {
        "hash": "sum of splitmix64_finalize((p<<16 | e<<9 | errcount<<1 | accept) + 0x9E3779B97F4A7C15) "
                "mod 2^64 over each chunk (tests/parity_hash.py)",
        "chunk": HASH_CHUNK, "seed": SEED, "profile": "paper",
        "writer": "tools/oracle_hashes.py (pairgen host generator + oracle.sweep_prefix)"})
    state.setdefault("workloads", {})
    for name in args.only.split(","):
        wl = WORKLOADS[name]
        wst = state["workloads"].setdefault(name, {"buckets": []})
        while len(wst["buckets"]) < len(wl.buckets):
            wst["buckets"].append(None)
        for bi, b in enumerate(wl.buckets):
            ch = chunks(b)
            bst = wst["buckets"][bi]
            if bst is None or bst.get("L") != b.L:
                bst = {"L": b.L, "es": list(b.es), "idx0": b.idx0, "n": b.n,
                       "hashes": {str(e): [] for e in b.es}}
                wst["buckets"][bi] = bst
            done = len(bst["hashes"][str(b.es[0])])
            t0 = time.time()
            for ci in range(done, len(ch)):
                p0, m = ch[ci]
                reads, refs = pairgen.gen_pairs(m, b.L, idx0=p0, nthreads=args.threads)
                acc, err = oracle.sweep_prefix(reads, refs, b.emax, nthreads=args.threads)
                hs = parity_hash.hash_rows_np(p0, acc[list(b.es)], err[list(b.es)], b.es)
                for e, h in zip(b.es, hs):
                    bst["hashes"][str(e)].append(f"{h:016x}")
                if ci % 4 == 3 or ci == len(ch) - 1:
                    with open(PARTIAL + ".tmp", "w") as f:
                        json.dump(state, f)
                    os.replace(PARTIAL + ".tmp", PARTIAL)
                el = time.time() - t0
                rate = (ci - done + 1) / el
                print(f"{name} bucket {bi} ({b.L} bp) chunk {ci + 1}/{len(ch)} "
                      f"{el:.0f}s eta {(len(ch) - ci - 1) / rate:.0f}s", flush=True)
        write_golden(state)
    write_golden(state)


def write_golden(state):
    complete = all(
        name in state["workloads"] and all(
            bst is not None and len(bst["hashes"][str(bst["es"][0])]) == len(chunks(b))
            for bst, b in zip(state["workloads"][name]["buckets"], WORKLOADS[name].buckets))
        for name in WORKLOADS)
    out = dict(state)
    out["complete"] = complete
    # only fully hashed workloads go into the golden file
    out["workloads"] = {
        name: w for name, w in state["workloads"].items()
        if all(bst is not None and len(bst["hashes"][str(bst["es"][0])]) == len(chunks(b))
               for bst, b in zip(w["buckets"], WORKLOADS[name].buckets))}
    with open(GOLDEN + ".tmp", "w") as f:
        json.dump(out, f, indent=0)
    os.replace(GOLDEN + ".tmp", GOLDEN)
    print("wrote", GOLDEN, "complete" if complete else "partial", flush=True)


if __name__ == "__main__":
    main()
