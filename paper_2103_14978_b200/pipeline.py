"""pipeline -- one step of the hot path over a resident batch, as the bench times it.

A *step* is one pass of every SURVEY.md 8(a) row over one batch of pairs that
already sits in HBM: a1 encode, a2-a6 filtration (for every threshold of the
workload), a7 compaction.  The classes below own the device buffers of a step
and launch it on a stream through the C ABI (via the ctypes binding), so that
bench.py, the full-size parity tools and the tests run exactly the same
launches.  Every launch is a libgk.so kernel; nothing here computes.

* :class:`SweepStep`   -- one batch, thresholds e = 0..e_max (C2-C4):
  path "packed": gk_encode x2, gk_filter_sweep (all e in one pass), gk_compact_rows;
  path "fused": gk_filter_ascii_sweep (encode + sweep in one kernel), gk_compact_rows.
* :class:`BucketStep`  -- one batch, one threshold e (a C5 length bucket):
  path "fused": gk_filter_ascii (a1-a6 in one kernel) + gk_compact;
  path "packed": gk_encode x2 + gk_filter + gk_compact.
"""
from __future__ import annotations

from . import (compact, compact_rows, compact_rows_workspace_bytes, compact_workspace_bytes,
               encode, filter, filter_ascii, filter_ascii_sweep, filter_sweep, packed_words,
               result_words, undef_words)

# Reads up to this length take the fused kernels in "auto" mode.  Measured
# (profiles/r02_ab_fused.jsonl): the tile-per-CTA fused kernels are still slower than
# encode + filter at every length (100 bp e=5: 2.40 vs 1.94 ms per 30M pairs; they
# are latency-bound on their span loads), so auto = the packed path for now.
FUSED_MAX_LEN = 0


class _Timer:
    """Optional CUDA events around each launch group (the last step's per-kernel times)."""

    def __init__(self, torch, names):
        self.names = list(names)
        self.ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for k in self.names}

    def start(self, k, stream):
        self.ev[k][0].record(stream)

    def stop(self, k, stream):
        self.ev[k][1].record(stream)

    def ms(self):
        return {k: a.elapsed_time(b) for k, (a, b) in self.ev.items()}


class SweepStep:
    """a1 once, a2-a6 for every e <= e_max in one pass, a7 for every e.
    path "packed": gk_encode x2 + gk_filter_sweep; "fused": gk_filter_ascii_sweep."""

    def __init__(self, torch, n: int, L: int, e_max: int, device, compact_indices: bool = True,
                 path: str = "packed"):
        if path not in ("fused", "packed"):
            raise ValueError(path)
        self.n, self.L, self.e_max, self.path = n, L, e_max, path
        self.kernels = (("filter_ascii_sweep", "compact_rows") if path == "fused"
                        else ("encode", "filter_sweep", "compact_rows"))
        rows = e_max + 1
        if path == "packed":
            self.pq = torch.empty(packed_words(n, L), dtype=torch.int32, device=device)
            self.pr = torch.empty_like(self.pq)
            self.uq = torch.empty(undef_words(n), dtype=torch.int32, device=device)
            self.ur = torch.empty_like(self.uq)
        self.accept = torch.empty((rows, result_words(n)), dtype=torch.int32, device=device)
        self.errc = torch.empty((rows, n), dtype=torch.uint8, device=device)
        self.idx = (torch.empty((rows, n), dtype=torch.int32, device=device)
                    if compact_indices else None)
        self.n_acc = torch.zeros(rows, dtype=torch.int64, device=device)
        self.ws = torch.empty(compact_rows_workspace_bytes(n, rows), dtype=torch.uint8,
                              device=device)
        self.timer = _Timer(torch, self.kernels)

    def run(self, reads, refs, stream, record: bool = False):
        t = self.timer if record else None
        if self.path == "fused":
            if t:
                t.start("filter_ascii_sweep", stream)
            filter_ascii_sweep(reads, refs, self.e_max, self.L, accept=self.accept,
                               errcount=self.errc, stream=stream)
            if t:
                t.stop("filter_ascii_sweep", stream)
                t.start("compact_rows", stream)
        else:
            if t:
                t.start("encode", stream)
            encode(reads, self.L, out=(self.pq, self.uq), stream=stream)
            encode(refs, self.L, out=(self.pr, self.ur), stream=stream)
            if t:
                t.stop("encode", stream)
                t.start("filter_sweep", stream)
            filter_sweep(self.pq, self.pr, self.uq, self.ur, self.n, self.L, self.e_max,
                         accept=self.accept, errcount=self.errc, stream=stream)
            if t:
                t.stop("filter_sweep", stream)
                t.start("compact_rows", stream)
        compact_rows(self.accept, self.n, idx=self.idx, n_acc=self.n_acc, workspace=self.ws,
                     want_indices=self.idx is not None, stream=stream)
        if t:
            t.stop("compact_rows", stream)


class BucketStep:
    """a1-a7 for one threshold e over one batch (a C5 length bucket)."""

    def __init__(self, torch, n: int, L: int, e: int, device, path: str = "fused",
                 compact_indices: bool = True):
        if path not in ("fused", "packed"):
            raise ValueError(path)
        self.n, self.L, self.e, self.path = n, L, e, path
        self.kernels = (("filter_ascii", "compact") if path == "fused"
                        else ("encode", "filter", "compact"))
        if path == "packed":
            self.pq = torch.empty(packed_words(n, L), dtype=torch.int32, device=device)
            self.pr = torch.empty_like(self.pq)
            self.uq = torch.empty(undef_words(n), dtype=torch.int32, device=device)
            self.ur = torch.empty_like(self.uq)
        self.accept = torch.empty((1, result_words(n)), dtype=torch.int32, device=device)
        self.errc = torch.empty((1, n), dtype=torch.uint8, device=device)
        self.idx = torch.empty(n, dtype=torch.int32, device=device) if compact_indices else None
        self.n_acc = torch.zeros(1, dtype=torch.int64, device=device)
        self.ws = torch.empty(compact_workspace_bytes(n), dtype=torch.uint8, device=device)
        self.timer = _Timer(torch, self.kernels)

    def run(self, reads, refs, stream, record: bool = False):
        t = self.timer if record else None
        if self.path == "fused":
            if t:
                t.start("filter_ascii", stream)
            filter_ascii(reads, refs, self.e, self.L, accept=self.accept[0], errcount=self.errc[0],
                         stream=stream)
            if t:
                t.stop("filter_ascii", stream)
        else:
            if t:
                t.start("encode", stream)
            encode(reads, self.L, out=(self.pq, self.uq), stream=stream)
            encode(refs, self.L, out=(self.pr, self.ur), stream=stream)
            if t:
                t.stop("encode", stream)
                t.start("filter", stream)
            filter(self.pq, self.pr, self.uq, self.ur, self.n, self.L, self.e,
                   accept=self.accept[0], errcount=self.errc[0], stream=stream)
            if t:
                t.stop("filter", stream)
        if t:
            t.start("compact", stream)
        compact(self.accept[0], self.n, idx=self.idx, n_acc=self.n_acc,
                workspace=self.ws, want_indices=self.idx is not None, stream=stream)
        if t:
            t.stop("compact", stream)

    @property
    def es(self):
        return (self.e,)


def auto_path(L: int) -> str:
    """The path the bench uses for read length L: fused below FUSED_MAX_LEN."""
    return "fused" if L <= FUSED_MAX_LEN else "packed"
