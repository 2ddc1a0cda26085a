"""oracle -- plain CPU oracle of GateKeeper-GPU's per-pair filter (arXiv 2103.14978).

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2103_14978_b200``) never imports it and
shares no code with it; see ``gk_oracle.c`` for the step-by-step algorithm
and its PAPER.md citations, and DESIGN.md ("Readings of the paper", "Oracle
pins") for what pins each part.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(HERE, "liboracle.so")
_SRC = os.path.join(HERE, "gk_oracle.c")
_lib = None
MAX_LEN = 508


def build() -> None:
    if not os.path.exists(_SO) or os.path.getmtime(_SRC) > os.path.getmtime(_SO):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", _SO, _SRC])


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P = ctypes.c_void_p
        I, I64 = ctypes.c_int, ctypes.c_int64
        lib.gko_code.argtypes = [ctypes.c_uint8]
        lib.gko_filter_pair.argtypes = [P, P, I, I, I, ctypes.POINTER(I), ctypes.POINTER(I), P]
        lib.gko_filter.argtypes = [P, P, I64, I, I64, I, I, P, P, I]
        lib.gko_sweep.argtypes = [P, P, I64, I, I64, I, I, P, P, I]
        lib.gko_sweep_prefix.argtypes = [P, P, I64, I, I64, I, I, P, P, I]
        lib.gko_levenshtein.argtypes = [P, I, P, I]
        lib.gko_pack.argtypes = [P, I64, I, I64, P, P]
        lib.gko_xor_row.argtypes = [P, P, I, I, P]
        lib.gko_amend.argtypes = [P, I, P]
        lib.gko_amend.restype = None
        lib.gko_count.argtypes = [P, I]
        lib.gko_edit_batch.argtypes = [P, P, I64, I, I64, P, I]
        for f in (lib.gko_code, lib.gko_filter_pair, lib.gko_filter, lib.gko_sweep,
                  lib.gko_sweep_prefix,
                  lib.gko_levenshtein, lib.gko_pack, lib.gko_xor_row, lib.gko_count,
                  lib.gko_edit_batch):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _as_bytes(s) -> np.ndarray:
    if isinstance(s, str):
        s = s.encode()
    if isinstance(s, (bytes, bytearray)):
        return np.frombuffer(bytes(s), dtype=np.uint8).copy()
    return np.ascontiguousarray(s, dtype=np.uint8)


def code(b) -> int:
    return _load().gko_code(ord(b) if isinstance(b, str) else int(b))


def filter_pair(read, ref, e: int, edge_fix: bool = True, masks: bool = False):
    """One filtration.  Returns (accept, err) or (accept, err, masks_dict)."""
    q, r = _as_bytes(read), _as_bytes(ref)
    L = int(q.shape[0])
    if r.shape[0] != L:
        raise ValueError("read and reference segment must have the same length")
    a, c = ctypes.c_int(), ctypes.c_int()
    buf = np.zeros(((4 * e + 3) * L,), dtype=np.uint8) if masks else None
    rc = _load().gko_filter_pair(q.ctypes.data, r.ctypes.data, L, e, int(edge_fix),
                                 ctypes.byref(a), ctypes.byref(c),
                                 buf.ctypes.data if masks else None)
    if rc:
        raise ValueError(f"gko_filter_pair rejected arguments (rc={rc})")
    if not masks:
        return a.value, c.value
    m = buf.reshape(4 * e + 3, L)
    d = {"H0": m[0], "A0": m[1], "F": m[2 + 4 * e]}
    for k in range(1, e + 1):
        b = 2 + 4 * (k - 1)
        d[f"D{k}"], d[f"AD{k}"], d[f"I{k}"], d[f"AI{k}"] = m[b], m[b + 1], m[b + 2], m[b + 3]
    return a.value, c.value, d


def filter(reads: np.ndarray, refs: np.ndarray, e: int, L: int | None = None,
           edge_fix: bool = True, nthreads: int | None = None):
    """Batch filtration.  reads/refs: uint8 (n, stride).  Returns (accept u8[n], err u8[n])."""
    reads = np.ascontiguousarray(reads, dtype=np.uint8)
    refs = np.ascontiguousarray(refs, dtype=np.uint8)
    n, stride = reads.shape
    L = stride if L is None else L
    nthreads = (os.cpu_count() or 1) if nthreads is None else nthreads
    acc = np.empty(n, dtype=np.uint8)
    err = np.empty(n, dtype=np.uint8)
    rc = _load().gko_filter(reads.ctypes.data, refs.ctypes.data, n, L, stride, e,
                            int(edge_fix), acc.ctypes.data, err.ctypes.data, nthreads)
    if rc:
        raise ValueError(f"gko_filter rejected arguments (rc={rc})")
    return acc, err


def sweep(reads: np.ndarray, refs: np.ndarray, emax: int, L: int | None = None,
          edge_fix: bool = True, nthreads: int | None = None):
    """accept/err for every e in 0..emax: arrays of shape (emax+1, n)."""
    reads = np.ascontiguousarray(reads, dtype=np.uint8)
    refs = np.ascontiguousarray(refs, dtype=np.uint8)
    n, stride = reads.shape
    L = stride if L is None else L
    nthreads = (os.cpu_count() or 1) if nthreads is None else nthreads
    acc = np.empty((emax + 1, n), dtype=np.uint8)
    err = np.empty((emax + 1, n), dtype=np.uint8)
    rc = _load().gko_sweep(reads.ctypes.data, refs.ctypes.data, n, L, stride, emax,
                           int(edge_fix), acc.ctypes.data, err.ctypes.data, nthreads)
    if rc:
        raise ValueError(f"gko_sweep rejected arguments (rc={rc})")
    return acc, err


def sweep_prefix(reads: np.ndarray, refs: np.ndarray, emax: int, L: int | None = None,
                 edge_fix: bool = True, nthreads: int | None = None):
    """Same outputs as :func:`sweep` in one pass per pair: F_e = F_{e-1} & A*D_e & A*I_e
    (gko_sweep_pair; pinned row for row against :func:`sweep`)."""
    reads = np.ascontiguousarray(reads, dtype=np.uint8)
    refs = np.ascontiguousarray(refs, dtype=np.uint8)
    n, stride = reads.shape
    L = stride if L is None else L
    nthreads = (os.cpu_count() or 1) if nthreads is None else nthreads
    acc = np.empty((emax + 1, n), dtype=np.uint8)
    err = np.empty((emax + 1, n), dtype=np.uint8)
    rc = _load().gko_sweep_prefix(reads.ctypes.data, refs.ctypes.data, n, L, stride, emax,
                                  int(edge_fix), acc.ctypes.data, err.ctypes.data, nthreads)
    if rc:
        raise ValueError(f"gko_sweep_prefix rejected arguments (rc={rc})")
    return acc, err


def levenshtein(a, b) -> int:
    x, y = _as_bytes(a), _as_bytes(b)
    return _load().gko_levenshtein(x.ctypes.data, int(x.shape[0]), y.ctypes.data, int(y.shape[0]))


def edit_distance(reads: np.ndarray, refs: np.ndarray, L: int | None = None,
                  nthreads: int | None = None) -> np.ndarray:
    """Global (Levenshtein) edit distance of every pair over its first L bytes."""
    reads = np.ascontiguousarray(reads, dtype=np.uint8)
    refs = np.ascontiguousarray(refs, dtype=np.uint8)
    n, stride = reads.shape
    L = stride if L is None else L
    nthreads = (os.cpu_count() or 1) if nthreads is None else nthreads
    out = np.empty(n, dtype=np.int32)
    rc = _load().gko_edit_batch(reads.ctypes.data, refs.ctypes.data, n, L, stride,
                                out.ctypes.data, nthreads)
    if rc:
        raise ValueError(f"gko_edit_batch rejected arguments (rc={rc})")
    return out


def xor_row(read, ref, shift: int) -> np.ndarray:
    q, r = _as_bytes(read), _as_bytes(ref)
    out = np.zeros(q.shape[0], dtype=np.uint8)
    rc = _load().gko_xor_row(q.ctypes.data, r.ctypes.data, int(q.shape[0]), shift, out.ctypes.data)
    if rc:
        raise ValueError(f"gko_xor_row failed (rc={rc})")
    return out


def amend(mask) -> np.ndarray:
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    out = np.zeros_like(m)
    _load().gko_amend(m.ctypes.data, int(m.shape[0]), out.ctypes.data)
    return out


def count(mask) -> int:
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    return _load().gko_count(m.ctypes.data, int(m.shape[0]))


def pack(seqs: np.ndarray, L: int | None = None):
    """Reference packer for the library's bit-sliced layout -> (words u32, undef u32)."""
    seqs = np.ascontiguousarray(seqs, dtype=np.uint8)
    n, stride = seqs.shape
    L = stride if L is None else L
    tiles = (n + 1023) // 1024
    words = np.zeros(tiles * L * 64, dtype=np.uint32)
    undef = np.zeros(tiles * 32, dtype=np.uint32)
    rc = _load().gko_pack(seqs.ctypes.data, n, L, stride, words.ctypes.data, undef.ctypes.data)
    if rc:
        raise ValueError(f"gko_pack rejected arguments (rc={rc})")
    return words, undef
