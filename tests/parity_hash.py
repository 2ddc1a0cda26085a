"""Per-chunk 64-bit hashes of (accept, errcount) rows for full-size parity.

TEST INFRASTRUCTURE (not method arithmetic).  For pair p (GLOBAL index of the
seeded stream), threshold e, accept bit a and error count c:

    key  = p << 16 | e << 9 | c << 1 | a
    hash = sum over the chunk's pairs of splitmix64_finalize(key + 0x9E3779B97F4A7C15)  (mod 2^64)

An order-independent sum, so the device side can reduce it with atomics.  The
oracle side (this numpy code, fed by oracle.sweep_prefix) and the device side
(tests/native/parity_hash.cu, fed by the CUDA path's outputs) implement the
same definition independently; a single differing (a, c) changes the chunk
hash with probability 1 - 2^-64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

GOLDEN_GAMMA = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)

HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(HERE, "native", "parity_hash.cu")
_SO = os.path.join(HERE, "native", "libparity_hash.so")
_lib = None


def hash_rows_np(p0: int, accept: np.ndarray, err: np.ndarray, es) -> list[int]:
    """accept/err: (rows, m) uint8 for pairs p0 .. p0+m-1; one hash per row."""
    m = accept.shape[1]
    p = (np.arange(m, dtype=np.uint64) + np.uint64(p0)) << np.uint64(16)
    out = []
    with np.errstate(over="ignore"):
        for j, e in enumerate(es):
            key = p | (np.uint64(e) << np.uint64(9)) | (err[j].astype(np.uint64) << np.uint64(1)) \
                | accept[j].astype(np.uint64)
            z = key + GOLDEN_GAMMA
            z = (z ^ (z >> np.uint64(30))) * C1
            z = (z ^ (z >> np.uint64(27))) * C2
            z = z ^ (z >> np.uint64(31))
            out.append(int(np.sum(z, dtype=np.uint64)))
    return out


def build() -> str:
    if not os.path.exists(_SO) or os.path.getmtime(_SRC) > os.path.getmtime(_SO):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-Xcompiler", "-fPIC", "-shared", "-o", _SO, _SRC])
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.ph_hash_rows.argtypes = [P, I64, P, I64, I64, I, P, I64, I64, I64, P, I64, P]
        lib.ph_hash_rows.restype = I
        _lib = lib
    return _lib


def hash_rows_cuda(accept_bits, errc, n: int, es, p_first: int, bucket_idx0: int,
                   out, chunk: int) -> None:
    """Accumulate (atomically) the hashes of a device batch into out[(rows, nchunks)].

    accept_bits: int32 (rows, words) bit rows (bit p%32 of word p/32); errc: uint8
    (rows, >= n); pair i of the batch is global pair p_first + i; its chunk is
    (p_first + i - bucket_idx0) // chunk.  out: int64 CUDA tensor, zeroed by the caller.
    """
    import torch

    rows = len(es)
    e_t = torch.tensor(list(es), dtype=torch.int32, device=out.device)
    rc = _load().ph_hash_rows(accept_bits.data_ptr(), accept_bits.stride(0), errc.data_ptr(),
                              errc.stride(0), n, rows, e_t.data_ptr(), p_first, bucket_idx0,
                              chunk, out.data_ptr(), out.shape[1],
                              ctypes.c_void_p(torch.cuda.current_stream(out.device).cuda_stream))
    if rc:
        raise RuntimeError(f"ph_hash_rows failed ({rc})")
    torch.cuda.synchronize(out.device)
    del e_t


def to_u64(x: int) -> int:
    return x & 0xFFFFFFFFFFFFFFFF
