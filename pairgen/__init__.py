"""pairgen -- seeded synthetic (read, reference segment) pairs.

TEST / BENCH INFRASTRUCTURE, not the product and not the oracle: it holds no
arithmetic of the GateKeeper-GPU method, only the input recipe (DESIGN.md,
"Input recipe").  The same C header (``pairgen.h``) is compiled for the host
(gcc -> ``libpairgen_host.so``, used to feed the CPU oracle) and for the device
(nvcc -> ``libpairgen_cuda.so``, used to fill HBM for the bench), so both sides
see byte-identical pairs (checked by tests/test_pairgen.py on a GPU box).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SEED = 2103149780
PROFILE_PAPER = 0
PROFILE_BALANCED = 1
MAX_LEN = 508

_HOST_SO = os.path.join(HERE, "libpairgen_host.so")
_CUDA_SO = os.path.join(HERE, "libpairgen_cuda.so")
_host = None
_cuda = None


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build(cuda: bool = True) -> None:
    """Compile the host generator (gcc) and, if ``cuda``, the device generator (nvcc)."""
    hdr = os.path.join(HERE, "pairgen.h")
    src = os.path.join(HERE, "pairgen_host.c")
    if _stale(_HOST_SO, [hdr, src]):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", _HOST_SO, src])
    if cuda:
        dsrc = os.path.join(HERE, "pairgen_dev.cu")
        if _stale(_CUDA_SO, [hdr, dsrc]):
            subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                                   "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
                                   "-o", _CUDA_SO, dsrc])


def _load_host():
    global _host
    if _host is None:
        build(cuda=False)
        lib = ctypes.CDLL(_HOST_SO)
        lib.pg_gen_pairs.restype = ctypes.c_int
        lib.pg_gen_pairs.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                     ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_int]
        _host = lib
    return _host


def _load_cuda():
    global _cuda
    if _cuda is None:
        if not os.path.exists(_CUDA_SO):
            build(cuda=True)
        lib = ctypes.CDLL(_CUDA_SO)
        lib.pg_gen_pairs_cuda.restype = ctypes.c_int
        lib.pg_gen_pairs_cuda.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                          ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p]
        _cuda = lib
    return _cuda


def default_emax(L: int) -> int:
    """Largest e the paper sweeps for a read length: 10% of L."""
    return max(0, (L + 9) // 10)


def gen_pairs(n: int, L: int, *, seed: int = SEED, idx0: int = 0,
              profile: int = PROFILE_PAPER, emax: int | None = None,
              stride: int | None = None, nthreads: int | None = None):
    """Return (reads, refs) as numpy uint8 arrays of shape (n, stride)."""
    stride = L if stride is None else stride
    emax = default_emax(L) if emax is None else emax
    nthreads = (os.cpu_count() or 1) if nthreads is None else nthreads
    reads = np.empty((n, stride), dtype=np.uint8)
    refs = np.empty((n, stride), dtype=np.uint8)
    rc = _load_host().pg_gen_pairs(seed, idx0, n, L, profile, emax,
                                   reads.ctypes.data, refs.ctypes.data, stride, nthreads)
    if rc != 0:
        raise ValueError(f"pg_gen_pairs rejected arguments (rc={rc})")
    return reads, refs


def gen_pairs_cuda(n: int, L: int, *, seed: int = SEED, idx0: int = 0,
                   profile: int = PROFILE_PAPER, emax: int | None = None,
                   stride: int | None = None, device=None):
    """Generate the same pairs as :func:`gen_pairs` directly into device memory.

    Returns (reads, refs) as torch.uint8 CUDA tensors of shape (n, stride).
    """
    import torch

    stride = L if stride is None else stride
    emax = default_emax(L) if emax is None else emax
    device = torch.device("cuda") if device is None else torch.device(device)
    reads = torch.empty((n, stride), dtype=torch.uint8, device=device)
    refs = torch.empty((n, stride), dtype=torch.uint8, device=device)
    stream = torch.cuda.current_stream(device).cuda_stream
    rc = _load_cuda().pg_gen_pairs_cuda(seed, idx0, n, L, profile, emax,
                                        reads.data_ptr(), refs.data_ptr(), stride, stream)
    if rc != 0:
        raise RuntimeError(f"pg_gen_pairs_cuda failed (rc={rc})")
    return reads, refs
