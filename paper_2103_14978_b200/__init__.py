"""paper_2103_14978_b200 -- B200-native GateKeeper-GPU pre-alignment filter.

Thin Python binding over the C ABI of ``libgk.so`` (include/gatekeeper.h):
argument marshalling only.  Every step of the filter runs in the library's
CUDA kernels; there is no CPU path.  If ``libgk.so`` is missing or cannot be
loaded, importing the functions below raises -- the product never falls back
to anything else.

Tensors are torch tensors (PyTorch provides device memory and streams only).
Names follow the paper: ``encode``, ``filter`` /
``filter_ascii`` (the filtration, :79, :105-109), ``compact`` (accepted pairs
handed to verification, :166-168).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GK_LIB", os.path.join(HERE, "libgk.so"))
GK_MAX_LEN = 508
GK_MAX_STRIDE = 1024
GK_TILE = 1024
GK_FLAG_GENERIC = 1
GK_FLAG_NO_EDGE_FIX = 2
GK_FLAG_BLOCKED = 4

_lib = None


class GateKeeperError(RuntimeError):
    pass


def load_library(path: str = LIB_PATH):
    """Load libgk.so and declare the C ABI.  Raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise GateKeeperError(
            f"{path} not found: build it with `python -m paper_2103_14978_b200._build` "
            "(or __graft_entry__.build()); there is no fallback path")
    lib = ctypes.CDLL(path)
    P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    sig = {
        "gk_version": (ctypes.c_int, []),
        "gk_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "gk_last_cuda_error": (ctypes.c_int, []),
        "gk_launch_count": (ctypes.c_uint64, []),
        "gk_packed_words": (SZ, [I64, I32]),
        "gk_undef_words": (SZ, [I64]),
        "gk_result_words": (SZ, [I64]),
        "gk_encode": (ctypes.c_int, [P, I64, I32, I64, P, P, P]),
        "gk_filter": (ctypes.c_int, [P, P, P, P, I64, I32, I32, P, P, P]),
        "gk_filter_ex": (ctypes.c_int, [P, P, P, P, I64, I32, I32, P, P, I32, P]),
        "gk_filter_sweep": (ctypes.c_int, [P, P, P, P, I64, I32, I32, P, P, I32, P]),
        "gk_filter_ascii": (ctypes.c_int, [P, P, I64, I64, I32, I32, P, P, P]),
        "gk_filter_ascii_sweep": (ctypes.c_int, [P, P, I64, I64, I32, I32, P, P, P]),
        "gk_compact_workspace_bytes": (SZ, [I64]),
        "gk_compact": (ctypes.c_int, [P, I64, P, P, P, SZ, P]),
        "gk_compact_rows_workspace_bytes": (SZ, [I64, I32]),
        "gk_edit_distance": (ctypes.c_int, [P, P, I64, I64, I32, P, P]),
        "gk_plane_words": (SZ, [I64]),
        "gk_host_index_workspace_bytes": (SZ, [I64, I32, I32]),
        "gk_filter_host_index": (ctypes.c_int, [P, I64, P, I64, P, P, I64, I32, I32, P, P, P, SZ,
                                                I64, P]),
        "gk_pack_planes": (ctypes.c_int, [P, I64, I64, I64, P, P]),
        "gk_gather_windows": (ctypes.c_int, [P, I64, P, I64, I32, P, P, P]),
        "gk_accuracy": (ctypes.c_int, [P, I64, P, I64, P, I64, P, I32, P, P]),
        "gk_compact_rows": (ctypes.c_int, [P, I32, I64, I64, P, I64, P, P, SZ, P]),
        "gk_host_workspace_bytes": (SZ, [I64, I64, I32]),
        "gk_filter_host": (ctypes.c_int, [P, P, I64, I64, I32, I32, P, P, P, P, P, SZ, I64, P]),
        "gk_host_sweep_workspace_bytes": (SZ, [I64, I64, I32, I32]),
        "gk_filter_host_sweep": (ctypes.c_int, [P, P, I64, I64, I32, P, I32, P, P, P, SZ, I64, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(rc: int, what: str):
    if rc != 0:
        lib = load_library()
        msg = lib.gk_status_string(rc).decode()
        if rc == -6:
            msg += f" (cudaError {lib.gk_last_cuda_error()})"
        raise GateKeeperError(f"{what} failed: {msg} [{rc}]")


def _stream(stream=None):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def launch_count() -> int:
    """Kernels launched through libgk.so by this process so far (gk_launch_count)."""
    return int(load_library().gk_launch_count())


# ---- size queries -------------------------------------------------------------
def packed_words(n: int, length: int) -> int:
    return load_library().gk_packed_words(n, length)


def undef_words(n: int) -> int:
    return load_library().gk_undef_words(n)


def result_words(n: int) -> int:
    return load_library().gk_result_words(n)


# ---- a1: encode ---------------------------------------------------------------
def encode(seqs, length: int | None = None, out=None, stream=None):
    """ASCII rows (uint8 CUDA tensor [n, stride]) -> (packed u32 words, undef u32 words)."""
    import torch
    n, stride = seqs.shape
    length = stride if length is None else length
    if out is None:
        packed = torch.empty(packed_words(n, length), dtype=torch.int32, device=seqs.device)
        undef = torch.empty(undef_words(n), dtype=torch.int32, device=seqs.device)
    else:
        packed, undef = out
    _check(load_library().gk_encode(seqs.data_ptr(), n, length, stride, _ptr(packed), _ptr(undef),
                                    _stream(stream)), "gk_encode")
    return packed, undef


# ---- a2..a6: filter -----------------------------------------------------------
def filter(reads_packed, refs_packed, read_undef, ref_undef, n: int, length: int, e: int,
           accept=None, errcount=None, want_errcount: bool = True, flags: int = 0,
           stream=None):
    """Filtration of n packed pairs -> (accept bits u32[ceil(n/32)], errcount u8[n] or None)."""
    import torch
    dev = reads_packed.device
    if accept is None:
        accept = torch.empty(max(1, result_words(n)), dtype=torch.int32, device=dev)
    if errcount is None and want_errcount:
        errcount = torch.empty(max(1, n), dtype=torch.uint8, device=dev)
    _check(load_library().gk_filter_ex(_ptr(reads_packed), _ptr(refs_packed), _ptr(read_undef),
                                       _ptr(ref_undef), n, length, e, _ptr(accept),
                                       _ptr(errcount), flags, _stream(stream)), "gk_filter")
    return accept, errcount


def filter_sweep(reads_packed, refs_packed, read_undef, ref_undef, n: int, length: int,
                 e_max: int, accept=None, errcount=None, want_errcount: bool = True,
                 flags: int = 0, stream=None):
    """Every threshold e = 0..e_max in one pass -> (accept bits u32[e_max+1, ceil(n/32)],
    errcount u8[e_max+1, n] or None); row e equals filter(..., e)."""
    import torch
    dev = reads_packed.device
    rows = e_max + 1
    if accept is None:
        accept = torch.empty((rows, max(1, result_words(n))), dtype=torch.int32, device=dev)
    if errcount is None and want_errcount:
        errcount = torch.empty((rows, max(1, n)), dtype=torch.uint8, device=dev)
    _check(load_library().gk_filter_sweep(_ptr(reads_packed), _ptr(refs_packed), _ptr(read_undef),
                                          _ptr(ref_undef), n, length, e_max, _ptr(accept),
                                          _ptr(errcount), flags, _stream(stream)), "gk_filter_sweep")
    return accept, errcount


def filter_ascii(reads, refs, e: int, length: int | None = None, accept=None, errcount=None,
                 want_errcount: bool = True, stream=None):
    """Fused a1..a6 from ASCII rows -> (accept bits, errcount or None)."""
    import torch
    n, stride = reads.shape
    length = stride if length is None else length
    if accept is None:
        accept = torch.empty(max(1, result_words(n)), dtype=torch.int32, device=reads.device)
    if errcount is None and want_errcount:
        errcount = torch.empty(max(1, n), dtype=torch.uint8, device=reads.device)
    _check(load_library().gk_filter_ascii(reads.data_ptr(), refs.data_ptr(), stride, n, length,
                                          e, _ptr(accept), _ptr(errcount), _stream(stream)),
           "gk_filter_ascii")
    return accept, errcount


def filter_ascii_sweep(reads, refs, e_max: int, length: int | None = None, accept=None,
                       errcount=None, want_errcount: bool = True, stream=None):
    """Fused a1..a6 for every e = 0..e_max from ASCII rows -> (accept bits [e_max+1, words],
    errcount [e_max+1, n] or None); row e equals filter_ascii(..., e)."""
    import torch
    n, stride = reads.shape
    length = stride if length is None else length
    rows = e_max + 1
    if accept is None:
        accept = torch.empty((rows, max(1, result_words(n))), dtype=torch.int32,
                             device=reads.device)
    if errcount is None and want_errcount:
        errcount = torch.empty((rows, max(1, n)), dtype=torch.uint8, device=reads.device)
    _check(load_library().gk_filter_ascii_sweep(reads.data_ptr(), refs.data_ptr(), stride, n,
                                                length, e_max, _ptr(accept), _ptr(errcount),
                                                _stream(stream)), "gk_filter_ascii_sweep")
    return accept, errcount


# ---- a7: compact --------------------------------------------------------------
def _check_index_range(n: int):
    if n >= 1 << 31:
        raise GateKeeperError(f"compact: n = {n} >= 2^31 would return negative int32 indices; "
                              "split the batch (the C ABI itself takes n < 2^32)")


def compact_workspace_bytes(n: int) -> int:
    return load_library().gk_compact_workspace_bytes(n)


def compact(accept, n: int, idx=None, n_acc=None, workspace=None, want_indices: bool = True,
            stream=None):
    """Ordered indices of accepted pairs -> (idx u32[n] (first n_acc valid), n_acc u64[1]).
    The indices are u32 (the C ABI's); the default idx tensor is int32, so n is capped
    below 2^31 here (pass a larger int32 buffer viewed as u32 to the C ABI directly)."""
    import torch
    _check_index_range(n)
    dev = accept.device
    if idx is None and want_indices:
        idx = torch.empty(max(1, n), dtype=torch.int32, device=dev)
    if n_acc is None:
        n_acc = torch.empty(1, dtype=torch.int64, device=dev)
    wsb = compact_workspace_bytes(n)
    if workspace is None:
        workspace = torch.empty(max(1, wsb), dtype=torch.uint8, device=dev)
    _check(load_library().gk_compact(accept.data_ptr(), n, _ptr(idx), n_acc.data_ptr(),
                                     workspace.data_ptr(), workspace.numel(), _stream(stream)),
           "gk_compact")
    return idx, n_acc


def compact_rows_workspace_bytes(n: int, rows: int) -> int:
    return load_library().gk_compact_rows_workspace_bytes(n, rows)


def compact_rows(accept, n: int, idx=None, n_acc=None, workspace=None, want_indices: bool = True,
                 stream=None):
    """a7 for every row of a 2-D accept tensor [rows, >= ceil(n/32)] (e.g. filter_sweep's)
    in one launch pair -> (idx u32 [rows, n] or None, n_acc i64 [rows]); n < 2^31 (see
    compact)."""
    import torch
    _check_index_range(n)
    rows = accept.shape[0]
    dev = accept.device
    if idx is None and want_indices:
        idx = torch.empty((rows, max(1, n)), dtype=torch.int32, device=dev)
    if n_acc is None:
        n_acc = torch.empty(rows, dtype=torch.int64, device=dev)
    if workspace is None:
        workspace = torch.empty(max(1, compact_rows_workspace_bytes(n, rows)), dtype=torch.uint8,
                                device=dev)
    _check(load_library().gk_compact_rows(accept.data_ptr(), rows, accept.stride(0), n, _ptr(idx),
                                          idx.stride(0) if idx is not None else 0, n_acc.data_ptr(),
                                          workspace.data_ptr(), workspace.numel(),
                                          _stream(stream)), "gk_compact_rows")
    return idx, n_acc


# ---- reference-index mode -----------------------------------------------------
def pack_planes(rows, length: int | None = None, stream=None):
    """ASCII rows (uint8 CUDA [n_rows, stride]; a genome is one row) -> interleaved bit
    planes, int32 [gk_plane_words(n_rows*length), 4] = (hi, lo, undef, 0) per 32 bases."""
    import torch
    n_rows, stride = rows.shape
    length = stride if length is None else length
    words = load_library().gk_plane_words(n_rows * length)
    planes = torch.empty((words, 4), dtype=torch.int32, device=rows.device)
    _check(load_library().gk_pack_planes(rows.data_ptr(), n_rows, length, stride,
                                         planes.data_ptr(), _stream(stream)), "gk_pack_planes")
    return planes


def gather_windows(planes, n_bases: int, offsets, length: int, out=None, stream=None):
    """Windows [offsets[p], offsets[p]+length) of bit planes -> (packed words, undef
    words) in the layout of encode()."""
    import torch
    n = offsets.numel()
    dev = offsets.device
    if out is None:
        packed = torch.empty(max(1, packed_words(n, length)), dtype=torch.int32, device=dev)
        undef = torch.empty(max(1, undef_words(n)), dtype=torch.int32, device=dev)
    else:
        packed, undef = out
    _check(load_library().gk_gather_windows(planes.data_ptr(), n_bases, offsets.data_ptr(), n,
                                            length, packed.data_ptr(), undef.data_ptr(),
                                            _stream(stream)),
           "gk_gather_windows")
    return packed, undef


def filter_host_index(read_planes, read_bases: int, ref_planes, ref_bases: int, read_offsets,
                      ref_offsets, length: int, e_max: int, accept=None, errcount=None,
                      workspace=None, chunk_pairs: int = 1 << 21, stream=None):
    """Index mode from HOST int64 offset tensors (planes on the device) -> host result
    rows (accept bits [e_max+1, words], errcount [e_max+1, n] or None)."""
    import torch
    n = read_offsets.numel()
    if accept is None:
        accept = torch.empty((e_max + 1, max(1, result_words(n))), dtype=torch.int32,
                             pin_memory=True)
    if workspace is None:
        workspace = torch.empty(load_library().gk_host_index_workspace_bytes(chunk_pairs, length,
                                                                             e_max),
                                dtype=torch.uint8, device=read_planes.device)
    _check(load_library().gk_filter_host_index(read_planes.data_ptr(), read_bases,
                                               ref_planes.data_ptr(), ref_bases,
                                               read_offsets.data_ptr(), ref_offsets.data_ptr(), n,
                                               length, e_max, accept.data_ptr(), _ptr(errcount),
                                               workspace.data_ptr(), workspace.numel(),
                                               chunk_pairs, _stream(stream)), "gk_filter_host_index")
    return accept, errcount


# ---- accuracy harness (not on the filtering path) ------------------------------
def edit_distance(reads, refs, length: int | None = None, out=None, stream=None):
    """Exact global edit distance of every (read, ref) row pair -> int32 [n]."""
    import torch
    n, stride = reads.shape
    length = stride if length is None else length
    if out is None:
        out = torch.empty(max(1, n), dtype=torch.int32, device=reads.device)
    _check(load_library().gk_edit_distance(reads.data_ptr(), refs.data_ptr(), stride, n, length,
                                           out.data_ptr(), _stream(stream)), "gk_edit_distance")
    return out


def accuracy(accept, errcount, dist, n: int, e_list, stream=None):
    """False-accept / false-reject tallies of decision rows (accept [rows, words],
    errcount [rows, n]) against distances -> int64 [rows, 4] (defined, accepted,
    false accepts, false rejects)."""
    import torch
    rows = accept.shape[0]
    es = torch.tensor(list(e_list), dtype=torch.int32, device=accept.device)
    counts = torch.empty((rows, 4), dtype=torch.int64, device=accept.device)
    _check(load_library().gk_accuracy(accept.data_ptr(), accept.stride(0), errcount.data_ptr(),
                                      errcount.stride(0), dist.data_ptr(), n, es.data_ptr(), rows,
                                      counts.data_ptr(), _stream(stream)), "gk_accuracy")
    return counts


# ---- end to end from host buffers ----------------------------------------------
def host_workspace_bytes(chunk_pairs: int, stride: int, length: int | None = None) -> int:
    return load_library().gk_host_workspace_bytes(chunk_pairs, stride,
                                                  stride if length is None else length)


def filter_host(reads, refs, e: int, length: int | None = None, accept=None, errcount=None,
                indices: bool = False, idx=None, workspace=None, chunk_pairs: int = 1 << 20,
                want_accept: bool = True, stream=None):
    """End-to-end filtration of HOST (CPU, ideally pinned) uint8 tensors; results in host
    memory -> (accept bits or None, errcount or None, accepted indices or None).  With
    indices=True the chunks are compacted on the device and only the ascending indices of
    the accepted pairs come back (a uint32 tensor of length n_acc)."""
    import torch
    n, stride = reads.shape
    length = stride if length is None else length
    if accept is None and want_accept:
        accept = torch.empty(max(1, result_words(n)), dtype=torch.int32, pin_memory=True)
    if indices and idx is None:
        idx = torch.empty(max(1, n), dtype=torch.uint32, pin_memory=True)
    n_acc = ctypes.c_uint64(0)
    if workspace is None:
        workspace = torch.empty(host_workspace_bytes(chunk_pairs, stride, length),
                                dtype=torch.uint8, device="cuda")
    _check(load_library().gk_filter_host(reads.data_ptr(), refs.data_ptr(), stride, n, length, e,
                                         _ptr(accept), _ptr(errcount),
                                         _ptr(idx) if indices else None,
                                         ctypes.byref(n_acc) if indices else None,
                                         workspace.data_ptr(), workspace.numel(), chunk_pairs,
                                         _stream(stream)),
           "gk_filter_host")
    return accept, errcount, (idx[:n_acc.value] if indices else None)


def host_sweep_workspace_bytes(chunk_pairs: int, stride: int, length: int, e_max: int) -> int:
    return load_library().gk_host_sweep_workspace_bytes(chunk_pairs, stride, length, e_max)


def filter_host_sweep(reads, refs, e_list, length: int | None = None, accept=None,
                      errcount=None, workspace=None, chunk_pairs: int = 1 << 20, stream=None):
    """Threshold sweep of HOST uint8 tensors: each chunk is copied and encoded once, then
    filtered for every e <= max(e_list) in one pass.  Returns (accept bits [n_e, words], errcount [n_e, n] or None)."""
    import torch
    n, stride = reads.shape
    length = stride if length is None else length
    es = (ctypes.c_int32 * len(e_list))(*e_list)
    if accept is None:
        accept = torch.empty((len(e_list), max(1, result_words(n))), dtype=torch.int32,
                             pin_memory=True)
    if workspace is None:
        workspace = torch.empty(host_sweep_workspace_bytes(chunk_pairs, stride, length,
                                                           max(e_list)),
                                dtype=torch.uint8, device="cuda")
    _check(load_library().gk_filter_host_sweep(reads.data_ptr(), refs.data_ptr(), stride, n,
                                               length, es, len(e_list), accept.data_ptr(),
                                               _ptr(errcount), workspace.data_ptr(),
                                               workspace.numel(), chunk_pairs, _stream(stream)),
           "gk_filter_host_sweep")
    return accept, errcount
