"""The C-ABI library loads, exports every symbol include/gatekeeper.h declares,
and validates arguments on the host before touching a GPU (CPU-only tests)."""
import ctypes
import os
import re

import pytest

import paper_2103_14978_b200 as gk
from paper_2103_14978_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gatekeeper.h")


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return gk.load_library()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gk_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["gk_encode", "gk_filter", "gk_filter_ascii", "gk_filter_sweep", "gk_compact", "gk_filter_host",
                 "gk_version", "gk_status_string", "gk_last_cuda_error"]:
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert ctypes.cast(getattr(lib, name), ctypes.c_void_p).value


def test_size_queries(lib):
    assert lib.gk_version() >= 10000
    assert lib.gk_packed_words(1, 100) == 100 * 64
    assert lib.gk_packed_words(1024, 100) == 100 * 64
    assert lib.gk_packed_words(1025, 100) == 2 * 100 * 64
    assert lib.gk_undef_words(2048) == 64
    assert lib.gk_result_words(33) == 2
    assert lib.gk_result_words(0) == 0
    assert lib.gk_compact_workspace_bytes(1) >= 4
    assert lib.gk_host_workspace_bytes(1024, 100, 100) > 2 * 1024 * 100


def test_status_strings(lib):
    for rc in range(0, -7, -1):
        assert lib.gk_status_string(rc)


def test_argument_validation_before_any_launch(lib):
    P = 1 << 12  # a fake, never dereferenced pointer (validation fails first)
    assert lib.gk_encode(P, 10, 0, 10, P, P, None) == -2          # len
    assert lib.gk_encode(P, 10, 509, 600, P, P, None) == -2       # len > GK_MAX_LEN
    assert lib.gk_encode(P, 10, 100, 99, P, P, None) == -1        # stride < len
    assert lib.gk_encode(P, -1, 100, 100, P, P, None) == -1       # n < 0
    assert lib.gk_encode(P, 10, 100, 100, P + 4, P, None) == -4   # packed not 16-aligned
    assert lib.gk_encode(None, 0, 100, 100, None, None, None) == 0  # n = 0 no-op
    assert lib.gk_filter(P, P, P, P, 10, 100, 100, P, None, None) == -3   # e >= len
    assert lib.gk_filter(P, P, P, P, 10, 100, -1, P, None, None) == -3
    assert lib.gk_filter(P, P, P, P, 10, 600, 2, P, None, None) == -2
    assert lib.gk_filter(P, P, P, P, 0, 100, 2, None, None, None) == 0
    assert lib.gk_filter(None, P, P, P, 10, 100, 2, P, None, None) == -1
    assert lib.gk_filter_ascii(P, P, 100, 10, 100, 100, P, None, None) == -3
    assert lib.gk_filter_sweep(P, P, P, P, 10, 100, 100, P, None, 0, None) == -3  # e_max >= len
    assert lib.gk_filter_sweep(P, P, P, P, 10, 100, -1, P, None, 0, None) == -3
    assert lib.gk_filter_sweep(P, P, P, P, 10, 0, 0, P, None, 0, None) == -2
    assert lib.gk_filter_sweep(P, P, P, P, 0, 100, 5, None, None, 0, None) == 0
    assert lib.gk_filter_sweep(P, P, None, P, 10, 100, 5, P, None, 0, None) == -1
    assert lib.gk_filter_sweep(P + 8, P, P, P, 10, 100, 5, P, None, 0, None) == -4
    assert lib.gk_filter_ascii(P, P, 2000, 10, 100, 2, P, None, None) == -1  # stride limit
    assert lib.gk_compact(P, 10, P, P, P, 0, None) == -5                    # workspace
    assert lib.gk_compact(P, 1 << 33, P, P, P, 1 << 20, None) == -1
    assert lib.gk_compact_rows(P, 3, 10, 100, P, 100, P, P, 0, None) == -5      # workspace
    assert lib.gk_compact_rows(P, 3, 2, 100, P, 100, P, P, 1 << 20, None) == -1  # bits stride
    assert lib.gk_compact_rows(P, 3, 4, 100, P, 50, P, P, 1 << 20, None) == -1   # idx stride
    assert lib.gk_compact_rows(P, -1, 4, 100, P, 100, P, P, 1 << 20, None) == -1
    assert lib.gk_compact_rows(P, 0, 4, 100, P, 100, P, P, 0, None) == 0
    assert lib.gk_compact_rows_workspace_bytes(100_000, 11) >= 11 * 4
    assert lib.gk_edit_distance(P, P, 100, 10, 0, P, None) == -2
    assert lib.gk_edit_distance(P, P, 99, 10, 100, P, None) == -1
    assert lib.gk_edit_distance(P, None, 100, 10, 100, P, None) == -1
    assert lib.gk_edit_distance(P, P, 100, 10, 100, P + 2, None) == -4
    assert lib.gk_edit_distance(None, None, 100, 0, 100, None, None) == 0
    assert lib.gk_accuracy(P, 4, P, 100, P, 100, P, 2, None, None) == -1    # no counts
    assert lib.gk_accuracy(P, 1, P, 100, P, 100, P, 2, P, None) == -1       # bits stride
    assert lib.gk_accuracy(P, 4, P, 100, P, 100, P, 0, P, None) == 0
    assert lib.gk_plane_words(0) == 1 and lib.gk_plane_words(33) == 3
    assert lib.gk_pack_planes(P, 1, 0, 10, P, None) == -2
    assert lib.gk_pack_planes(P, 1, 100, 10, P, None) == -1     # stride < len
    assert lib.gk_pack_planes(P, 1, 100, 100, P + 4, None) == -4
    assert lib.gk_pack_planes(P, 0, 100, 100, None, None) == 0
    assert lib.gk_gather_windows(P, 1000, P, 10, 0, P, P, None) == -2
    assert lib.gk_gather_windows(P, 1000, P + 4, 10, 100, P, P, None) == -4  # offsets
    assert lib.gk_gather_windows(P, 1000, P, 10, 100, P + 8, P, None) == -4  # packed
    assert lib.gk_gather_windows(P + 8, 1000, P, 10, 100, P, P, None) == -4  # planes
    assert lib.gk_gather_windows(P, 1000, None, 10, 100, P, P, None) == -1
    assert lib.gk_host_index_workspace_bytes(1024, 100, 10) > 2 * 1024 * 16
    assert lib.gk_filter_host_index(P, 10, P, 10, P, P, 10, 100, 100, P, None, P, 1 << 30, 1024,
                                    None) == -3
    assert lib.gk_filter_host_index(P, 10, P, 10, P, P, 10, 100, 5, P, None, P, 1 << 30, 1000,
                                    None) == -1
    assert lib.gk_filter_host_index(P, 10, P, 10, P, P, 10, 100, 5, P, None, P, 10, 1024,
                                    None) == -5
    assert lib.gk_host_workspace_bytes(1024, 100, 100) > 2 * 1024 * 100
    assert lib.gk_filter_host(P, P, 100, 10, 100, 2, P, None, None, None, P, 1 << 30, 1000,
                              None) == -1  # chunk
    assert lib.gk_filter_host(P, P, 100, 10, 100, 2, P, None, None, None, P, 10, 1024, None) == -5
    # indices need a count; neither accept bits nor indices is an error
    assert lib.gk_filter_host(P, P, 100, 10, 100, 2, P, None, P, None, P, 1 << 30, 1024,
                              None) == -1
    assert lib.gk_filter_host(P, P, 100, 10, 100, 2, None, None, None, None, P, 1 << 30, 1024,
                              None) == -1
    import ctypes as C
    es = (C.c_int32 * 2)(1, 100)
    assert lib.gk_filter_host_sweep(P, P, 100, 10, 100, es, 2, P, None, P, 1 << 30, 1024,
                                    None) == -3
    es = (C.c_int32 * 2)(1, 5)
    assert lib.gk_filter_host_sweep(P, P, 100, 10, 100, es, 2, P, None, P, 10, 1024, None) == -5
    assert lib.gk_filter_host_sweep(P, P, 100, 10, 100, es, 0, P, None, P, 10, 1024, None) == -1


def test_product_package_does_not_import_the_oracle():
    src_dir = os.path.join(ROOT, "paper_2103_14978_b200")
    for dirpath, _, files in os.walk(src_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "gk_oracle" not in text and "gko_" not in text, f
                assert "pairgen" not in text, f
