"""Pins of the CPU oracle to values the paper prints (tests/golden/*.json).

These tests do not retype the oracle's formulas: every expected value is text
printed in PAPER.md (cited per fixture) and decoded with the display rule
stated next to it.  A dropped term, a wrong shift direction, a wrong amendment
boundary rule or a popcount-style count each fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.filterwarnings("ignore")


def _bits(s: str) -> np.ndarray:
    return np.array([int(c) for c in s], dtype=np.uint8)


@pytest.fixture(scope="module")
def figS1(golden_dir):
    with open(os.path.join(golden_dir, "figS1.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def fig2(golden_dir):
    with open(os.path.join(golden_dir, "fig2.json")) as f:
        return json.load(f)


def _strip_display(text: str, e: int) -> str:
    s = text.replace(" ", "")
    return s[e:len(s) - e]


def test_figS1_masks_original_gatekeeper(figS1):
    """Fig. S.1: every printed mask of GateKeeper's worked
    example, e = 2, edge fix OFF (the figure shows the original GateKeeper)."""
    e = figS1["e"]
    acc, err, m = oracle.filter_pair(figS1["read"], figS1["reference_segment"], e,
                                     edge_fix=False, masks=True)
    assert len(figS1["reference_segment"]) == 17
    for item in figS1["printed"]:
        expect = _bits(_strip_display(item["text"], e))
        got = m[item["mask"]]
        assert got.tolist() == expect.tolist(), f"PAPER.md:{item['line']} {item['mask']}"
    # Hamming-stage error count printed as 5 (:468): 17 ones in 5 windows.
    assert oracle.count(m["A0"]) == figS1["hamming_stage_count"]
    assert int(m["A0"].sum()) == 17
    # REJECTED (:469-471)
    assert acc == 0


def test_figS1_decision_gatekeeper_gpu(figS1):
    """Same pair with GateKeeper-GPU's edge fix: still rejected."""
    acc, err = oracle.filter_pair(figS1["read"], figS1["reference_segment"], figS1["e"])
    assert acc == 0


def test_figS1_count_is_not_popcount(figS1):
    """17 mismatching bases counted as 5 errors rules out a plain
    popcount and an 8-base window (which gives 3)."""
    a0 = oracle.filter_pair(figS1["read"], figS1["reference_segment"], 2, masks=True)[2]["A0"]
    assert oracle.count(a0) == 5 != int(a0.sum())


def test_fig2_codes_and_xor_rows(fig2):
    """Fig. 2: 2-bit codes of both sequences and the XOR rows
    of the deletion (shift +1) and insertion (shift -1) masks."""
    ref, read = fig2["reference"], fig2["read"]
    codes = lambda s: " ".join(format(oracle.code(c), "02b") for c in s)
    assert codes(ref) == fig2["reference_codes"]
    assert codes(read) == fig2["read_codes"]
    d = fig2["deletion_xor_row"]["text"].split()
    got = [format(int(x), "02b") for x in oracle.xor_row(read, ref, +1)]
    assert got == d[:11]
    i = fig2["insertion_xor_row"]["text"].split()
    got = [format(int(x), "02b") for x in oracle.xor_row(read, ref, -1)]
    assert got == i[1:]


def test_fig2_edge_fix_direction(fig2):
    """Fig. 2 A[D1]* forces the LEADING vacated bit, A[I1]* the TRAILING one
    (PAPER.md:119-131); GateKeeper leaves both at 0."""
    ref, read = fig2["reference"], fig2["read"]
    _, _, off = oracle.filter_pair(read, ref, 1, edge_fix=False, masks=True)
    _, _, on = oracle.filter_pair(read, ref, 1, edge_fix=True, masks=True)
    assert off["AD1"][0] == 0 and on["AD1"][0] == 1
    assert off["AI1"][-1] == 0 and on["AI1"][-1] == 1
    # printed A[D1]* starts with 1, printed A[I1]* ends with 1
    assert fig2["amended_rows"]["A[D1]*"]["text"].split()[0] == "1"
    assert fig2["amended_rows"]["A[I1]*"]["text"].split()[-1] == "1"
    # apart from the forced edges the masks are unchanged
    assert off["AD1"][1:].tolist() == on["AD1"][1:].tolist()
    assert off["AI1"][:-1].tolist() == on["AI1"][:-1].tolist()


def test_undefined_pair_passes():
    """Pairs containing 'N' pass the filter without filtration."""
    ref = "ACGTACGTACGTACGT"
    assert oracle.filter_pair("ACGTNCGTACGTACGT", ref, 0) == (1, 255)
    assert oracle.filter_pair(ref, "ACGTACGTACNTACGT", 3) == (1, 255)
    # a completely different but defined pair is rejected at e = 0
    assert oracle.filter_pair("TTTTTTTTTTTTTTTT", ref, 0)[0] == 0


def test_levenshtein_textbook_values():
    """Ground truth: textbook edit distances."""
    assert oracle.levenshtein("kitten", "sitting") == 3
    assert oracle.levenshtein("flaw", "lawn") == 2
    assert oracle.levenshtein("", "ACGT") == 4
    assert oracle.levenshtein("ACGT", "ACGT") == 0
    assert oracle.levenshtein("GATTACA", "GCATGCU") == 4
