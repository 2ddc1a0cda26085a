"""Invariants, closed forms and brute force that pin the CPU oracle.

Each property follows from the paper's definitions or claims, not from the
oracle's code:
  P4  e = 0 accepts a defined pair iff read == reference (amendment cannot
      create 1s in an all-zero Hamming mask; :49, :228 no FA at e=0).
  P5  Hamming distance <= e  ==>  accept (count(amend(H0)) <= popcount(H0)).
  P6  no false rejects against exact edit distance (:224, :530), brute force
      over every pair of length 4 and a sample of length 5..32.
  P7  invariance under a permutation of {A,C,G,T} applied to both sequences
      (masks depend on base equality only, :49 XOR + OR).
  P8  for L = 0 mod 4, reversing both sequences gives the same result
      (deletion and insertion masks swap roles, windows map onto windows).
  P9  accept(e) ==> accept(e+1) (observed, soft).
  P10 closed forms: identical pair, A^L vs C^L, single substitution.
"""
import itertools

import numpy as np
import pytest

import oracle
import pairgen

BASES = np.frombuffer(b"ACGT", dtype=np.uint8)


def all_pairs(L: int):
    n = 4 ** (2 * L)
    idx = np.arange(n, dtype=np.int64)
    digits = np.stack([(idx >> (2 * t)) & 3 for t in range(2 * L)], axis=1)
    seq = BASES[digits]
    return np.ascontiguousarray(seq[:, :L]), np.ascontiguousarray(seq[:, L:])


@pytest.fixture(scope="module")
def pairs4():
    return all_pairs(4)


def test_e0_is_exact_match(pairs4):
    reads, refs = pairs4
    acc, err = oracle.filter(reads, refs, 0)
    equal = (reads == refs).all(axis=1)
    assert (acc.astype(bool) == equal).all()
    assert (err[equal] == 0).all() and (err[~equal] > 0).all()


@pytest.mark.parametrize("e", [0, 1, 2, 3])
def test_no_false_rejects_exhaustive_L4(pairs4, e):
    reads, refs = pairs4
    acc, _ = oracle.filter(reads, refs, e)
    dist = oracle.edit_distance(reads, refs)
    assert ((acc == 0) & (dist <= e)).sum() == 0
    ham = (reads != refs).sum(axis=1)
    assert (acc[ham <= e] == 1).all()  # P5


@pytest.mark.parametrize("L,e", [(5, 1), (5, 2)])
def test_no_false_rejects_exhaustive_L5(L, e):
    reads, refs = all_pairs(L)
    acc, _ = oracle.filter(reads, refs, e)
    dist = oracle.edit_distance(reads, refs)
    assert ((acc == 0) & (dist <= e)).sum() == 0


@pytest.mark.parametrize("L", [7, 13, 16, 31, 32, 33, 64, 100])
def test_no_false_rejects_random(L):
    emax = max(1, L // 10 + 1)
    reads, refs = pairgen.gen_pairs(3000, L, profile=pairgen.PROFILE_BALANCED, emax=emax,
                                    seed=pairgen.SEED + L)
    acc, err = oracle.sweep(reads, refs, emax)
    dist = oracle.edit_distance(reads, refs)
    undefined = err[0] == 255
    for e in range(emax + 1):
        assert ((acc[e] == 0) & (dist <= e) & ~undefined).sum() == 0, e
        ham = (reads[:, :L] != refs[:, :L]).sum(axis=1)
        assert (acc[e][(ham <= e) & ~undefined] == 1).all()


def test_alphabet_permutation_invariance():
    reads, refs = pairgen.gen_pairs(2000, 48, profile=pairgen.PROFILE_PAPER)
    base = [oracle.filter(reads, refs, e) for e in (0, 2, 5)]
    for perm in [b"CATG", b"TGCA", b"GTAC"]:
        lut = np.arange(256, dtype=np.uint8)
        lut[BASES] = np.frombuffer(perm, dtype=np.uint8)
        pr, pf = lut[reads], lut[refs]
        for (a0, c0), e in zip(base, (0, 2, 5)):
            a1, c1 = oracle.filter(pr, pf, e)
            assert (a0 == a1).all() and (c0 == c1).all()


@pytest.mark.parametrize("L", [16, 100])
def test_reversal_invariance(L):
    reads, refs = pairgen.gen_pairs(2000, L, profile=pairgen.PROFILE_PAPER, seed=7)
    for e in (0, 1, 3, 6):
        a0, c0 = oracle.filter(reads, refs, e)
        a1, c1 = oracle.filter(reads[:, ::-1].copy(), refs[:, ::-1].copy(), e)
        assert (a0 == a1).all() and (c0 == c1).all()


def test_accept_monotone_in_e():
    reads, refs = pairgen.gen_pairs(4000, 100, profile=pairgen.PROFILE_PAPER, seed=11)
    acc, _ = oracle.sweep(reads, refs, 10)
    for e in range(10):
        assert ((acc[e] == 1) & (acc[e + 1] == 0)).sum() == 0


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 17, 100, 150, 250, 508])
def test_closed_forms(L):
    rng = np.random.default_rng(L)
    q = bytes(BASES[rng.integers(0, 4, L)])
    for e in sorted({0, 1, L // 10, L - 1}):
        if e >= L:
            continue
        assert oracle.filter_pair(q, q, e) == (1, 0)
    nwin = (L + 3) // 4
    for e in sorted({0, 1, nwin - 1, nwin, L - 1}):
        if e < 0 or e >= L:
            continue
        acc, err = oracle.filter_pair(b"A" * L, b"C" * L, e)
        assert err == nwin and acc == int(nwin <= e)
    # a single substitution is one error; accepted iff e >= 1
    p = L // 2
    r = bytearray(q)
    r[p] = ord("A") if q[p] != ord("A") else ord("C")
    assert oracle.filter_pair(bytes(r), q, 0) == (0, 1)
    if L > 1:
        assert oracle.filter_pair(bytes(r), q, 1) == (1, 1)


def test_amend_examples():
    """Amendment: bounded short 0-runs become 1 (GateKeeper patterns 101, 1001);
    runs touching either end never do (Fig. S.1 :455 '0001', :458 trailing '00')."""
    amend = lambda s: "".join(map(str, oracle.amend(np.array([int(c) for c in s]))))
    assert amend("101") == "111"
    assert amend("1001") == "1111"
    assert amend("10001") == "10001"
    assert amend("0111") == "0111"
    assert amend("0011") == "0011"
    assert amend("1100") == "1100"
    assert amend("110100110001") == "111111110001"


def test_amend_properties():
    for L in range(1, 11):
        for bits in itertools.product([0, 1], repeat=L):
            m = np.array(bits, dtype=np.uint8)
            a = oracle.amend(m)
            assert (a >= m).all()
            assert (oracle.amend(a) == a).all()
            assert oracle.count(a) <= int(m.sum())


def test_count_examples():
    cnt = lambda s: oracle.count(np.array([int(c) for c in s], dtype=np.uint8))
    assert cnt("1111") == 1
    assert cnt("1010") == 2 and cnt("1001") == 2 and cnt("0110") == 1
    assert cnt("1111" * 4 + "1") == 5          # Fig. S.1: 17 ones -> 5 (:468)
    assert cnt("0001" + "1000") == 2           # runs do not cross windows
    assert cnt("00") == 0 and cnt("1") == 1


def test_appendix_vectors():
    """Hand-worked vectors of SURVEY.md Appendix A (readings R1-R9)."""
    ref = "ACGTACGTACGTACGT"
    assert [oracle.filter_pair("ACGTACTACGTACGTA", ref, e) for e in range(4)] == \
        [(0, 3), (1, 1), (1, 1), (1, 3)]
    assert [oracle.filter_pair("ACGTACGGTACGTACG", ref, e) for e in range(4)] == \
        [(0, 3), (1, 1), (1, 1), (1, 3)]
    assert [oracle.filter_pair("ACGTAGGTACGTACGT", ref, e) for e in range(2)] == [(0, 1), (1, 1)]
    assert oracle.filter_pair("TCGAGATTAAA", "ACCTGCCAGCT", 2) == (0, 3)
    assert oracle.filter_pair("TCGAGATTAAA", "ACCTGCCAGCT", 3) == (1, 3)
    assert oracle.filter_pair("A" * 12, "C" * 12, 2) == (0, 3)
    assert oracle.filter_pair("A" * 12, "C" * 12, 3) == (1, 3)


def test_lowercase_is_same_base():
    q, r = pairgen.gen_pairs(500, 60, seed=5)
    for e in (0, 3):
        a0, c0 = oracle.filter(q, r, e)
        a1, c1 = oracle.filter(q | 0x20, r, e)
        assert (a0 == a1).all() and (c0 == c1).all()


def test_edge_fix_reduces_false_accepts():
    """P11: GateKeeper-GPU's edge fix rejects pairs GateKeeper falsely accepts
     -- never the reverse on an accept that is correct, and
    in aggregate fewer false accepts."""
    reads, refs = pairgen.gen_pairs(6000, 100, seed=3)
    dist = oracle.edit_distance(reads, refs)
    for e in (2, 5, 8):
        a_gpu, c_gpu = oracle.filter(reads, refs, e, edge_fix=True)
        a_gk, _ = oracle.filter(reads, refs, e, edge_fix=False)
        defined = c_gpu != 255
        fa_gpu = ((a_gpu == 1) & (dist > e) & defined).sum()
        fa_gk = ((a_gk == 1) & (dist > e) & defined).sum()
        assert fa_gpu <= fa_gk
        # forcing the vacated bits to 1 can only add 1s to the AND (more errors); it
        # must still never reject a pair within edit distance e (:224, :530)
        assert ((a_gpu == 0) & (dist <= e) & defined).sum() == 0
