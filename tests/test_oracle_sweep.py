"""Pins of the oracle's one-pass threshold sweep (gko_sweep_pair / oracle.sweep_prefix).

The one-pass sweep relies on the prefix property of the AND chain
(PAPER.md:49 "2e+1 masks", :51 "AND"): F_e = F_{e-1} AND A*D_e AND A*I_e.  It is
pinned row for row against e_max+1 independent filtrations (oracle.sweep, i.e.
gko_filter_pair at each e, itself pinned by test_oracle_pins / _invariants), on
inputs with every feature the readings touch: undefined bytes (R8), lower case,
IUPAC codes, early accepts (R5), e = 0, edge fix on and off (R4, NEXT-4), and
lengths that are not multiples of 4 or 32 (R7, R13).  It also reproduces the
Appendix A vectors, whose errcount is not monotone in e (R5).
"""
import numpy as np
import pytest

import oracle
import pairgen


@pytest.mark.parametrize("L,emax", [(1, 0), (2, 1), (5, 3), (13, 4), (31, 6), (33, 7),
                                    (100, 10), (150, 15), (250, 25)])
@pytest.mark.parametrize("edge_fix", [True, False])
def test_prefix_sweep_equals_independent_filtrations(L, emax, edge_fix):
    n = 3000 if L < 200 else 1200
    reads, refs = pairgen.gen_pairs(n, L, profile=pairgen.PROFILE_BALANCED, emax=max(emax, 1),
                                    seed=pairgen.SEED + 17 * L)
    a1, c1 = oracle.sweep(reads, refs, emax, edge_fix=edge_fix)
    a2, c2 = oracle.sweep_prefix(reads, refs, emax, edge_fix=edge_fix)
    for e in range(emax + 1):
        assert (a1[e] == a2[e]).all(), e
        assert (c1[e] == c2[e]).all(), e


def test_prefix_sweep_paper_profile_with_stride():
    L, emax = 100, 10
    reads, refs = pairgen.gen_pairs(4000, L, stride=112)
    a1, c1 = oracle.sweep(reads, refs, emax, L=L)
    a2, c2 = oracle.sweep_prefix(reads, refs, emax, L=L)
    assert (a1 == a2).all() and (c1 == c2).all()


def test_prefix_sweep_appendix_a_vectors():
    # del1@6 -> e = 0/1/2/3 gives (0,3) (1,1) (1,1) (1,3)
    read = np.frombuffer(b"ACGTACTACGTACGTA", dtype=np.uint8)[None, :]
    ref = np.frombuffer(b"ACGTACGTACGTACGT", dtype=np.uint8)[None, :]
    a, c = oracle.sweep_prefix(read, ref, 3)
    assert a[:, 0].tolist() == [0, 1, 1, 1]
    assert c[:, 0].tolist() == [3, 1, 1, 3]
    # Fig. S.1 pair: REJECT with 5 at e=0, 4 at e = 1..3
    read = np.frombuffer(b"TCGAGATTAAATCTCCT", dtype=np.uint8)[None, :]
    ref = np.frombuffer(b"ACCTGCCACCCGGAGTC", dtype=np.uint8)[None, :]
    a, c = oracle.sweep_prefix(read, ref, 3)
    assert a[:, 0].tolist() == [0, 0, 0, 0]
    assert c[:, 0].tolist() == [5, 4, 4, 4]
    # an 'N' makes every row (1, 255)
    read = np.frombuffer(b"ACGTNCGTACGTACGT", dtype=np.uint8)[None, :]
    a, c = oracle.sweep_prefix(read, ref[:, :16], 5)
    assert (a == 1).all() and (c == 255).all()


def test_prefix_sweep_rejects_bad_arguments():
    r = np.zeros((2, 8), dtype=np.uint8) + ord("A")
    with pytest.raises(ValueError):
        oracle.sweep_prefix(r, r, 8)   # e must be < L
    with pytest.raises(ValueError):
        oracle.sweep_prefix(r, r, -1)
