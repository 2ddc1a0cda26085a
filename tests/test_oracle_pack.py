"""Pins of the oracle's reference packer (gko_pack) with hand-computed words.

gko_pack is the checker of gk_encode's output, so a wrong plane order or a
transposed tile / lane / bit index in it would let the same mistake in the
encoder pass.  The expected words below are worked out by hand from the
layout definition (include/gatekeeper.h, "packed sequence layout"):

    sequence s -> tile t = s // 1024, lane g = (s // 32) % 32, bit j = s % 32;
    word ((t * L + i) * 32 + g) * 2 + p holds at bit j the plane p of base i,
    p = 0: high bit, p = 1: low bit of the 2-bit code A=00 C=01 G=10 T=11
    (PAPER.md:49); undef[t * 32 + g] bit j = 1 iff s has a byte outside
    {A,C,G,T,a,c,g,t} (reading R8).

No value here is produced by the oracle or by the CUDA path.
"""
import numpy as np

import oracle


def _rows(seqs):
    return np.array([np.frombuffer(s.encode(), dtype=np.uint8) for s in seqs])


def _w(L, t, i, g, p):
    return ((t * L + i) * 32 + g) * 2 + p


def test_pack_33_sequences_by_hand():
    L = 3
    seqs = ["AAA"] * 33
    seqs[0] = "ACG"    # codes 00 01 10
    seqs[1] = "TTT"    # 11 11 11
    seqs[2] = "gca"    # 10 01 00 (lower case = same base, R8)
    seqs[5] = "ANA"    # undefined
    seqs[32] = "CCC"   # tile 0, lane 1, bit 0
    words, undef = oracle.pack(_rows(seqs), L)
    assert words.shape == (1 * L * 64,) and undef.shape == (32,)
    expect = np.zeros_like(words)
    # lane 0: bits 0 (ACG), 1 (TTT), 2 (gca)
    # base 0: A=00 T=11 g=10 -> high {1,2} = 0b110, low {1} = 0b010
    expect[_w(L, 0, 0, 0, 0)] = 0b110
    expect[_w(L, 0, 0, 0, 1)] = 0b010
    # base 1: C=01 T=11 c=01 -> high {1} = 0b010, low {0,1,2} = 0b111
    expect[_w(L, 0, 1, 0, 0)] = 0b010
    expect[_w(L, 0, 1, 0, 1)] = 0b111
    # base 2: G=10 T=11 a=00 -> high {0,1} = 0b011, low {1} = 0b010
    expect[_w(L, 0, 2, 0, 0)] = 0b011
    expect[_w(L, 0, 2, 0, 1)] = 0b010
    # lane 1: only sequence 32 = CCC -> low plane bit 0 at every base
    for i in range(L):
        expect[_w(L, 0, i, 1, 1)] = 0b1
    assert (words == expect).all(), np.nonzero(words != expect)
    expect_u = np.zeros_like(undef)
    expect_u[0] = 1 << 5
    assert (undef == expect_u).all()


def test_pack_1025_sequences_by_hand():
    L = 3
    seqs = ["AAA"] * 1025
    seqs[1000] = "tac"    # lane 31 (1000 // 32), bit 8 (1000 % 32)
    seqs[1023] = "NNN"    # lane 31, bit 31: undefined
    seqs[1024] = "TGC"    # tile 1, lane 0, bit 0
    seqs[64] = "AaT"      # lane 2, bit 0
    words, undef = oracle.pack(_rows(seqs), L)
    assert words.shape == (2 * L * 64,) and undef.shape == (64,)
    expect = np.zeros_like(words)
    # tile 0 lane 31 bit 8: t=11, a=00, c=01
    expect[_w(L, 0, 0, 31, 0)] = 1 << 8
    expect[_w(L, 0, 0, 31, 1)] = 1 << 8
    expect[_w(L, 0, 2, 31, 1)] = 1 << 8
    # tile 0 lane 2 bit 0: A, a, T -> only base 2 (T = 11)
    expect[_w(L, 0, 2, 2, 0)] = 1
    expect[_w(L, 0, 2, 2, 1)] = 1
    # tile 1 lane 0 bit 0: T=11, G=10, C=01
    expect[_w(L, 1, 0, 0, 0)] = 1
    expect[_w(L, 1, 0, 0, 1)] = 1
    expect[_w(L, 1, 1, 0, 0)] = 1
    expect[_w(L, 1, 2, 0, 1)] = 1
    assert (words == expect).all(), np.nonzero(words != expect)
    expect_u = np.zeros_like(undef)
    expect_u[31] = 1 << 31
    assert (undef == expect_u).all()


def test_pack_respects_stride_and_length():
    # only the first L bytes of a row are read (bytes beyond are 'N' here)
    rows = _rows(["ACGTNNNN", "TGCANNNN"])
    words, undef = oracle.pack(rows, 4)
    assert (undef == 0).all()
    # base 3: T (11) for seq 0, A (00) for seq 1 -> high 0b01, low 0b01
    assert words[_w(4, 0, 3, 0, 0)] == 0b01 and words[_w(4, 0, 3, 0, 1)] == 0b01
    # base 0: A (00), T (11) -> 0b10 in both planes
    assert words[_w(4, 0, 0, 0, 0)] == 0b10 and words[_w(4, 0, 0, 0, 1)] == 0b10
