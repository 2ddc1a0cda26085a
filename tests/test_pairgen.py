"""The seeded input generator (test infrastructure): determinism and recipe stats."""
import numpy as np
import pytest

import oracle
import pairgen


def test_deterministic_and_threading_independent():
    a = pairgen.gen_pairs(5000, 100, nthreads=1)
    b = pairgen.gen_pairs(5000, 100, nthreads=8)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    c = pairgen.gen_pairs(1000, 100, idx0=4000, nthreads=3)
    assert (c[0] == a[0][4000:]).all() and (c[1] == a[1][4000:]).all()
    d = pairgen.gen_pairs(1000, 100, seed=pairgen.SEED + 1)
    assert (d[0] != a[0][:1000]).any()


def test_stride_padding():
    r, f = pairgen.gen_pairs(100, 37, stride=48)
    r2, f2 = pairgen.gen_pairs(100, 37)
    assert (r[:, :37] == r2).all() and (f[:, :37] == f2).all()
    assert (r[:, 37:] == ord("\n")).all() and (f[:, 37:] == ord("\n")).all()


def test_paper_profile_alphabet_and_undefined_rate():
    r, f = pairgen.gen_pairs(200000, 100)
    both = np.concatenate([r.ravel(), f.ravel()])
    assert set(np.unique(both).tolist()) <= set(b"ACGTN")
    und = ((r == ord("N")).any(1) | (f == ord("N")).any(1)).mean()
    assert 0.0015 < und < 0.0045   # Set_3: 0.31% undefined


def test_balanced_profile_has_edge_alphabet():
    r, f = pairgen.gen_pairs(20000, 100, profile=pairgen.PROFILE_BALANCED, emax=5)
    both = set(np.unique(np.concatenate([r.ravel(), f.ravel()])).tolist())
    assert set(b"acgt") <= both and ord("N") in both
    assert len(both - set(b"ACGTNacgtn")) > 0   # IUPAC codes


def test_paper_profile_accept_rate_is_in_the_paper_range():
    """Calibration check against Table S.2: GateKeeper-GPU accepts
    1.1% / 10.3% / 57.4% of Set_3 at e = 2 / 5 / 10.  The synthetic mix is a
    coarse analogue; it must land within a factor of ~3 at each point."""
    r, f = pairgen.gen_pairs(20000, 100)
    acc, _ = oracle.sweep(r, f, 10)
    rates = acc.mean(axis=1)
    for e, paper in [(2, 0.011), (5, 0.103), (10, 0.574)]:
        assert paper / 3.5 < rates[e] < paper * 3.5, (e, rates[e])


def test_far_pairs_share_a_seed():
    r, f = pairgen.gen_pairs(2000, 100)
    # every pair shares at least 16 equal consecutive bases or is an edited copy
    eq = (r == f)
    run = np.zeros(len(r), dtype=int)
    cur = np.zeros(len(r), dtype=int)
    for i in range(100):
        cur = np.where(eq[:, i], cur + 1, 0)
        run = np.maximum(run, cur)
    assert (run >= 1).all()


@pytest.mark.gpu
def test_host_and_device_generators_agree():
    import torch
    for L, prof, stride in [(100, 0, 100), (150, 1, 160), (37, 1, 37), (250, 0, 256)]:
        hr, hf = pairgen.gen_pairs(20000, L, profile=prof, stride=stride, idx0=12345)
        dr, df = pairgen.gen_pairs_cuda(20000, L, profile=prof, stride=stride, idx0=12345)
        torch.cuda.synchronize()
        assert (dr.cpu().numpy() == hr).all() and (df.cpu().numpy() == hf).all()
