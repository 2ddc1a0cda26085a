"""Full-size parity (PAPER.md:176/:186 evaluate every one of the
30M pairs per set and claim zero false rejects over all of them, :224/:530):
every pair of C2, C3, C4 and all three C5 buckets, on the bench's own path,
compared with the CPU oracle through per-chunk hashes (tests/full_parity.py,
golden written by tools/oracle_hashes.py).  Plus a 1M-pair slice of each that
also runs the non-default paths.
"""
import pytest

import full_parity

pytestmark = pytest.mark.gpu


def _golden_or_skip(name):
    g = full_parity.load_golden()
    if g is None or name not in g.get("workloads", {}):
        pytest.skip(f"no golden hashes for {name} (run tools/oracle_hashes.py)")
    return g


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_size_parity(gk, name):
    _golden_or_skip(name)
    rec = full_parity.run_workload(name)
    assert rec["chunks_mismatching"] == 0, rec


@pytest.mark.parametrize("name,path", [("c2", "packed"), ("c2", "fused"), ("c3", "packed"),
                                       ("c3", "fused"), ("c5", "packed"), ("c5", "fused")])
def test_slice_parity_other_paths(gk, name, path):
    """Both the fused and the encode + filter paths on a 2M-pair slice of every bucket."""
    _golden_or_skip(name)
    rec = full_parity.run_workload(name, path=path, max_pairs=2 << 20)
    assert rec["chunks_mismatching"] == 0, rec
