"""workloads -- the synthetic workloads of BASELINE.json's configs, in one place.

TEST / BENCH INFRASTRUCTURE (no method arithmetic): sizes, read lengths,
thresholds and the pair-index ranges of the seeded stream (pairgen) that
bench.py, tools/ and tests/ all use, so that a bench line, a parity record and
the oracle's golden hashes describe the same pairs.

Pair p of a workload is pairgen pair p (seed 2103149780, profile "paper").
C5's three length buckets are consecutive ranges of one 1B-pair index space:
[0, 333333334) at 100 bp, [333333334, 666666667) at 150 bp and
[666666667, 1000000000) at 250 bp, with e = floor(5% of L) (BASELINE configs[4]).
"""
from __future__ import annotations

from dataclasses import dataclass, field

SEED = 2103149780
HASH_CHUNK = 1 << 20  # pairs per parity-hash chunk (bucket-relative)


@dataclass(frozen=True)
class Bucket:
    L: int          # read length (bp)
    es: tuple       # thresholds computed for this bucket (rows)
    idx0: int       # first global pair index
    n: int          # pairs

    @property
    def emax(self) -> int:
        return max(self.es)


@dataclass(frozen=True)
class Workload:
    name: str
    config_index: int          # BASELINE.json configs[i]
    description: str
    buckets: tuple = field(default_factory=tuple)

    @property
    def n_total(self) -> int:
        return sum(b.n for b in self.buckets)


def _c5_buckets(total: int = 1_000_000_000):
    lens = [(100, 5), (150, 7), (250, 12)]
    out, start = [], 0
    for b, (L, e) in enumerate(lens):
        n = total // 3 + (1 if b < total % 3 else 0)
        out.append(Bucket(L, (e,), start, n))
        start += n
    return tuple(out)


WORKLOADS = {
    "c2": Workload("c2", 1, "30M pairs, 100 bp, e swept 0-10",
                   (Bucket(100, tuple(range(11)), 0, 30_000_000),)),
    "c3": Workload("c3", 2, "30M pairs, 150 bp, e swept 0-15",
                   (Bucket(150, tuple(range(16)), 0, 30_000_000),)),
    "c4": Workload("c4", 3, "30M pairs, 250 bp, e swept 0-25 (multi-word masks)",
                   (Bucket(250, tuple(range(26)), 0, 30_000_000),)),
    "c5": Workload("c5", 4, "1B pairs, 100/150/250 bp mix, e = 5% of L (5/7/12)",
                   _c5_buckets()),
}


def chunks(bucket: Bucket, chunk: int = HASH_CHUNK):
    """(first global index, count) of every parity-hash chunk of a bucket."""
    out = []
    for c0 in range(0, bucket.n, chunk):
        out.append((bucket.idx0 + c0, min(chunk, bucket.n - c0)))
    return out
