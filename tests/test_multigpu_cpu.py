"""Multi-rank host logic (world size 2, gloo, CPU): sharding of the seeded pair
stream, max-over-ranks timing and the accepted-pair totals all-reduce used by
bench.py.  Each rank filters its shard with the oracle; the all-reduced totals
must equal a single-process run over the whole batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_14978_b200 import sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_per_rank, L, es, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import pairgen

    idx0, n = sharding.weak_shard(n_per_rank, rank)
    reads, refs = pairgen.gen_pairs(n, L, idx0=idx0, nthreads=1)
    counts = []
    for e in es:
        acc, _ = oracle.filter(reads, refs, e, nthreads=1)
        counts.append(int(acc.sum()))
    totals = sharding.sum_over_ranks(counts)
    tmax = sharding.max_over_ranks(float(rank + 1))
    if rank == 0:
        out.put((totals, tmax))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_totals_match_single_process():
    world, n_per_rank, L, es = 2, 1500, 100, [0, 2, 5]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_per_rank, L, es, q))
             for r in range(world)]
    for p in procs:
        p.start()
    totals, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    import oracle
    import pairgen

    reads, refs = pairgen.gen_pairs(world * n_per_rank, L)
    expect = [int(oracle.filter(reads, refs, e)[0].sum()) for e in es]
    assert totals == expect
    assert tmax == float(world)


def test_shard_ranges_cover_the_stream():
    for world in (1, 2, 3, 8):
        n_total = 1_000_003
        spans = [sharding.even_shard(n_total, r, world) for r in range(world)]
        assert spans[0][0] == 0
        assert sum(c for _, c in spans) == n_total
        for (a, c), (b, _) in zip(spans, spans[1:]):
            assert a + c == b
    assert sharding.weak_shard(30_000_000, 3) == (90_000_000, 30_000_000)


def test_weak_shards_are_disjoint_slices_of_one_stream():
    import pairgen

    a = pairgen.gen_pairs(200, 50, idx0=0)
    b = pairgen.gen_pairs(100, 50, idx0=sharding.weak_shard(100, 1)[0])
    assert (a[0][100:] == b[0]).all() and (a[1][100:] == b[1]).all()
