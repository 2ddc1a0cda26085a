"""bench.py's host-side orchestration on CPU (no GPU): `--gpus 2` re-launches itself
under torch.distributed.run with two ranks (gloo in --dry-run), shards every bucket
of the workload, reduces over ranks and prints one JSON line with n_gpus = 2."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=300):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                       capture_output=True, text=True, timeout=timeout, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus", [1, 2])
def test_dry_run_c5_strong_shards(gpus):
    d = _run(["--gpus", str(gpus), "--dry-run"])
    assert d["n_gpus"] == gpus and d["dry_run"] is True and d["scaling"] == "strong"
    # every bucket of the 1B-pair mix is covered exactly once over the ranks
    assert d["pairs_all_ranks"] == [b["pairs"] for b in d["config"]["buckets"]]
    assert sum(d["pairs_all_ranks"]) == 1_000_000_000
    assert d["max_over_ranks_of_rank_plus_1"] == float(gpus)
    assert d["config"]["parallelism"].startswith(f"dp{gpus}")


def test_dry_run_c2_weak_shards():
    d = _run(["--gpus", "2", "--dry-run", "--config", "c2"])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["pairs_all_ranks"] == [60_000_000]
    assert d["rank0_shards"] == [[100, 0, 30_000_000]]


def test_reference_arm_config_matches_ours():
    sys.path.insert(0, ROOT)
    import bench
    a = bench.parse(["--config", "c5"])
    b = bench.parse(["--config", "c5", "--impl", "reference"])
    assert bench.config_of(a, 1) == bench.config_of(b, 1)
    assert bench.unit_of(a) == bench.unit_of(b)
