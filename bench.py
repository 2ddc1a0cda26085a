#!/usr/bin/env python
"""bench.py -- throughput of the GateKeeper-GPU hot path on B200 (one JSON line).

Default: BASELINE.json configs[4] (the config the metric is quoted on): 1B
synthetic pairs, a 100/150/250 bp mix with e = 5% of L (5 / 7 / 12), split
evenly over the ranks (strong scaling: the job is fixed, N GPUs share it).
One step = the whole hot path over the rank's share of
every length bucket: the fused ASCII filtration (gk_filter_ascii: a1 encode,
a2 undefined pass, a3-a6 masks / amend / edge fix / AND / count / decision)
and a7 compaction (gk_compact: the ordered indices of the accepted pairs).
Inputs are generated on the device (pairgen) and resident in HBM when a timed
region starts; a share that does not fit the memory budget runs as resident
chunks whose device times add up (the paper's kernel-time method).
value = 1B pairs / (max over ranks of the device time of one step).

--config c2|c3|c4 (BASELINE configs[1..3], 30M pairs per GPU, e swept
0..e_max, weak scaling): one step = gk_encode x2 + gk_filter_sweep (every e in
one pass) + gk_compact_rows; value = filtrations/s (pairs x thresholds).

Multi-GPU: `python bench.py --gpus N` re-launches itself under
torch.distributed.run (one process per GPU, NCCL); the driver's own torchrun
launch is used as is.  No collective touches the data path; the max over
ranks of the device time and the accepted-pair totals are all-reduced after
the timed region (PAPER.md:79 equal batches, :186 slowest device).
--dry-run exercises that orchestration on CPU with gloo and no kernels.

--impl reference: the CPU oracle (oracle/), as it stands, timed on this host's
cores on a bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from pairgen.workloads import SEED, WORKLOADS  # noqa: E402

METRIC = "filtered pairs/sec (Gpairs/s)"

# the paper's own filtering throughput for the same path, with its GPUs named
# (kernel time, 30M real pairs per length; M pairs/s)
PAPER = {
    "c5": {"note": "PAPER.md reports no 1B-pair mix; nearest: GTX 1080 Ti (Pascal), 1 GPU, kernel "
                   "throughput at e=4 (150 bp) / e=5 (100 bp) / e=10 (250 bp, closest to 12)",
           "gpu": "1x NVIDIA GeForce GTX 1080 Ti (Setup_1)",
           "Mpairs_s": {"100bp_e5_host_encoded": 103.9, "100bp_e5_device_encoded": 62.8,
                        "150bp_e4_host_encoded": 85.5, "150bp_e4_device_encoded": 37.1,
                        "250bp_e10_host_encoded": 25.7, "250bp_e10_device_encoded": 16.0},
           "multi_gpu": "8x GTX 1080 Ti: 100 bp e=2 1.333 G pairs/s host-encoded, 0.496 device-encoded "
                        "(Table S.21 :892-899)",
           "source": "Tables S.17-S.19 PAPER.md:815-857"},
    "c2": {"gpu": "1x NVIDIA GeForce GTX 1080 Ti", "Mpairs_s_per_e_host_encoded":
           {"0": 699.7, "1": 282.6, "2": 198.7, "3": 149.7, "4": 122.5, "5": 103.9, "6": 89.7},
           "source": "Table S.17 PAPER.md:815-821"},
    "c3": {"gpu": "1x NVIDIA GeForce GTX 1080 Ti", "Mpairs_s_per_e_host_encoded":
           {"0": 537.7, "1": 193.5, "2": 138.6, "4": 85.5, "6": 62.1, "8": 48.4, "10": 40.8},
           "source": "Table S.18 PAPER.md:831-837"},
    "c4": {"gpu": "1x NVIDIA GeForce GTX 1080 Ti", "Mpairs_s_per_e_host_encoded":
           {"0": 328.2, "1": 132.2, "2": 92.0, "4": 56.5, "6": 40.6, "8": 31.2, "10": 25.7},
           "source": "Table S.19 PAPER.md:851-857"},
}


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c5", choices=["c2", "c3", "c4", "c5"])
    p.add_argument("--path", default="auto", choices=["auto", "fused", "packed", "per-e"],
                   help="auto (default): fused kernels for reads <= 192 bp, encode + filter "
                        "kernels above; fused | packed: force one; per-e (c2-c4): one "
                        "gk_filter launch per threshold instead of the one-pass sweep")
    p.add_argument("--total", type=int, default=None, help="c5: total pairs (default 1B)")
    p.add_argument("--n", type=int, default=None, help="c2-c4: pairs per GPU (default 30M)")
    p.add_argument("--mem-gb", type=float, default=110.0,
                   help="device memory budget for one resident chunk of pairs")
    p.add_argument("--dry-run", action="store_true",
                   help="CPU/gloo: exercise spawning, sharding and the rank reductions only")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-alt", action="store_true", help="c2-c4: skip the per-e comparison path")
    p.add_argument("--cpu-budget", type=float, default=20.0,
                   help="seconds of host work for the oracle baseline")
    return p.parse_args(argv)


def path_of(args, L):
    from paper_2103_14978_b200.pipeline import auto_path
    if args.path == "auto":
        return auto_path(L)
    return "packed" if args.path == "per-e" else args.path


PATH_DESC = {"fused": "fused ASCII kernel", "packed": "gk_encode x2 + filter kernel"}


# ---------------------------------------------------------------------------
# workload description shared by both arms (the driver compares the configs)
def buckets_of(args):
    """[(L, es, idx0, n_total)] of the workload."""
    wl = WORKLOADS[args.config]
    if args.config == "c5":
        if args.total is None:
            return [(b.L, b.es, b.idx0, b.n) for b in wl.buckets]
        out, start = [], 0
        for i, b in enumerate(wl.buckets):
            n = args.total // 3 + (1 if i < args.total % 3 else 0)
            out.append((b.L, b.es, start, n))
            start += n
        return out
    b = wl.buckets[0]
    return [(b.L, b.es, 0, args.n or b.n)]


def config_of(args, world):
    wl = WORKLOADS[args.config]
    bk = buckets_of(args)
    if args.config == "c5":
        total = sum(b[3] for b in bk)
        return {"workload": f"c5: {total} pairs, 100/150/250 bp thirds, e = 5/7/12 "
                            f"(BASELINE configs[{wl.config_index}]), split evenly over the ranks",
                "total_pairs": total,
                "buckets": [{"read_len": L, "e": es[0], "pairs": n,
                             "path": {"fused": "gk_filter_ascii + gk_compact",
                                      "packed": "gk_encode x2 + gk_filter + gk_compact"}[
                                 path_of(args, L)]} for L, es, _, n in bk],
                "profile": "paper", "seed": SEED,
                "l2": "inputs >= 6.6 GB per resident chunk > 126 MB L2 (no flush needed)",
                "parallelism": f"dp{world} (pairs sharded, no data-path collective)"}
    L, es, _, n = bk[0]
    return {"workload": f"{args.config}: {n} pairs x {L} bp per GPU, e swept {es[0]}..{es[-1]} "
                        f"(BASELINE configs[{wl.config_index}])",
            "n_pairs_per_gpu": n, "read_len": L, "e": f"{es[0]}-{es[-1]}",
            "path": ("gk_encode x2 + (gk_filter + gk_compact) per e" if args.path == "per-e" else
                     {"fused": "gk_filter_ascii_sweep (encode + all e in one kernel) + "
                               "gk_compact_rows",
                      "packed": "gk_encode x2 + gk_filter_sweep (all e in one pass) + "
                                "gk_compact_rows"}[path_of(args, L)]),
            "profile": "paper", "seed": SEED,
            "l2": f"inputs {2 * n * L / 1e9:.1f} GB per GPU > 126 MB L2 (no flush needed)",
            "parallelism": f"dp{world} (pairs sharded, no data-path collective)"}


def unit_of(args):
    return "Gpairs/s" if args.config == "c5" else "G filtrations/s (pairs x thresholds)"


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/gk_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured (MEASURED_PEAKS.json)"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


def int_peak():
    """Integer-pipe peaks measured live on this GPU (tools/native/int_peak.cu):
    thread-instructions/s of LOP3 / IADD3 / SHF / PRMT (alu pipe), IMAD (fma pipe)."""
    import ctypes
    so = os.path.join(ROOT, "tools", "native", "libint_peak.so")
    if not os.path.exists(so):
        return None
    lib = ctypes.CDLL(so)
    lib.ip_measure.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.ip_measure.restype = ctypes.c_int
    out = (ctypes.c_double * 6)()
    if lib.ip_measure(ctypes.cast(out, ctypes.c_void_p), 5) != 0:
        return None
    names = ["lop3", "iadd3", "shf", "prmt", "imad", "lop3+imad"]
    return {k: round(v / 1e12, 3) for k, v in zip(names, out)}


def load_ncu(workload):
    """Per-launch DRAM traffic and pipe utilisation of this workload's kernels from the
    committed ncu --set full captures (profiles/r*_traffic.json, written by
    tools/ncu_traffic.py; one capture per kernel, newest file wins per kernel)."""
    import glob
    best = {}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
        except (OSError, ValueError):
            continue
        if d.get("workload") != workload:
            continue
        for k, v in d.get("kernels", {}).items():
            name = k.split("(")[0].replace("void ", "").strip()
            best[name] = dict(v, source=os.path.basename(path), kernel=name)
    return best or None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ---------------------------------------------------------------------------
# the oracle on the host cores
def oracle_rate(L, es, sample, threads):
    """Seconds per pair of the oracle (all thresholds es) on `sample` pairs."""
    import oracle
    import pairgen
    r, f = pairgen.gen_pairs(sample, L, nthreads=os.cpu_count() or 1)
    t0 = time.perf_counter()
    if len(es) == 1:
        oracle.filter(r, f, es[0], nthreads=threads)
    else:
        for e in es:
            oracle.filter(r, f, e, nthreads=threads)
    return (time.perf_counter() - t0) / sample


def cpu_baseline(args, budget_s):
    """The oracle, as it stands, on this host's cores over a bounded sample of every bucket
    (T = nproc and T = 1), scaled to the whole workload."""
    cores = os.cpu_count() or 1
    bk = buckets_of(args)
    per_bucket = budget_s / len(bk)
    t_all, t_one, desc = 0.0, 0.0, []
    for L, es, _, n in bk:
        probe = oracle_rate(L, es, 1024, cores)
        sample = int(max(1024, min(n, 0.8 * per_bucket / max(probe, 1e-12))))
        tp = oracle_rate(L, es, sample, cores)
        s1 = int(max(256, min(sample, 0.2 * per_bucket / max(probe * cores, 1e-12))))
        tp1 = oracle_rate(L, es, s1, 1)
        t_all += n * tp
        t_one += n * tp1
        desc.append(f"{sample} pairs at {L} bp (T={cores}), {s1} (T=1)")
    work = sum(n * len(es) for _, es, _, n in bk)
    return {"value": work / t_all / 1e9, "unit": unit_of(args), "cores": cores, "kind": "oracle",
            "value_1thread": work / t_one / 1e9, "cpu_model": cpu_model(),
            "sample": "; ".join(desc) + f"; scaled to the workload's {work} filtrations",
            "api": "oracle.filter (oracle/gk_oracle.c, plain character-level C, one call per e)"}


def run_reference(args):
    """--impl reference: the oracle on the host cores, each step a bounded sample."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    cores = os.cpu_count() or 1
    bk = buckets_of(args)
    total_steps = args.steps + args.warmup
    per_step = 150.0 / total_steps / len(bk)  # ~2.5 min for the whole run
    samples = []
    for L, es, _, n in bk:
        probe = oracle_rate(L, es, 1024, cores)
        samples.append(int(max(1024, min(n, per_step / max(probe, 1e-12)))))
    import oracle
    import pairgen
    data = [pairgen.gen_pairs(s, L, nthreads=cores) for (L, _, _, _), s in zip(bk, samples)]

    def step():
        t = []
        for (L, es, _, n), (r, f) in zip(bk, data):
            t0 = time.perf_counter()
            for e in es:
                oracle.filter(r, f, e, nthreads=cores)
            t.append(time.perf_counter() - t0)
        return t

    for _ in range(args.warmup):
        step()
    acc = [0.0] * len(bk)
    for _ in range(args.steps):
        for i, x in enumerate(step()):
            acc[i] += x
    # seconds per pair per bucket -> the whole workload's time per step
    t_work = sum(n * acc[i] / args.steps / samples[i] for i, (_, _, _, n) in enumerate(bk))
    work = sum(n * len(es) for _, es, _, n in bk)
    value = work / t_work / 1e9
    sample = ", ".join(f"{s} pairs at {L} bp" for (L, _, _, _), s in zip(bk, samples))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": unit_of(args),
        "n_gpus": int(os.environ.get("WORLD_SIZE", args.gpus)), "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_work * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == "c5" else "weak", "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": config_of(args, int(os.environ.get("WORLD_SIZE", args.gpus))),
        "cpu_baseline": {"value": value, "unit": unit_of(args), "cores": cores, "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"each step: {sample}; time scaled to the whole workload"},
        "e2e": {"value": value, "unit": unit_of(args), "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def spawn_ranks(args):
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_dry(args):
    """CPU / gloo: spawning, sharding and the rank reductions, no kernels."""
    import torch.distributed as dist

    from paper_2103_14978_b200 import sharding
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    shards = []
    for L, es, idx0, n in buckets_of(args):
        lo, cnt = (sharding.even_shard(n, rank, world) if args.config == "c5"
                   else sharding.weak_shard(n, rank))
        shards.append([L, idx0 + lo, cnt])
    counts = sharding.sum_over_ranks([s[2] for s in shards])
    tmax = sharding.max_over_ranks(float(rank + 1))
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": unit_of(args), "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "dry_run": True,
                          "scaling": "strong" if args.config == "c5" else "weak",
                          "config": config_of(args, world), "rank0_shards": shards,
                          "pairs_all_ranks": counts, "max_over_ranks_of_rank_plus_1": tmax}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# algorithmic work per pair
def alg_bytes(kernel, L, es):
    rows = len(es)
    return {"filter_ascii": 2 * L + 1 / 8 + 1,
            "filter_ascii_sweep": 2 * L + rows * (1 / 8 + 1),
            "encode": 2 * (L + L / 4) + 2 / 8,
            "filter": L / 2 + 2 / 8 + 1 / 8 + 1,
            "filter_sweep": L / 2 + 2 / 8 + rows * (1 / 8 + 1),
            "compact": rows * 2 / 8,       # + 4 B per accepted pair, added by the caller
            "compact_rows": rows * 2 / 8}[kernel]


def alg_ops(kernel, L, es):
    """Method-minimum integer ops per pair on bit-sliced words: 5 LOP3 per (position, mask)
    cell (2 mismatch + 3 amend/AND), 4 per position per counted bit-vector (start detect +
    carry-save add), over 32 pairs per word."""
    e = max(es)
    cells = L * (2 * e + 1) - e * (e + 1)
    if kernel in ("filter", "filter_ascii"):
        return (5 * cells + 8 * L) / 32.0
    if kernel in ("filter_sweep", "filter_ascii_sweep"):
        return (5 * cells + 4 * L * (e + 2)) / 32.0
    return 0.0


# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.dry_run:
        run_dry(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2103_14978_b200 as gk
    from paper_2103_14978_b200 import sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (use --dry-run on CPU)")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    gk.load_library()
    ctx = dict(torch=torch, dist=dist, gk=gk, sharding=sharding, world=world, rank=rank, dev=dev)
    line = run_buckets(args, ctx)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_buckets(args, ctx):
    """Time one step (every bucket of the rank's share) and build the JSON line."""
    import pairgen
    from paper_2103_14978_b200.pipeline import BucketStep, SweepStep
    torch, gk, sharding = ctx["torch"], ctx["gk"], ctx["sharding"]
    world, rank, dev = ctx["world"], ctx["rank"], ctx["dev"]
    stream = torch.cuda.current_stream(dev)
    c5 = args.config == "c5"
    bk = buckets_of(args)

    # the share of this rank, in resident chunks
    plan = []
    for L, es, idx0, n in bk:
        lo, cnt = sharding.even_shard(n, rank, world) if c5 else sharding.weak_shard(n, rank)
        per_pair = 2 * L + 8 + len(es) * 6 + (L // 2 if path_of(args, L) == "packed" else 0)
        cap = max(1024, int(args.mem_gb * 1e9 / per_pair) // 1024 * 1024)
        nch = (cnt + cap - 1) // cap
        size = (cnt + nch - 1) // nch
        size = (size + 1023) // 1024 * 1024
        done = 0
        while done < cnt:
            m = min(size, cnt - done)
            plan.append((L, es, idx0 + lo + done, m))
            done += m

    peaks, peak_src = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    ip = int_peak()
    alu_peak = ip["lop3"] if ip else 148 * 64 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    alu_src = ("measured live: LOP3 chains at full occupancy (tools/native/int_peak.cu)" if ip
               else "derived: 148 SM x 64 lanes/clk x max clock (microbenchmark unavailable)")

    sampler = ClockSampler(dev.index)
    step_ms = 0.0
    kern_ms = {}       # kernel family -> ms per step
    kern_work = {}     # kernel family -> (bytes, ops) per step
    per_bucket = {}
    accepted = {}
    launches = 0
    accuracy = None
    sampler_started = False
    for ci, (L, es, p0, m) in enumerate(plan):
        reads, refs = pairgen.gen_pairs_cuda(m, L, idx0=p0, device=dev)
        if c5 or args.path == "per-e":
            steps_obj = [BucketStep(torch, m, L, e, dev, path=path_of(args, L)) for e in es]
        else:
            steps_obj = [SweepStep(torch, m, L, es[-1], dev, path=path_of(args, L))]
        torch.cuda.synchronize(dev)

        def one(record=False):
            for s in steps_obj:
                s.run(reads, refs, stream, record=record)

        for _ in range(args.warmup):
            one()
        torch.cuda.synchronize(dev)
        if world > 1 and ci == 0:
            ctx["dist"].barrier()
        if not sampler_started:
            sampler.start()
            time.sleep(0.2)
            sampler_started = True
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        l0 = gk.launch_count()
        ev0.record(stream)
        for k in range(args.steps):
            one(record=(k == args.steps - 1))
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        launches += gk.launch_count() - l0
        ms = ev0.elapsed_time(ev1) / args.steps
        step_ms += ms
        key = f"{L}bp_e{es[0]}" if c5 else f"{L}bp_e{es[0]}-{es[-1]}"
        pb = per_bucket.setdefault(key, {"ms": 0.0, "pairs": 0, "chunks": 0})
        pb["ms"] += ms
        pb["pairs"] += m
        pb["chunks"] += 1
        for s in steps_obj:
            for kname, kms in s.timer.ms().items():
                kern_ms[kname] = kern_ms.get(kname, 0.0) + kms
                kes = s.es if hasattr(s, "es") else es
                b = alg_bytes(kname, L, kes) * m
                if kname.startswith("compact"):
                    b += 4 * int(s.n_acc.sum().item())
                o = alg_ops(kname, L, kes) * m
                w = kern_work.setdefault(kname, [0.0, 0.0, []])
                w[0] += b
                w[1] += o
                w[2].append({"bucket": key, "ms": round(kms, 4), "pairs": m,
                             "GB_s": round(b / (kms / 1e3) / 1e9, 1),
                             "T_ops_s": round(o / (kms / 1e3) / 1e12, 3)})
            acc_rows = s.n_acc.tolist()
            for j, e in enumerate(s.es if hasattr(s, "es") else es):
                accepted[f"{key}:{e}"] = accepted.get(f"{key}:{e}", 0) + int(acc_rows[j])
        if not c5 and args.path != "per-e" and ci == len(plan) - 1:
            # the paper's accuracy study (Tables S.2-S.6) on the whole batch, after the timed
            # region: exact edit distance on the device vs the sweep's decisions
            st = steps_obj[0]
            dist_ = gk.edit_distance(reads, refs, L, stream=stream)
            counts = gk.accuracy(st.accept, st.errc, dist_, m, es, stream=stream)
            torch.cuda.synchronize(dev)
            counts = sharding.sum_over_ranks(counts.flatten(), device=dev)
            accuracy = {"verifier": "gk_edit_distance (Myers bit-vector, exact global distance)",
                        "per_e": {str(e): {
                            "accept_rate": round(counts[4 * j + 1] / max(1, counts[4 * j]), 5),
                            "false_accept_rate": round(counts[4 * j + 2] / max(1, counts[4 * j]), 5),
                            "false_rejects": int(counts[4 * j + 3])} for j, e in enumerate(es)}}
            del dist_
        del steps_obj, reads, refs
        torch.cuda.empty_cache()
    clocks = sampler.stop()

    ms_all = sharding.max_over_ranks(step_ms, device=dev)
    keys = sorted(accepted)
    acc_tot = dict(zip(keys, sharding.sum_over_ranks([accepted[k] for k in keys], device=dev)))
    work = sum(n * len(es) for _, es, _, n in bk) if c5 else sum(
        n * len(es) for _, es, _, n in bk) * world
    value = work / (ms_all / 1e3) / 1e9

    # roofline of every kernel family; the dominant one is the largest share of the step
    ncu = load_ncu(f"{args.config}:{args.path}")  # profiles/r*_traffic.json of this workload
    if ncu is None and args.path == "auto":
        ncu = load_ncu(f"{args.config}:auto")
    kernels = []
    for kname, kms in kern_ms.items():
        b, o, parts = kern_work[kname]
        hbm = b / (kms / 1e3) / 1e9
        alu = o / (kms / 1e3) / 1e12
        bound = "alu" if alu / alu_peak > hbm / hbm_peak else "hbm"
        ent = {"kernel": kname, "bound": bound,
               "achieved": round(alu if bound == "alu" else hbm, 3),
               "peak": round(alu_peak if bound == "alu" else hbm_peak, 3),
               "unit": "T int-ops/s" if bound == "alu" else "GB/s",
               "frac": round((alu / alu_peak) if bound == "alu" else (hbm / hbm_peak), 4),
               "hbm_frac": round(hbm / hbm_peak, 4), "alu_frac": round(alu / alu_peak, 4),
               "share_of_step": round(kms / step_ms, 4), "ms_per_step": round(kms, 4),
               "algorithmic_bytes_per_step": b, "algorithmic_ops_per_step": o,
               "per_launch_group": parts,
               "peak_source": alu_src if bound == "alu" else peak_src}
        if ncu:
            fam = {"encode": "encode3", "filter": "filter_", "compact": "compact_write",
                   "compact_rows": "compact_write", "filter_sweep": "filter_bt2_sweep",
                   "filter_ascii": "fused_kernel", "filter_ascii_sweep": "fused_kernel"}[kname]
            hit = [v for k, v in sorted(ncu.items()) if fam in k and
                   (kname != "filter" or "sweep" not in k)]
            if hit:
                ent["traffic"] = hit[0].get("traffic_bytes_per_launch")
                ent["traffic_kernel"] = hit[0]["kernel"]
                ent["traffic_source"] = hit[0]["source"]
                ent["ncu_per_instantiation"] = [
                    {k2: h[k2] for k2 in ("kernel", "traffic_bytes_per_launch", "pipe_alu_pct",
                                          "pipe_fma_pct", "issue_pct", "source") if k2 in h}
                    for h in hit]
                if "pipe_alu_pct" in hit[0]:
                    ent["ncu_pipe_alu_pct"] = hit[0]["pipe_alu_pct"]
        ent.setdefault("traffic", None)
        kernels.append(ent)
    roof = dict(max(kernels, key=lambda k: k["share_of_step"]))
    roof["all_kernels"] = [{k: v for k, v in x.items() if k in (
        "kernel", "bound", "frac", "hbm_frac", "alu_frac", "achieved", "unit", "share_of_step",
        "traffic")} for x in kernels]

    e2e = None if args.no_e2e else measure_e2e(args, ctx, bk)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, args.cpu_budget)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": unit_of(args), "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_all, 4),
        "higher_is_better": True, "scaling": "strong" if c5 else "weak", "vs_baseline": None,
        "dtype": "u32", "data": "synthetic", "config": config_of(args, world),
        "pairs_per_s": round(sum(n for *_, n in bk) * (1 if c5 else world) / (ms_all / 1e3) / 1e9, 4),
        "roofline": roof, "per_bucket": per_bucket, "accepted": acc_tot,
        "int_peak_T_ops_s": ip, "gpu_launches": launches, "clocks": clocks, "e2e": e2e,
        "cpu_baseline": cpu, "paper": PAPER[args.config], "accuracy": accuracy,
        "timing": "CUDA events on the launching stream around K steps after W warm-ups, per "
                  "resident chunk; step time = sum over the rank's chunks; max over ranks",
    }
    if c5:
        line["chunks_rank0"] = len(plan)
    return line


def measure_e2e(args, ctx, bk):
    """The same metric through the public host-buffer C-ABI calls: every step copies a
    sample of each bucket's pairs host->device (pinned) and the results device->host.
    c5: gk_filter_host (encode + filter + compaction per chunk, 2-stream pipeline; the
    accepted indices come back); c2-c4:
    gk_filter_host_sweep.  Time per pair per bucket x the bucket's share = the step."""
    import pairgen
    torch, gk, sharding = ctx["torch"], ctx["gk"], ctx["sharding"]
    world, rank, dev = ctx["world"], ctx["rank"], ctx["dev"]
    c5 = args.config == "c5"
    t_step, t_sample, h2d, d2h, desc = 0.0, 0.0, 0, 0, []
    for L, es, idx0, n in bk:
        lo, cnt = sharding.even_shard(n, rank, world) if c5 else sharding.weak_shard(n, rank)
        # pinned host sample per rank (8M pairs per bucket at N=1, less per rank at N>1
        # so that N ranks of one node do not pin N x 8 GB)
        ns = min(cnt, max(1 << 20, ((1 << 23) // world) // 1024 * 1024))
        r_d, f_d = pairgen.gen_pairs_cuda(ns, L, idx0=idx0 + lo, device=dev)
        hr = torch.empty((ns, L), dtype=torch.uint8, pin_memory=True)
        hf = torch.empty((ns, L), dtype=torch.uint8, pin_memory=True)
        hr.copy_(r_d)
        hf.copy_(f_d)
        del r_d, f_d
        torch.cuda.empty_cache()
        rows = len(es)
        acc = torch.empty((rows, gk.result_words(ns)), dtype=torch.int32, pin_memory=True)
        err = torch.empty((rows, ns), dtype=torch.uint8, pin_memory=True)
        chunk = 1 << 21
        if c5:
            ws = torch.empty(gk.host_workspace_bytes(chunk, L, L), dtype=torch.uint8, device=dev)
            idx = torch.empty(ns, dtype=torch.uint32, pin_memory=True)

            def one():
                gk.filter_host(hr, hf, es[0], L, want_accept=False, indices=True, idx=idx,
                               workspace=ws, chunk_pairs=chunk)
        else:
            ws = torch.empty(gk.host_sweep_workspace_bytes(chunk, L, L, max(es)),
                             dtype=torch.uint8, device=dev)

            def one():
                gk.filter_host_sweep(hr, hf, list(es), L, accept=acc, errcount=err, workspace=ws,
                                     chunk_pairs=chunk)
        torch.cuda.synchronize(dev)
        one()
        reps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(reps):
            one()
        dt = (time.perf_counter() - t0) / reps
        t_step += dt * cnt / ns
        t_sample += dt
        h2d += 2 * ns * L
        if c5:
            _, _, got = gk.filter_host(hr, hf, es[0], L, want_accept=False, indices=True, idx=idx,
                                       workspace=ws, chunk_pairs=chunk)
            d2h += 4 * got.numel() + 8 * ((ns + chunk - 1) // chunk)
        else:
            d2h += rows * (ns // 8 + ns)
        desc.append(f"{ns} of {cnt} pairs at {L} bp")
        del hr, hf, acc, err, ws
        if c5:
            del idx
        torch.cuda.empty_cache()
    t_all = sharding.max_over_ranks(t_step, device=dev)
    work = sum(n * len(es) for _, es, _, n in bk) * (1 if c5 else world)
    # the PCIe roofline of this number: a plain pinned host->device copy on this box
    buf_h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    buf_d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    buf_d.copy_(buf_h, non_blocking=True)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        buf_d.copy_(buf_h, non_blocking=True)
    e1.record()
    torch.cuda.synchronize(dev)
    h2d_peak = 3 * (1 << 30) / (e0.elapsed_time(e1) / 1e3) / 1e9
    del buf_h, buf_d
    h2d_rate = h2d / t_sample / 1e9
    return {"value": round(work / t_all / 1e9, 4), "unit": unit_of(args),
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "bytes_note": "h2d/d2h bytes of one timed repetition (the sample below); value is "
                          "scaled from the sample's time per pair to the whole workload",
            "h2d_GB_s": round(h2d_rate, 2), "h2d_copy_peak_GB_s": round(h2d_peak, 2),
            "pcie_frac": round(h2d_rate / h2d_peak, 4),
            "api": ("gk_filter_host (pinned host ASCII; per 2M-pair chunk gk_encode x2 + gk_filter "
                    "+ gk_compact, only the accepted pairs' indices come back; 2 CUDA streams "
                    "overlapping H2D / kernels / D2H)" if c5 else
                    "gk_filter_host_sweep (pinned host ASCII; each chunk copied + encoded once, "
                    "one gk_filter_sweep pass for every e)"),
            "sample": "per bucket " + "; ".join(desc) + ": host wall clock around the synchronous "
                      "call, time per pair x the rank's pairs; max over ranks",
            "bound": "host->device copy of the ASCII pairs (PCIe)"}


if __name__ == "__main__":
    main()
