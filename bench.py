#!/usr/bin/env python
"""bench.py -- throughput of the GateKeeper-GPU hot path on B200 (one JSON line).

Default (N=1): BASELINE.json configs[1] -- 30M synthetic pairs of 100 bp, error
threshold swept e = 0..10.  One step = the whole hot path (SURVEY.md 8(a)
a1..a7) over the batch for every e of the sweep: gk_encode of the reads and of
the reference segments (a1, independent of e, once per step), then per e
gk_filter (a2..a6: Hamming / shifted masks, amendment, edge fix, AND, windowed
count, decision) and gk_compact (a7: ordered indices of the accepted pairs).
--path fused runs gk_filter_ascii (a1..a6 in one kernel, re-encoding for every
e) + gk_compact instead.  The metric is filtrations per second (pairs x
thresholds / s), in G pairs/s.

Multi-GPU (torchrun, one process per GPU): every rank filters its own shard of
the same size (weak scaling, no collective on the data path); time = max over
ranks of the device time; an NCCL all-reduce of the accepted-pair totals runs
after the timed region only.

--impl reference: the CPU oracle (oracle/), as it stands, timed on this host's
cores on a bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (n_pairs per GPU, read length, e values, BASELINE configs index)
    "c2": (30_000_000, 100, list(range(0, 11)), 1),
    "c3": (30_000_000, 150, list(range(0, 16)), 2),
    "c4": (30_000_000, 250, list(range(0, 26)), 3),
}
BASE_SEED = 2103149780


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2", choices=sorted(CONFIGS) + ["c5"])
    p.add_argument("--total", type=int, default=1_000_000_000,
                   help="c5: total pairs over all ranks (the 100/150/250 bp mix)")
    p.add_argument("--mem-gb", type=float, default=100.0,
                   help="c5: device memory budget for resident inputs per rank")
    p.add_argument("--path", default="sweep", choices=["sweep", "packed", "fused"],
                   help="sweep: gk_encode x2 + gk_filter_sweep (all e in one pass); packed: "
                        "gk_encode x2 + gk_filter per e; fused: gk_filter_ascii per e")
    p.add_argument("--no-alt", action="store_true",
                   help="skip the extra timing of the per-e packed path")
    p.add_argument("--n", type=int, default=None, help="override pairs per GPU")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample", type=int, default=None)
    return p.parse_args()


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
                 "--format=csv,noheader,nounits", "-lms", "200"],
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
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def load_traffic(workload):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    kernels of this workload, from the newest committed ncu --set full capture
    (profiles/r*_traffic.json, written by tools/ncu_traffic.py); None if absent."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json"))):
        try:
            with open(path) as f:
                d = json.load(f)
        except (OSError, ValueError):
            continue
        if d.get("workload") == workload:
            best = {}
            for k, v in d.get("kernels", {}).items():
                name = k.split("(")[0].strip()
                best[name] = int(v["traffic_bytes_per_launch"])
                # a templated kernel is also found by its base name
                best.setdefault(name.split("<")[0].strip(), best[name])
    return best


def cpu_baseline(cfg_name, sample_pairs=None, budget_s=15.0):
    """The oracle, as it stands, on this host's cores over a bounded sample."""
    import oracle
    import pairgen
    n_full, L, es, _ = CONFIGS[cfg_name]
    cores = os.cpu_count() or 1
    sample = sample_pairs
    if sample is None:
        # calibrate: ~budget_s of CPU work over the e sweep
        probe = 2000
        r, f = pairgen.gen_pairs(probe, L)
        t0 = time.perf_counter()
        for e in es:
            oracle.filter(r, f, e, nthreads=cores)
        dt = time.perf_counter() - t0
        sample = int(max(1024, min(n_full, probe * budget_s / max(dt, 1e-6))))
    r, f = pairgen.gen_pairs(sample, L)
    t0 = time.perf_counter()
    for e in es:
        oracle.filter(r, f, e, nthreads=cores)
    dt = time.perf_counter() - t0
    value = sample * len(es) / dt / 1e9
    return {"value": value, "unit": "Gpairs/s", "cores": cores, "kind": "oracle",
            "sample": f"first {sample} pairs of the {n_full}-pair {L} bp batch, e = {es[0]}..{es[-1]}, "
                      f"{dt:.1f} s wall on {cores} threads"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_full, L, es, cidx = CONFIGS[args.config]
    import oracle
    import pairgen
    cores = os.cpu_count() or 1
    # bounded sample per step so that warmup + steps end within a few minutes
    probe = 2000
    r, f = pairgen.gen_pairs(probe, L)
    t0 = time.perf_counter()
    for e in es:
        oracle.filter(r, f, e, nthreads=cores)
    per_pair = (time.perf_counter() - t0) / probe
    total_steps = args.steps + args.warmup
    sample = int(max(1024, min(n_full, 120.0 / total_steps / max(per_pair, 1e-9))))
    r, f = pairgen.gen_pairs(sample, L)
    for _ in range(args.warmup):
        for e in es:
            oracle.filter(r, f, e, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for e in es:
            oracle.filter(r, f, e, nthreads=cores)
    dt = time.perf_counter() - t0
    value = sample * len(es) * args.steps / dt / 1e9
    line = {
        "impl": "reference", "metric": "filtered pairs/sec (Gpairs/s)", "value": value,
        "unit": "Gpairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1000 / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": f"{args.config}: {n_full} pairs x {L} bp, e {es[0]}..{es[-1]} "
                               f"(BASELINE configs[{cidx}]); each step a {sample}-pair sample",
                   "read_len": L, "e": f"{es[0]}-{es[-1]}", "profile": "paper", "seed": BASE_SEED},
        "cpu_baseline": {"value": value, "unit": "Gpairs/s", "cores": cores, "kind": "oracle",
                         "sample": f"{sample} pairs per step x {len(es)} thresholds"},
        "e2e": {"value": value, "unit": "Gpairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import pairgen
    import paper_2103_14978_b200 as gk
    from paper_2103_14978_b200 import sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    gk.load_library()

    if args.config == "c5":
        run_c5(args, torch, dist, pairgen, gk, sharding, world, rank, dev)
        if world > 1:
            dist.destroy_process_group()
        return

    n_cfg, L, es, cidx = CONFIGS[args.config]
    n = args.n or n_cfg
    # this rank's shard: pairs [rank*n, (rank+1)*n) of the seeded stream
    idx0, n = sharding.weak_shard(n, rank)
    reads, refs = pairgen.gen_pairs_cuda(n, L, idx0=idx0, device=dev)
    stream = torch.cuda.current_stream(dev)
    rows = len(es) if args.path == "sweep" else 1
    assert es == list(range(len(es)))
    accept = torch.empty((rows, gk.result_words(n)), dtype=torch.int32, device=dev)
    errc = torch.empty((rows, n), dtype=torch.uint8, device=dev)
    idx = torch.empty(n, dtype=torch.int32, device=dev)
    n_acc = torch.zeros(len(es), dtype=torch.int64, device=dev)
    ws = torch.empty(gk.compact_workspace_bytes(n), dtype=torch.uint8, device=dev)
    if args.path == "sweep":
        # a7 for every row in one launch pair: one index list per e
        idx_rows = torch.empty((rows, n), dtype=torch.int32, device=dev)
        ws_rows = torch.empty(gk.compact_rows_workspace_bytes(n, rows), dtype=torch.uint8,
                              device=dev)
    if args.path in ("packed", "sweep"):
        pq = torch.empty(gk.packed_words(n, L), dtype=torch.int32, device=dev)
        pr = torch.empty_like(pq)
        uq = torch.empty(gk.undef_words(n), dtype=torch.int32, device=dev)
        ur = torch.empty_like(uq)
    torch.cuda.synchronize(dev)

    n_ev = len(es)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_ev)]
    ev_enc = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    enc_launches = 0
    if args.path in ("packed", "sweep"):
        enc_launches = 2 * (1 + (1 if n % 128 else 0) + (1 if (n + 1023) // 1024 * 32 > (n + 31) // 32 else 0))
    if args.path == "sweep":
        launches_per_step = 1 + 2 + enc_launches
    else:
        launches_per_step = len(es) * 3 + enc_launches

    def step(record=False, path=args.path):
        if path in ("packed", "sweep"):
            if record:
                ev_enc[0].record(stream)
            gk.encode(reads, L, out=(pq, uq), stream=stream)
            gk.encode(refs, L, out=(pr, ur), stream=stream)
            if record:
                ev_enc[1].record(stream)
        if path == "sweep":
            # a2-a6 for every e in one pass, then a7 per e
            if record:
                ev[0][0].record(stream)
            gk.filter_sweep(pq, pr, uq, ur, n, L, es[-1], accept=accept, errcount=errc,
                            stream=stream)
            if record:
                ev[0][1].record(stream)
            gk.compact_rows(accept, n, idx=idx_rows, n_acc=n_acc, workspace=ws_rows,
                            stream=stream)
            if record:
                ev[0][2].record(stream)
            return
        for j, e in enumerate(es):
            if record:
                ev[j][0].record(stream)
            if path == "fused":
                gk.filter_ascii(reads, refs, e, L, accept=accept[0], errcount=errc[0], stream=stream)
            else:
                gk.filter(pq, pr, uq, ur, n, L, e, accept=accept[0], errcount=errc[0], stream=stream)
            if record:
                ev[j][1].record(stream)
            gk.compact(accept[0], n, idx=idx, n_acc=n_acc[j:j + 1], workspace=ws, stream=stream)
            if record:
                ev[j][2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    time.sleep(0.3)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    filt_ms = [0.0] * n_ev
    comp_ms = [0.0] * n_ev
    t_start.record(stream)
    for _ in range(args.steps):
        step(record=True)
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    # kernel times of the LAST step's launches (events are reused each step)
    n_rec = 1 if args.path == "sweep" else n_ev
    for j in range(n_rec):
        filt_ms[j] = ev[j][0].elapsed_time(ev[j][1])
        comp_ms[j] = ev[j][1].elapsed_time(ev[j][2])
    elapsed = sharding.max_over_ranks(t_start.elapsed_time(t_end), device=dev)
    n_acc_tot = sharding.sum_over_ranks(n_acc, device=dev)
    if world > 1:
        dist.barrier()

    # accuracy (outside the timed region): the paper's FA / FR study (Tables S.2-S.6)
    # on the whole batch -- exact edit distance on the device (gk_edit_distance)
    # against the sweep's decisions (gk_accuracy)
    accuracy = None
    if args.path == "sweep":
        v0 = torch.cuda.Event(enable_timing=True)
        v1 = torch.cuda.Event(enable_timing=True)
        v0.record(stream)
        dist = gk.edit_distance(reads, refs, L, stream=stream)
        v1.record(stream)
        counts = gk.accuracy(accept, errc, dist, n, es, stream=stream)
        torch.cuda.synchronize(dev)
        counts = sharding.sum_over_ranks(counts.flatten(), device=dev)
        accuracy = {"verifier": "gk_edit_distance (Myers bit-vector, exact global distance)",
                    "verifier_ms": round(v0.elapsed_time(v1), 3),
                    "per_e": {str(e): {"accept_rate": round(counts[4 * j + 1] / max(1, counts[4 * j]), 5),
                                       "false_accept_rate": round(counts[4 * j + 2] / max(1, counts[4 * j]), 5),
                                       "false_rejects": int(counts[4 * j + 3])}
                              for j, e in enumerate(es)}}
        del dist

    # the per-e packed path on the same data (context for the sweep's speed-up)
    alt = None
    if args.path == "sweep" and not args.no_alt:
        for _ in range(2):
            step(path="packed")
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a0.record(stream)
        for _ in range(3):
            step(path="packed")
        a1.record(stream)
        torch.cuda.synchronize(dev)
        alt_ms = sharding.max_over_ranks(a0.elapsed_time(a1) / 3, device=dev)
        alt = {"path": "gk_encode x2 + (gk_filter + gk_compact) per e", "steps": 3,
               "ms_per_step": round(alt_ms, 4),
               "value": round(n * len(es) * world / (alt_ms / 1e3) / 1e9, 4)}

    ms_per_step = elapsed / args.steps
    filtrations = n * len(es) * world
    value = filtrations / (ms_per_step / 1e3) / 1e9

    peaks, peak_src = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    clk_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    alu_peak = 148 * 64 * clk_mhz * 1e6 / 1e12  # T int-ops/s: 148 SMs x 4 SMSPs x 16 ALU lanes
    enc_ms = ev_enc[0].elapsed_time(ev_enc[1]) if args.path in ("packed", "sweep") else 0.0

    def alg_ops(e):
        # method-minimum integer ops per pair on bit-sliced words:
        # 5 LOP3 per (position, mask) cell + 8 per position for two window counters
        cells = L * (2 * e + 1) - e * (e + 1)
        return (5 * cells + 8 * L) / 32.0

    def sweep_ops(emax):
        # one pass: the 2*emax+1 masks once + one window counter per e (4 ops per position)
        cells = L * (2 * emax + 1) - emax * (emax + 1)
        return (5 * cells + 4 * L * (emax + 2)) / 32.0

    if args.path == "fused":
        bytes_launch = n * (2 * L) + n / 8 + n
        kname = "gk_filter_ascii (filter_ascii_kernel)"
    elif args.path == "sweep":
        bytes_launch = n * (L / 2) + (n / 8 + n) * n_ev
        kname = "gk_filter_sweep (filter_bt_sweep_kernel)"
    else:
        bytes_launch = n * (L / 2) + n / 8 + n
        kname = "gk_filter (filter_sp_kernel<E> / filter_bt_kernel)"
    tot_ms = sum(filt_ms)
    n_launch = n_rec
    hbm_ach = bytes_launch * n_launch / (tot_ms / 1e3) / 1e9
    if args.path == "sweep":
        alu_ach = n * sweep_ops(es[-1]) / (tot_ms / 1e3) / 1e12
    else:
        alu_ach = sum(n * alg_ops(e) for e in es) / (tot_ms / 1e3) / 1e12
    traffic = load_traffic(f"{args.config}:{args.path}:{n}")

    def entry(kernel, bound, ach, peak, unit, launch_ms, share, extra):
        d = {"bound": bound, "achieved": round(ach, 3), "peak": round(peak, 3), "unit": unit,
             "frac": round(ach / peak, 4), "kernel": kernel,
             "traffic": (traffic.get(kernel, traffic.get(kernel.split("<")[0].strip()))
                         if traffic else None),
             "peak_source": peak_src if unit == "GB/s" else
             f"derived: 148 SM x 64 ALU lanes/clk x {clk_mhz:.0f} MHz (DESIGN.md section 6)",
             "mean_launch_ms": round(launch_ms, 4), "share_of_step": round(share, 4)}
        d.update(extra)
        return d

    kernels = []
    fkernel = {"fused": "filter_ascii_tma_kernel", "sweep": "filter_bt_sweep_kernel",
               "packed": "filter_sp_kernel<E>/filter_bt_kernel"}[args.path]
    fextra = {"api": kname, "bytes_per_launch": bytes_launch,
              "ops_per_pair": round(sweep_ops(es[-1]) if args.path == "sweep" else
                                    sum(alg_ops(e) for e in es) / n_ev, 2),
              "hbm_frac": round(hbm_ach / hbm_peak, 4), "alu_frac": round(alu_ach / alu_peak, 4)}
    if args.path == "fused" or hbm_ach / hbm_peak > alu_ach / alu_peak:
        kernels.append(entry(fkernel, "hbm", hbm_ach, hbm_peak, "GB/s", tot_ms / n_launch,
                             tot_ms / ms_per_step, fextra))
    else:
        kernels.append(entry(fkernel, "alu", alu_ach, alu_peak, "T int-ops/s", tot_ms / n_launch,
                             tot_ms / ms_per_step, fextra))
    if args.path in ("packed", "sweep"):
        enc_bytes_launch = n * L + n * L / 4 + n / 8
        kernels.append(entry("encode_tma_kernel<128, 0, 0, 1>" if L <= 128 else "encode_tma_kernel",
                             "hbm", enc_bytes_launch / (enc_ms / 2 / 1e3) / 1e9, hbm_peak, "GB/s",
                             enc_ms / 2, enc_ms / ms_per_step,
                             {"api": "gk_encode (2 launches per step: reads, reference segments)",
                              "bytes_per_launch": enc_bytes_launch}))
    comp_tot = sum(comp_ms[:n_rec])
    if comp_tot > 0:
        n_claunch = 1 if args.path == "sweep" else n_ev
        comp_bytes = (2 * (n / 8) + 4 * sum(int(x) for x in n_acc_tot) / world) / n_claunch
        kernels.append(entry("compact_write_kernel", "hbm",
                             comp_bytes / (comp_tot / n_claunch / 1e3) / 1e9, hbm_peak, "GB/s",
                             comp_tot / n_claunch, comp_tot / ms_per_step,
                             {"api": "gk_compact_rows (all e)" if args.path == "sweep"
                              else "gk_compact per e", "bytes_per_launch": comp_bytes,
                              "note": "count + write kernels; bytes = accept bits read twice + indices"}))
    # the dominant kernel = the largest share of the step
    roof = dict(max(kernels, key=lambda k: k["share_of_step"]))
    roof["all_kernels"] = [{k: v for k, v in x.items() if k in ("kernel", "bound", "frac", "achieved",
                                                               "unit", "share_of_step", "traffic")}
                           for x in kernels]
    per_e = {}
    for j, e in enumerate(es):
        if args.path == "sweep":
            per_e[str(e)] = {"accepted": int(n_acc_tot[j])}
            continue
        t = filt_ms[j] / 1e3
        per_e[str(e)] = {"filter_ms": round(filt_ms[j], 4), "compact_ms": round(comp_ms[j], 4),
                         "Gpairs_s_filter": round(n / t / 1e9, 3),
                         "hbm_frac": round(bytes_launch / t / 1e9 / hbm_peak, 4),
                         "alu_frac": round(n * alg_ops(e) / t / 1e12 / alu_peak, 4),
                         "accepted": int(n_acc_tot[j])}
    if args.path == "sweep":
        per_e["compact_ms_all_e"] = round(comp_ms[0], 4)
    encode = None
    if args.path in ("packed", "sweep"):
        enc_bytes = 2 * (n * L + n * L / 4 + n / 8)
        encode = {"ms": round(enc_ms, 4), "GB_s": round(enc_bytes / (enc_ms / 1e3) / 1e9, 1),
                  "hbm_frac": round(enc_bytes / (enc_ms / 1e3) / 1e9 / hbm_peak, 4),
                  "bytes": enc_bytes, "share_of_step": round(enc_ms / ms_per_step, 4)}

    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(gk, torch, dev, n, L, es, rank, world, args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.cpu_sample)

    if rank == 0:
        line = {
            "metric": "filtered pairs/sec (Gpairs/s)",
            "value": round(value, 4), "unit": "Gpairs/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {
                "workload": f"{args.config}: {n} pairs x {L} bp per GPU, e swept {es[0]}..{es[-1]} "
                            f"(BASELINE configs[{cidx}]); step = "
                            + ("a1 once, a2-a6 for all e in one pass, a7 per e" if args.path == "sweep"
                               else "per e: a1-a6 + a7"),
                "n_pairs_per_gpu": n, "read_len": L, "e": f"{es[0]}-{es[-1]}",
                "path": {"fused": "gk_filter_ascii + gk_compact per e",
                         "packed": "gk_encode x2 + (gk_filter + gk_compact) per e",
                         "sweep": "gk_encode x2 + gk_filter_sweep + gk_compact_rows (all e)"}[args.path],
                "profile": "paper", "seed": BASE_SEED,
                "l2": f"inputs {2 * n * L / 1e9:.1f} GB per GPU > 126 MB L2 (no flush needed)",
                "parallelism": f"dp{world} (pairs sharded, no data-path collective)"},
            "roofline": roof,
            "encode": encode,
            "per_e": per_e,
            "alt_path": alt,
            "accuracy": accuracy,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


C5_BUCKETS = [(100, 5), (150, 7), (250, 12)]  # e = floor(5% of L) (BASELINE configs[4])


def run_c5(args, torch, dist, pairgen, gk, sharding, world, rank, dev):
    """BASELINE configs[4]: 1B pairs, a 100/150/250 bp mix with e = 5% of L, split
    evenly over the ranks (strong scaling).  Each rank filters its third of every
    length bucket; when its share does not fit in --mem-gb of HBM it is processed in
    resident chunks and the time is the sum of the chunks' device times (the
    paper's kernel-time methodology; inputs generated between chunks,
    outside the timed spans).  One step = the rank's whole share."""
    stream = torch.cuda.current_stream(dev)
    total = args.total
    per_bucket = [total // 3 + (1 if b < total % 3 else 0) for b in range(3)]
    bucket_ms = [0.0, 0.0, 0.0]
    accepted = [0, 0, 0]
    chunks_run = 0
    launches = 0
    for b, (L, e) in enumerate(C5_BUCKETS):
        lo, cnt = sharding.even_shard(per_bucket[b], rank, world)
        bytes_per_pair = 2 * L + L // 2 + 16
        cap = max(1024, int(args.mem_gb * 1e9 / bytes_per_pair) // 1024 * 1024)
        done = 0
        while done < cnt:
            m = min(cap, cnt - done)
            reads, refs = pairgen.gen_pairs_cuda(m, L, idx0=lo + done, device=dev)
            pq = torch.empty(gk.packed_words(m, L), dtype=torch.int32, device=dev)
            pr = torch.empty_like(pq)
            uq = torch.empty(gk.undef_words(m), dtype=torch.int32, device=dev)
            ur = torch.empty_like(uq)
            acc = torch.empty(gk.result_words(m), dtype=torch.int32, device=dev)
            errc = torch.empty(m, dtype=torch.uint8, device=dev)
            idx = torch.empty(m, dtype=torch.int32, device=dev)
            n_acc = torch.zeros(1, dtype=torch.int64, device=dev)
            ws = torch.empty(gk.compact_workspace_bytes(m), dtype=torch.uint8, device=dev)

            def step():
                gk.encode(reads, L, out=(pq, uq), stream=stream)
                gk.encode(refs, L, out=(pr, ur), stream=stream)
                gk.filter(pq, pr, uq, ur, m, L, e, accept=acc, errcount=errc, stream=stream)
                gk.compact(acc, m, idx=idx, n_acc=n_acc, workspace=ws, stream=stream)

            for _ in range(args.warmup):
                step()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            t0.record(stream)
            for _ in range(args.steps):
                step()
            t1.record(stream)
            torch.cuda.synchronize(dev)
            bucket_ms[b] += t0.elapsed_time(t1) / args.steps
            accepted[b] += int(n_acc.item())
            launches += 7 * args.steps
            chunks_run += 1
            done += m
            del reads, refs, pq, pr, uq, ur, acc, errc, idx, ws
            torch.cuda.empty_cache()
    ms_rank = sum(bucket_ms)
    ms = sharding.max_over_ranks(ms_rank, device=dev)
    acc_tot = sharding.sum_over_ranks(accepted, device=dev)
    value = total / (ms / 1e3) / 1e9
    if rank == 0:
        line = {
            "metric": "filtered pairs/sec (Gpairs/s)", "value": round(value, 4), "unit": "Gpairs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"c5: {total} pairs, 100/150/250 bp thirds, e = 5/7/12 "
                                   "(BASELINE configs[4]), split evenly over the ranks",
                       "path": "gk_encode x2 + gk_filter + gk_compact per bucket",
                       "timing": "sum over resident chunks of CUDA-event device time; "
                                 "max over ranks",
                       "parallelism": f"dp{world} (pairs sharded, no data-path collective)"},
            "per_bucket": {f"{L}bp_e{e}": {"ms_rank0": round(bucket_ms[b], 4),
                                           "accepted": acc_tot[b]}
                           for b, (L, e) in enumerate(C5_BUCKETS)},
            "chunks_rank0": chunks_run, "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)


def measure_e2e(gk, torch, dev, n, L, es, rank, world, args):
    """Same metric through the public host-buffer API (gk_filter_host_sweep): every
    step copies the batch host->device once and the results of every e device->host."""
    import pairgen
    n_e2e = n
    # host copies of this rank's shard (pinned)
    r_h, f_h = pairgen.gen_pairs_cuda(n_e2e, L, idx0=rank * n, device=dev)
    hr = torch.empty((n_e2e, L), dtype=torch.uint8, pin_memory=True)
    hf = torch.empty((n_e2e, L), dtype=torch.uint8, pin_memory=True)
    hr.copy_(r_h)
    hf.copy_(f_h)
    del r_h, f_h
    acc = torch.empty((len(es), gk.result_words(n_e2e)), dtype=torch.int32, pin_memory=True)
    err = torch.empty((len(es), n_e2e), dtype=torch.uint8, pin_memory=True)
    chunk = 1 << 21
    ws = torch.empty(gk.host_sweep_workspace_bytes(chunk, L, L, max(es)), dtype=torch.uint8,
                     device=dev)
    torch.cuda.synchronize(dev)

    def one():
        gk.filter_host_sweep(hr, hf, es, L, accept=acc, errcount=err, workspace=ws,
                             chunk_pairs=chunk)

    one()  # warm-up
    steps = max(1, min(args.steps, 3))
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    value = n_e2e * len(es) * world / dt / 1e9
    return {"value": round(value, 4), "unit": "Gpairs/s",
            "h2d_GB_s": round(2 * n_e2e * L / dt / 1e9, 1),
            "note": "bound by the host->device copy of the ASCII pairs (PCIe Gen5 x16, ~55-60 GB/s "
                    "pinned); the device work of a step is ~4 ms of the ~110 ms",
            "h2d_bytes_per_step": 2 * n_e2e * L,
            "d2h_bytes_per_step": (n_e2e // 8 + n_e2e) * len(es),
            "api": "gk_filter_host_sweep (pinned host buffers; each chunk copied + encoded once, "
                   "filtered for every e in one gk_filter_sweep pass; 2-stream pipeline)",
            "n_pairs_per_gpu": n_e2e, "timer": "host wall clock around the synchronous call"}


if __name__ == "__main__":
    main()
