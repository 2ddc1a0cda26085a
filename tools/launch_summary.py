"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def main(path, cmd):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
    untimed = ("pg_gen", "at::", "edit_distance", "accuracy_kernel", "peak_kernel")
    tot = sum(t for k, (c, t) in agg.items() if not any(u in k for u in untimed))
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) of")
    print(f"  {cmd}")
    print("shares exclude the input generator (pg_gen_kernel, untimed setup), torch fills, the")
    print("accuracy harness (edit_distance / accuracy kernels, run after the timed region) and the")
    print("integer-peak microbenchmark (peak_kernel, run before it)")
    print(f"{'kernel':48s} {'launches':>8s} {'total_us':>12s} {'us/launch':>10s} {'share':>7s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = f"{t / tot:7.3f}" if not any(u in k for u in untimed) else "      -"
        print(f"{k:48s} {c:8d} {t:12.1f} {t / c:10.1f} {share}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]) or "?")
