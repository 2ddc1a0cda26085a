#!/usr/bin/env python
"""Full-size parity record: every pair of C2-C5 on the bench path vs the oracle's golden
chunk hashes (tests/full_parity.py).  Writes profiles/<tag>_full_parity.json.

    python tools/full_parity.py --tag r02a [--only c2,c5] [--path packed]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import full_parity  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--only", default="c2,c3,c4,c5")
    ap.add_argument("--path", default=None)
    a = ap.parse_args()
    import torch

    import paper_2103_14978_b200 as gk
    gk.load_library()
    recs = []
    for name in a.only.split(","):
        recs.append(full_parity.run_workload(name, path=a.path))
    out = {"tag": a.tag, "gpu": torch.cuda.get_device_name(0),
           "golden": "tests/golden/full_parity.json (tools/oracle_hashes.py: pairgen + oracle only)",
           "all_match": all(r["chunks_mismatching"] == 0 for r in recs),
           "pairs_compared": sum(r["pairs_compared"] for r in recs), "workloads": recs}
    path = os.path.join(ROOT, "profiles", f"{a.tag}_full_parity.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "workloads"}))
    sys.exit(0 if out["all_match"] else 1)


if __name__ == "__main__":
    main()
