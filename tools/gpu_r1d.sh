#!/bin/bash
# Re-validate the restored tree: bt kernel parity + timing vs the dispatch default,
# the full GPU suite, and the default bench line.
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "sweep or random_lengths or adversarial or ragged or original" > gpurun_out/pytest_bt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bt.log
timeout 600 python tools/cmp_filters.py --L 100 --e 2 5 10 --flags 0 4 > gpurun_out/cmp_bt.jsonl 2>&1
timeout 600 python tools/cmp_filters.py --L 150 --e 7 12 15 --flags 0 4 >> gpurun_out/cmp_bt.jsonl 2>&1
timeout 600 python tools/cmp_filters.py --L 250 --e 5 11 12 18 25 --flags 0 4 >> gpurun_out/cmp_bt.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
tail -3 gpurun_out/pytest_bt.log gpurun_out/pytest_gpu.log
cat gpurun_out/cmp_bt.jsonl gpurun_out/bench_c2.json
