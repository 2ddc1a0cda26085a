#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "sweep" > gpurun_out/pytest_sw2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sw2.log
tail -n 3 gpurun_out/pytest_sw2.log
timeout 600 python tools/cmp_sweep.py --L 100 --emax 10 > gpurun_out/cmp_sw2.jsonl 2>&1
timeout 600 python tools/cmp_sweep.py --L 150 --emax 15 >> gpurun_out/cmp_sw2.jsonl 2>&1
timeout 600 python tools/cmp_sweep.py --L 250 --emax 25 >> gpurun_out/cmp_sw2.jsonl 2>&1
cat gpurun_out/cmp_sw2.jsonl
