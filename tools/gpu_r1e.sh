#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "sweep or host" > gpurun_out/pytest_e.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_e.log
tail -n 3 gpurun_out/pytest_e.log
timeout 600 python bench.py > gpurun_out/bench_c2_sweep.json 2> gpurun_out/bench_c2_sweep.err
timeout 600 python bench.py --config c3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_sweep.json 2> gpurun_out/bench_c3_sweep.err
timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_sweep.json 2> gpurun_out/bench_c4_sweep.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"filter_bt|filter_sp" -c 3 \
    -o gpurun_out/prof_sweep python tools/prof_sweep.py --n 4000000 --L 100 --emax 10 > gpurun_out/ncu_sweep.log 2>&1
tail -n 2 gpurun_out/ncu_sweep.log
cat gpurun_out/bench_c2_sweep.json | head -c 1500; echo; tail -n 3 gpurun_out/bench_c2_sweep.err
