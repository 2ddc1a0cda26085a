#!/bin/bash
# Full GPU pass on the current tree: parity suite, bench lines (C2 default = sweep,
# C3, C4, C5), the ncu launch list of the default bench command and ncu --set full
# captures of the dominant kernels at the bench launch configuration.
set -u
TAG=${1:-r01f}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
tail -n 2 gpurun_out/smoke_${TAG}.log
tail -n 2 gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err
timeout 600 python bench.py --config c3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_${TAG}.json 2> gpurun_out/bench_c3_${TAG}.err
timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_${TAG}.json 2> gpurun_out/bench_c4_${TAG}.err
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5_${TAG}.json 2> gpurun_out/bench_c5_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"filter_bt_sweep|encode_tma|compact" -c 5 \
    -o gpurun_out/prof_bench_${TAG} python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-alt > gpurun_out/ncu_bench_${TAG}.log 2>&1
tail -n 2 gpurun_out/ncu_bench_${TAG}.log
head -c 700 gpurun_out/bench_c2_${TAG}.json
