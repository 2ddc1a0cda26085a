#!/bin/bash
# Re-confirm a restored tree on the GPU: parity tests, C2/C3/C4 bench lines, the
# launch list of the default bench and a full ncu capture of the filter kernels
# (small e, e=10, and the large-e warp-pair kernel at 250 bp).  Outputs in gpurun_out/.
set -u
TAG=${1:-r01c}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_c2_${TAG}.json 2> gpurun_out/bench_c2_${TAG}.err
timeout 600 python bench.py --config c3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c3_${TAG}.json 2> gpurun_out/bench_c3_${TAG}.err
timeout 600 python bench.py --config c4 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4_${TAG}.json 2> gpurun_out/bench_c4_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_tma|filter_sp_kernel|filter_spq" -s 2 -c 6 \
    -o gpurun_out/prof_${TAG} python tools/prof_run.py --n 4000000 --L 100 --e 2 10 --reps 2 > gpurun_out/ncu_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"filter_spq" -c 2 \
    -o gpurun_out/prof_q_${TAG} python tools/prof_run.py --n 2000000 --L 250 --e 12 25 --reps 1 > gpurun_out/ncu_q_${TAG}.log 2>&1
tail -3 gpurun_out/pytest_gpu_${TAG}.log
