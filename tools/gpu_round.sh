#!/bin/bash
# One GPU round: parity tests, the default bench line, the ncu launch list of the
# bench command and a full ncu capture of the top kernels.  Outputs in gpurun_out/.
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
python bench.py --path fused --no-e2e --no-cpu-baseline > gpurun_out/bench_fused_${TAG}.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"encode_tma|filter_sp_kernel|compact_write|filter_ascii_tma" -s 2 -c 6 \
    -o gpurun_out/prof_${TAG} python tools/prof_run.py --n 4000000 --L 100 --e 2 10 --reps 2 > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/pytest_gpu_${TAG}.log
