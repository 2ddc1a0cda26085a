set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"filter_bt" -c 1 \
    -o gpurun_out/prof_bt python tools/cmp_filters.py --L 250 --n 4000000 --e 12 --flags 4 --reps 1 > gpurun_out/ncu_bt.log 2>&1
tail -2 gpurun_out/ncu_bt.log
