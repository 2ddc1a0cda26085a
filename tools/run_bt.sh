set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "sweep or random_lengths or adversarial or ragged or original" > gpurun_out/pytest_bt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_bt.log
tail -3 gpurun_out/pytest_bt.log
timeout 600 python tools/cmp_filters.py --L 100 --e 5 10 --flags 0 4 > gpurun_out/cmp_bt.jsonl 2>&1
timeout 600 python tools/cmp_filters.py --L 150 --e 12 15 --flags 0 4 >> gpurun_out/cmp_bt.jsonl 2>&1
timeout 600 python tools/cmp_filters.py --L 250 --e 12 18 25 --flags 0 4 >> gpurun_out/cmp_bt.jsonl 2>&1
cat gpurun_out/cmp_bt.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"filter_bt" -c 1 \
    -o gpurun_out/prof_bt python tools/cmp_filters.py --L 250 --n 4000000 --e 12 --flags 4 --reps 1 > gpurun_out/ncu_bt.log 2>&1
