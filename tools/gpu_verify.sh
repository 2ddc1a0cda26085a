#!/bin/bash
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "edit_distance or accuracy or compact_rows" > gpurun_out/pytest_ver.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ver.log
tail -n 3 gpurun_out/pytest_ver.log
timeout 600 python bench.py --no-e2e > gpurun_out/bench_c2_ver.json 2> gpurun_out/bench_c2_ver.err
tail -n 3 gpurun_out/bench_c2_ver.err
python -c "import json; d=json.loads(open('gpurun_out/bench_c2_ver.json').read().strip().splitlines()[-1]); print(d['value'], json.dumps(d['accuracy']))"
