#!/bin/bash
# A/B of the sweep kernel's minimum-CTAs-per-SM launch bound (GK_SWEEP_MINB):
# default (6: 158 regs) vs libgk_bt4.so (200 regs, 8 warps/SM) / libgk_bt5.so (162 regs, 10 warps/SM);
# and the encoder variant libgk_mb5.so; bench lines of C2/C3/C4 (device-timed step).
set -u
mkdir -p gpurun_out
for rep in 1 2; do
for lib in libgk libgk_bt4 libgk_bt5; do
  for c in c2 c3 c4; do
    GK_LIB=$PWD/paper_2103_14978_b200/$lib.so timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-alt 2>/dev/null | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$lib','cfg':'$c','value':d['value'],'ms':d['ms_per_step'],'kern':[(k['kernel'],k.get('mean_launch_ms'),k['frac']) for k in d['roofline']['all_kernels']]}))" >> gpurun_out/sweepab2.jsonl
  done
done
done
cat gpurun_out/sweepab2.jsonl
