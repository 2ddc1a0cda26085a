#!/bin/bash
# A/B of the compaction write kernel: default (shuffle loop, direct global stores)
# vs libgk_cp1.so (GK_COMPACT_STAGED=1: ffs expansion into shared memory, coalesced
# copy-out).  Parity tests on the variant first, then bench lines of C2/C3/C4.
set -u
mkdir -p gpurun_out
GK_LIB=$PWD/paper_2103_14978_b200/libgk_cp1.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_cp1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cp1.log
tail -n 3 gpurun_out/pytest_cp1.log
for rep in 1 2; do
for lib in libgk libgk_cp1; do
  for c in c2 c3 c4; do
    GK_LIB=$PWD/paper_2103_14978_b200/$lib.so timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-alt 2>/dev/null | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$lib','cfg':'$c','value':d['value'],'ms':d['ms_per_step'],'kern':[(k['kernel'],k['frac'],k['share_of_step']) for k in d['roofline']['all_kernels']]}))" >> gpurun_out/compactab.jsonl
  done
done
done
cat gpurun_out/compactab.jsonl
