#!/bin/bash
# A/B of the 256/512-byte staging encoder's launch bound (GK_ENC_MINB_WIDE):
# default 1 (244 registers, 2 CTAs/SM) vs libgk_ew3.so (3: 168 registers, 3 CTAs/SM).
# Encode parity tests on the variant, encoder times at 150/250 bp, bench C3/C4.
set -u
mkdir -p gpurun_out
GK_LIB=$PWD/paper_2103_14978_b200/libgk_ew3.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ew3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ew3.log
tail -n 2 gpurun_out/pytest_ew3.log
for rep in 1 2; do
for lib in libgk libgk_ew3; do
  GK_LIB=$PWD/paper_2103_14978_b200/$lib.so timeout 300 python tools/time_enc.py --L 150 250 | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/encwide.jsonl
  for c in c3 c4; do
    GK_LIB=$PWD/paper_2103_14978_b200/$lib.so timeout 300 python bench.py --config $c --no-e2e --no-cpu-baseline --no-alt 2>/dev/null | tail -1 \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$lib','cfg':'$c','value':d['value'],'ms':d['ms_per_step']}))" >> gpurun_out/encwide.jsonl
  done
done
done
cat gpurun_out/encwide.jsonl
