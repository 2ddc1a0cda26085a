#!/bin/bash
# A/B of the TMA encoder's minimum-CTAs-per-SM launch bound (GK_ENC_MINB): the
# default library vs variant builds libgk_mb5.so / libgk_mb6.so.
set -u
mkdir -p gpurun_out
for lib in libgk libgk_mb5 libgk_mb6; do
  for rep in 1 2; do
    GK_LIB=$PWD/paper_2103_14978_b200/$lib.so timeout 300 python tools/time_enc.py --L 100 150 250 \
      | sed "s/^{/{\"lib\": \"$lib\", /" >> gpurun_out/encab.jsonl
  done
done
cat gpurun_out/encab.jsonl
