#!/bin/bash
# A/B timing of every libgk*.so in the package dir with tools/time_filters2.py.
#   gpurun -- bash tools/ab_run.sh TAG [time_filters2 args...]
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for lib in paper_2103_14978_b200/libgk*.so; do
  GK_LIB=$PWD/$lib timeout 600 python tools/time_filters2.py --tag $(basename $lib) "$@" >> $OUT/times.jsonl 2>> $OUT/err.log
done
cat $OUT/times.jsonl; tail -3 $OUT/err.log
