#!/bin/bash
# A/B timing of filter kernels: every libgk*.so in the package dir through tools/time_filters.py
set -u
OUT=gpurun_out/${1:-ab}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for lib in paper_2103_14978_b200/libgk*.so; do
  GK_LIB=$PWD/$lib timeout 600 python tools/time_filters.py --tag $(basename $lib) >> $OUT/times.jsonl 2>> $OUT/err.log
done
cat $OUT/times.jsonl
