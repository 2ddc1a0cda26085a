#!/bin/bash
# Evidence for profiles/: full-size parity record, bench lines (c5 default, c2-c4), ncu
# launch lists of the default and c2 benches, and one ncu --set full capture per hot
# kernel (summarised on the box; only the listed .ncu-rep files come back).
#   gpurun --timeout 3600 -- bash tools/gpu_evidence.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
python -c "import bench, json; print(json.dumps(bench.int_peak()))" > $OUT/int_peak.json 2>&1
timeout 900 python tools/full_parity.py --tag $TAG > $OUT/parity.log 2>&1; echo "parity rc=$?"; tail -1 $OUT/parity.log
cp profiles/${TAG}_full_parity.json $OUT/ 2>/dev/null
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench c5 rc=$?"
for c in c2 c3 c4; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/launches_c5.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/launches_c2.log 2>&1; echo "launches c2 rc=$?"
KEEP="encode3_c5 filter_bt2_sweep_c4"
for spec in "encode3@c5" "filter_sp@c5" "filter_sp2@c5" "compact_write@c5" "filter_bt2_sweep@c2" "filter_bt2_sweep@c3" "filter_bt2_sweep@c4" "encode3@c2" "encode3@c4"; do
  k=${spec%%@*}; cfg=${spec#*@}; name=ncu_${k}_$cfg
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 -o $OUT/$name python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/$name.log 2>&1; echo "ncu $k $cfg rc=$?"
  python tools/ncu_summary.py $OUT/$name.ncu-rep > $OUT/$name.summary.txt 2>&1
  python tools/ncu_sass_mix.py $OUT/$name.ncu-rep >> $OUT/$name.summary.txt 2>&1
  python tools/ncu_traffic.py $OUT/$name.ncu-rep --workload $cfg:auto > $OUT/$name.traffic.json 2>&1
  case " $KEEP " in *" ${k}_$cfg "*) ;; *) rm -f $OUT/$name.ncu-rep ;; esac
done
du -sh $OUT
