#!/bin/bash
# One gpurun session: build, then the named steps; outputs land in gpurun_out/<tag>/.
#   gpurun --timeout 1800 -- bash tools/gpu.sh TAG test bench c2 peak ncu ...
# steps: test (pytest -m gpu), smoke, peak (INT microbenchmark), bench (default c5),
#        c2|c3|c4 (bench --config), parity (tools/full_parity.py), launches (ncu launch list
#        of the default bench), ncu:<kernel-regex> (ncu --set full of one launch)
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { cat $OUT/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
for step in "$@"; do
  case $step in
    test) timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/test.log 2>&1; echo "test rc=$?"; tail -3 $OUT/test.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log ;;
    peak) timeout 120 python -c "import bench, json; print(json.dumps(bench.int_peak()))" > $OUT/int_peak.json 2>&1; cat $OUT/int_peak.json ;;
    bench) timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_c5.json 2> $OUT/bench_c5.err; echo "bench rc=$?"; tail -c 600 $OUT/bench_c5.json ;;
    c2|c3|c4) timeout 900 python bench.py --config $step --steps 10 --warmup 3 > $OUT/bench_$step.json 2> $OUT/bench_$step.err; echo "$step rc=$?"; tail -c 300 $OUT/bench_$step.json ;;
    parity) timeout 1500 python tools/full_parity.py --tag ${TAG} > $OUT/parity.log 2>&1; echo "parity rc=$?"; tail -5 $OUT/parity.log; cp profiles/${TAG}_full_parity.json $OUT/ 2>/dev/null ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/launches.log 2>&1; echo "launches rc=$?" ;;
    launches:*) cfg=${step#launches:}; timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/launches_$cfg.log 2>&1; echo "launches $cfg rc=$?" ;;
    ncu:*) spec=${step#ncu:}; k=${spec%%@*}; cfg=${spec#*@}; [ "$cfg" = "$spec" ] && cfg=c5
      timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 -o $OUT/ncu_${k//[^a-zA-Z0-9_]/}_$cfg python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_$cfg.log 2>&1; echo "ncu $k $cfg rc=$?" ;;
    *) echo "unknown step $step" ;;
  esac
done
