set -u
OUT=gpurun_out/l2d; mkdir -p $OUT
for lib in libgk.so libgk_sp4.so; do
  GK_LIB=$PWD/paper_2103_14978_b200/$lib timeout 300 python tools/time_l2.py --tag $lib --buckets 0,1 >> $OUT/times.jsonl 2>> $OUT/err.log
done
cat $OUT/times.jsonl
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_l2 -c 1 -o $OUT/ncu_l2_100 python tools/time_l2.py --buckets 0 --reps 1 > $OUT/ncu.log 2>&1; echo ncu rc=$?
python tools/ncu_summary.py $OUT/ncu_l2_100.ncu-rep > $OUT/ncu_l2_100.txt 2>&1
python tools/ncu_sass_mix.py $OUT/ncu_l2_100.ncu-rep >> $OUT/ncu_l2_100.txt 2>&1
head -3 $OUT/ncu_l2_100.txt; tail -1 $OUT/ncu_l2_100.txt
