set -u
OUT=gpurun_out
mkdir -p $OUT
rm -f $OUT/r2o_bisect.log
run() { python tools/prof_case.py "$@" reps=3 >> $OUT/r2o_bisect.log 2>&1; }
for v in 64fd904 28841ed b998b6a; do
  echo "-- $v" >> $OUT/r2o_bisect.log
  export LDPC_B200_LIB=$PWD/paper_2102_11089_b200/lib/exp/libldpc_b200_$v.so
  for c in "C1 lmdrbp 100000" "C1 slmdrbp 100000" "C1 rbp 100000"; do run $c; done
done
unset LDPC_B200_LIB
echo "-- current" >> $OUT/r2o_bisect.log
for c in "C1 lmdrbp 100000" "C1 slmdrbp 100000" "C1 rbp 100000"; do run $c; done
cut -c1-150 $OUT/r2o_bisect.log
