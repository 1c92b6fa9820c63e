set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r2l}
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or c0_batch or c1_batch or me_selection or placements or fp32_messages or small_batches" > $OUT/${TAG}_pytest1.log 2>&1
echo pytest1=$?; tail -3 $OUT/${TAG}_pytest1.log
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_boundary.py tests/test_gpu_trace.py -q -x > $OUT/${TAG}_pytest2.log 2>&1
echo pytest2=$?; tail -3 $OUT/${TAG}_pytest2.log
for c in "C3 rbp 4736 imax=1" "C3 cirbp 4736 imax=1" "C3 me_cirbp 4736 imax=1 n_p=64" "C1 me_cirbp 100000 n_p=4" "C1 rbp 100000" "C1 cirbp 100000" "C1 lmdrbp 100000" "C2 cirbp 20000" "C2 rbp 20000" "C2 me_cirbp 20000 n_p=16"; do
  python tools/prof_case.py $c reps=2 >> $OUT/${TAG}_plain.log 2>&1
done
cat $OUT/${TAG}_plain.log
SECS="--section LaunchStats --section Occupancy --section WarpStateStats --section SourceCounters --section MemoryWorkloadAnalysis --section SchedulerStats --section InstructionStats --section SpeedOfLight"
timeout 600 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -f -o $OUT/${TAG}_c1_mecirbp python tools/prof_case.py C1 me_cirbp 20000 n_p=4 > $OUT/${TAG}_ncu1.log 2>&1
echo ncu1=$?
timeout 900 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -f -o $OUT/${TAG}_c3_cirbp python tools/prof_case.py C3 cirbp 1184 imax=1 res=1184 > $OUT/${TAG}_ncu2.log 2>&1
echo ncu2=$?
timeout 900 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -f -o $OUT/${TAG}_c3_rbp python tools/prof_case.py C3 rbp 1184 imax=1 res=1184 > $OUT/${TAG}_ncu3.log 2>&1
echo ncu3=$?
ls -la $OUT | tail -20
