set -u
OUT=gpurun_out
mkdir -p $OUT
SECS="--section LaunchStats --section Occupancy --section WarpStateStats --section SourceCounters --section MemoryWorkloadAnalysis --section SchedulerStats --section SpeedOfLight --section InstructionStats"
python tools/prof_case.py C3 rbp 4736 imax=1 > $OUT/r2k_plain.log 2>&1
python tools/prof_case.py C3 cirbp 4736 imax=1 >> $OUT/r2k_plain.log 2>&1
python tools/prof_case.py C3 me_cirbp 4736 imax=1 n_p=64 >> $OUT/r2k_plain.log 2>&1
python tools/prof_case.py C1 me_cirbp 100000 n_p=4 >> $OUT/r2k_plain.log 2>&1
python tools/prof_case.py C1 rbp 100000 >> $OUT/r2k_plain.log 2>&1
python tools/prof_case.py C2 cirbp 20000 >> $OUT/r2k_plain.log 2>&1
cat $OUT/r2k_plain.log
timeout 900 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -f -o $OUT/r2k_c3_rbp python tools/prof_case.py C3 rbp 4736 imax=1 > $OUT/r2k_ncu1.log 2>&1
echo ncu1=$?
timeout 900 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -f -o $OUT/r2k_c3_cirbp python tools/prof_case.py C3 cirbp 4736 imax=1 > $OUT/r2k_ncu2.log 2>&1
echo ncu2=$?
timeout 900 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -f -o $OUT/r2k_c1_mecirbp python tools/prof_case.py C1 me_cirbp 100000 n_p=4 > $OUT/r2k_ncu3.log 2>&1
echo ncu3=$?
ls -la $OUT
