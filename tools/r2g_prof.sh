set -u
OUT=gpurun_out
SECS="--section LaunchStats --section Occupancy --section WarpStateStats --section SourceCounters --section MemoryWorkloadAnalysis --section SchedulerStats --section SpeedOfLight"
timeout 900 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -o $OUT/r2g_c1_cirbp python tools/prof_case.py C1 cirbp 100000 > $OUT/r2g_ncu1.log 2>&1
echo ncu1=$?
timeout 900 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -o $OUT/r2g_c1_mecirbp python tools/prof_case.py C1 me_cirbp 100000 n_p=4 > $OUT/r2g_ncu2.log 2>&1
echo ncu2=$?
timeout 1200 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -o $OUT/r2g_c3_cirbp_hbm python tools/prof_case.py C3 cirbp 1184 imax=1 > $OUT/r2g_ncu3.log 2>&1
echo ncu3=$?
timeout 900 python tools/grid.py c1 --out $OUT/r2g_grid_c1.jsonl > $OUT/r2g_grid.log 2>&1
echo grid_c1=$?
timeout 600 python tools/grid.py c0 --out $OUT/r2g_grid_c0.jsonl >> $OUT/r2g_grid.log 2>&1
echo grid_c0=$?
