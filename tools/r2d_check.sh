set -u
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -x -q -k "c0_batch or c1_batch or placements or small_batches or selection or boundary or two_streams or lane or select_vns or variant" > $OUT/r2d_pytest.log 2>&1
echo pytest=$?
tail -3 $OUT/r2d_pytest.log
timeout 900 python tools/dyn_sweep.py C3 rbp,cirbp,me_cirbp/64 4096 f64 auto 0 > $OUT/r2d_sweep.jsonl 2> $OUT/r2d_sweep.err
echo sweep=$?
cat $OUT/r2d_sweep.jsonl
SECS="--section LaunchStats --section Occupancy --section WarpStateStats --section SourceCounters --section MemoryWorkloadAnalysis --section SchedulerStats --section SpeedOfLight"
timeout 900 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -o $OUT/r2d_c3_rbp python tools/prof_case.py C3 rbp 148 imax=1 > $OUT/r2d_ncu_rbp.log 2>&1
echo ncu1=$?
tail -2 $OUT/r2d_ncu_rbp.log
