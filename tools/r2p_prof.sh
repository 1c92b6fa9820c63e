set -u
OUT=gpurun_out
mkdir -p $OUT
SECS="--section LaunchStats --section Occupancy --section WarpStateStats --section SourceCounters --section SchedulerStats --section InstructionStats --section MemoryWorkloadAnalysis"
export LDPC_B200_LIB=$PWD/paper_2102_11089_b200/lib/exp/libldpc_b200_64fd904.so
timeout 600 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -f -o $OUT/r2p_lmd_old python tools/prof_case.py C1 lmdrbp 20000 > $OUT/r2p_ncu1.log 2>&1
echo ncu1=$?
unset LDPC_B200_LIB
timeout 600 ncu $SECS --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -f -o $OUT/r2p_lmd_new python tools/prof_case.py C1 lmdrbp 20000 > $OUT/r2p_ncu2.log 2>&1
echo ncu2=$?
