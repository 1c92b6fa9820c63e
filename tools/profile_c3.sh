#!/bin/bash
# BG1 (C3) fixed-schedule evidence: bench lines (f32, f64), launch list, full
# captures of the check-phase and VN-phase kernels.
# Usage (GPU box): bash tools/profile_c3.sh TAG
set -u
TAG=$1
OUT=gpurun_out
python bench.py --workload C3F --precision f32 --no-cpu-baseline > $OUT/bench_C3F_f32_$TAG.json 2> $OUT/c3f32.err
python bench.py --workload C3F --precision f64 --no-cpu-baseline > $OUT/bench_C3F_f64_$TAG.json 2> $OUT/c3f64.err
export BENCH_ALLOW_SHORT=1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c3f_$TAG.csv \
    python bench.py --workload C3F --precision f32 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/c3f_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:phase_check_tma -s 5 -c 1 \
    -o $OUT/prof_c3f_check_$TAG python bench.py --workload C3F --precision f32 --only flooding --steps 1 --warmup 1 \
    --no-cpu-baseline > $OUT/c3f_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:phase_vn_tma -s 2 -c 1 \
    -o $OUT/prof_c3f_vn_$TAG python bench.py --workload C3F --precision f32 --only flooding --steps 1 --warmup 1 \
    --no-cpu-baseline > $OUT/c3f_ncu_vn.log 2>&1
tail -n 1 $OUT/c3f_ncu_full.log; tail -n 1 $OUT/c3f_ncu_vn.log
