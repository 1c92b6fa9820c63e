set -u
OUT=gpurun_out
timeout 600 python tools/dyn_sweep.py C3 rbp 4096 f64 auto,hbm,trees,split 0 > $OUT/r2c_sweep.jsonl 2> $OUT/r2c_sweep.err
echo sweep=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -o $OUT/r2c_c3_rbp python tools/prof_case.py C3 rbp 1184 imax=1 > $OUT/r2c_ncu_rbp.log 2>&1
echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dyn_decode -s 1 -c 1 -o $OUT/r2c_c3_cirbp python tools/prof_case.py C3 cirbp 1184 imax=1 > $OUT/r2c_ncu_cirbp.log 2>&1
echo ncu2=$?
