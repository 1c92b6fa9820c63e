set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r2n}
rm -f $OUT/${TAG}_plain.log
run() { python tools/prof_case.py "$@" reps=2 >> $OUT/${TAG}_plain.log 2>&1; }
for c in "C3 rbp 4736 imax=1" "C3 cirbp 4736 imax=1" "C3 me_cirbp 4736 imax=1 n_p=64" "C1 me_cirbp 100000 n_p=4" "C1 rbp 100000" "C1 cirbp 100000" "C1 lmdrbp 100000" "C1 slmdrbp 100000" "C1 lmd_cirbp 100000" "C1 me_rbp 100000 n_p=4" "C2 cirbp 20000" "C2 rbp 20000" "C2 me_cirbp 20000 n_p=16" \
         "C3 rbp 4736 imax=1 f32" "C3 cirbp 4736 imax=1 f32" "C3 me_cirbp 4736 imax=1 n_p=64 f32" "C1 me_cirbp 100000 n_p=4 f32" "C1 rbp 100000 f32" "C2 cirbp 20000 f32"; do run $c; done
for v in rb4 rb5; do
  echo "-- $v" >> $OUT/${TAG}_plain.log
  export LDPC_B200_LIB=$PWD/paper_2102_11089_b200/lib/exp/libldpc_b200_$v.so
  for c in "C1 rbp 100000" "C1 lmdrbp 100000" "C1 slmdrbp 100000" "C2 rbp 20000"; do run $c; done
done
unset LDPC_B200_LIB
cut -c1-150 $OUT/${TAG}_plain.log
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum"
i=0
for c in "C3 rbp 4736 imax=1" "C3 cirbp 4736 imax=1" "C3 me_cirbp 4736 imax=1 n_p=64" "C1 me_cirbp 100000 n_p=4" "C1 rbp 100000" "C3 rbp 4736 imax=1 f32"; do
  i=$((i+1))
  timeout 600 ncu $M --clock-control none -k regex:dyn_decode -s 1 -c 1 --csv --log-file $OUT/${TAG}_traffic_$i.csv python tools/prof_case.py $c > $OUT/${TAG}_traffic_$i.log 2>&1
  echo "traffic $i ($c) rc=$?"; grep -E "dram__bytes|gpu__time|inst_executed|sector" $OUT/${TAG}_traffic_$i.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_boundary.py tests/test_gpu_trace.py -q -x > $OUT/${TAG}_pytest2.log 2>&1
echo pytest2=$?; tail -3 $OUT/${TAG}_pytest2.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or c0_batch or c1_batch or c2_batch or me_selection or placements or fp32 or small_batches or minsum" > $OUT/${TAG}_pytest1.log 2>&1
echo pytest1=$?; tail -3 $OUT/${TAG}_pytest1.log
