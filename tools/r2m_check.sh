set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r2m}
./tools/micro/randbw > $OUT/${TAG}_randbw.json 2>&1
echo randbw=$?; cat $OUT/${TAG}_randbw.json
rm -f $OUT/${TAG}_plain.log
run() { python tools/prof_case.py "$@" reps=2 >> $OUT/${TAG}_plain.log 2>&1; }
for c in "C3 rbp 4736 imax=1" "C3 cirbp 4736 imax=1" "C3 me_cirbp 4736 imax=1 n_p=64" "C1 me_cirbp 100000 n_p=4" "C1 rbp 100000" "C1 cirbp 100000" "C1 lmdrbp 100000" "C1 lmd_cirbp 100000" "C2 cirbp 20000" "C2 rbp 20000" "C2 me_cirbp 20000 n_p=16"; do run $c; done
for v in rb4 rb5; do
  echo "-- $v" >> $OUT/${TAG}_plain.log
  export LDPC_B200_LIB=$PWD/paper_2102_11089_b200/lib/exp/libldpc_b200_$v.so
  for c in "C3 rbp 4736 imax=1" "C1 rbp 100000" "C1 lmdrbp 100000" "C2 rbp 20000"; do run $c; done
done
echo "-- ci3" >> $OUT/${TAG}_plain.log
export LDPC_B200_LIB=$PWD/paper_2102_11089_b200/lib/exp/libldpc_b200_ci3.so
for c in "C3 cirbp 4736 imax=1" "C3 me_cirbp 4736 imax=1 n_p=64" "C1 me_cirbp 100000 n_p=4" "C1 cirbp 100000" "C1 lmd_cirbp 100000" "C2 cirbp 20000"; do run $c; done
unset LDPC_B200_LIB
cut -c1-150 $OUT/${TAG}_plain.log
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_boundary.py tests/test_gpu_trace.py -q -x > $OUT/${TAG}_pytest2.log 2>&1
echo pytest2=$?; tail -3 $OUT/${TAG}_pytest2.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or c0_batch or c1_batch or me_selection or placements or fp32_messages or small_batches" > $OUT/${TAG}_pytest1.log 2>&1
echo pytest1=$?; tail -3 $OUT/${TAG}_pytest1.log
