set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r2q}
rm -f $OUT/${TAG}_plain.log
run() { python tools/prof_case.py "$@" reps=2 >> $OUT/${TAG}_plain.log 2>&1; }
for c in "C3 rbp 4736 imax=1" "C3 cirbp 4736 imax=1" "C3 me_cirbp 4736 imax=1 n_p=64" "C1 me_cirbp 100000 n_p=4" "C1 rbp 100000" "C1 cirbp 100000" "C1 lmdrbp 100000" "C1 slmdrbp 100000" "C1 lmd_cirbp 100000" "C1 me_rbp 100000 n_p=4" "C2 cirbp 20000" "C2 rbp 20000" "C2 me_cirbp 20000 n_p=16" \
         "C3 rbp 4736 imax=1 f32" "C3 cirbp 4736 imax=1 f32" "C3 me_cirbp 4736 imax=1 n_p=64 f32" "C1 me_cirbp 100000 n_p=4 f32"; do run $c; done
cut -c1-150 $OUT/${TAG}_plain.log
timeout 900 python -m pytest tests/test_gpu_replay.py tests/test_gpu_boundary.py tests/test_gpu_trace.py -q -x > $OUT/${TAG}_pytest2.log 2>&1
echo pytest2=$?; tail -3 $OUT/${TAG}_pytest2.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or c0_batch or c1_batch or c2_batch or me_selection or placements or fp32 or small_batches or minsum" > $OUT/${TAG}_pytest1.log 2>&1
echo pytest1=$?; tail -3 $OUT/${TAG}_pytest1.log
