set -u
OUT=gpurun_out
mkdir -p $OUT
( time python bench.py ) > $OUT/r2v_bench.json 2> $OUT/r2v_bench.err
echo bench=$?; tail -3 $OUT/r2v_bench.err
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/r2v_gpu_tests.log 2>&1
echo pytest=$?; tail -3 $OUT/r2v_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2v_smoke.log 2>&1
echo smoke=$?
M="--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_sector_hit_rate.pct"
i=0
for c in "C3 rbp 4736 imax=1" "C3 cirbp 4736 imax=1" "C3 me_cirbp 4736 imax=1 n_p=64"; do
  i=$((i+1))
  timeout 600 ncu $M --clock-control none -k regex:dyn_decode -s 1 -c 1 --csv --log-file $OUT/r2v_traffic_$i.csv python tools/prof_case.py $c > $OUT/r2v_traffic_$i.log 2>&1
  echo "traffic $i ($c) rc=$?"; grep -E "dram__bytes|gpu__time|inst_executed|hit_rate" $OUT/r2v_traffic_$i.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
