set -u
OUT=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_multirank.py -q -x > $OUT/r2i_pytest.log 2>&1
echo pytest=$?; tail -3 $OUT/r2i_pytest.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "golden or me_selection or c1_batch or c2_batch" > $OUT/r2i_pytest2.log 2>&1
echo pytest2=$?; tail -3 $OUT/r2i_pytest2.log
BENCH_ALLOW_SHORT=1 timeout 300 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-secondary > $OUT/r2i_bench_C1.json 2> $OUT/r2i_bench.err
echo bench=$?
timeout 900 python tools/dyn_sweep.py C3 me_cirbp/64 4096 f64 auto 0 > $OUT/r2i_sweep.jsonl 2> $OUT/r2i_sweep.err
echo sweep=$?; cat $OUT/r2i_sweep.jsonl
