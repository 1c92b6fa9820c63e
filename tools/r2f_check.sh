set -u
OUT=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_replay.py tests/test_gpu_boundary.py -q -x > $OUT/r2f_pytest.log 2>&1
echo pytest=$?; tail -3 $OUT/r2f_pytest.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32" > $OUT/r2f_pytest_fp32.log 2>&1
echo pytest_fp32=$?; tail -3 $OUT/r2f_pytest_fp32.log
timeout 1800 python bench.py --steps 2 --warmup 3 > $OUT/r2f_bench.json 2> $OUT/r2f_bench.err
echo bench=$?; grep -E "Elapsed|Maximum resident" $OUT/r2f_bench.err
