set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/r2s_gpu_tests.log 2>&1
echo pytest=$?; tail -3 $OUT/r2s_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r2s_smoke.log 2>&1
echo smoke=$?; tail -4 $OUT/r2s_smoke.log
( time bash tools/profile_bench.sh r2s ) > $OUT/r2s_profile_bench.log 2>&1
echo profile_bench=$?; tail -5 $OUT/r2s_profile_bench.log
( time python bench.py --impl reference --steps 2 --warmup 1 ) > $OUT/r2s_reference_arm.json 2> $OUT/r2s_reference_arm.err
echo ref=$?; tail -c 600 $OUT/r2s_reference_arm.json
BENCH_ALLOW_SHORT=1 timeout 900 python bench.py --workload C3 --precision f32 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/r2s_bench_C3_f32.json 2> $OUT/r2s_bench_C3_f32.err
echo c3f32=$?
ls -la $OUT | tail -25
