set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -x -k "me_ or golden or c3_batch or select" > $OUT/r2u_pytest.log 2>&1
echo pytest=$?; tail -3 $OUT/r2u_pytest.log
BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --workload C3 --only me_cirbp/M64 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/r2u_bench_C3_me.json 2> $OUT/r2u_bench_C3_me.err
echo bench=$?; python -c "
import json; d=json.load(open('$OUT/r2u_bench_C3_me.json'))
for k,v in d['per_schedule'].items(): print(k, v['ms'], '%.3e'%v['edge_updates_per_s'], v['frames_per_s'])"
BENCH_ALLOW_SHORT=1 timeout 600 python bench.py --workload C3 --only rbp --steps 1 --warmup 1 --no-cpu-baseline > $OUT/r2u_bench_C3_rbp.json 2> $OUT/r2u_bench_C3_rbp.err
python -c "
import json; d=json.load(open('$OUT/r2u_bench_C3_rbp.json'))
for k,v in d['per_schedule'].items(): print(k, v['ms'], '%.3e'%v['edge_updates_per_s'], v['frames_per_s'])"
python tools/prof_case.py C1 me_cirbp 100000 n_p=4 reps=2; python tools/prof_case.py C2 me_cirbp 20000 n_p=16 reps=2; python tools/prof_case.py C3 me_cirbp 4736 imax=1 n_p=64 reps=2
