set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -q -x -k "me_ or golden or c3_batch or select or gamma" > $OUT/r2x_pytest.log 2>&1
echo pytest=$?; tail -3 $OUT/r2x_pytest.log
python tools/prof_case.py C1 me_cirbp 100000 n_p=4 reps=3; python tools/prof_case.py C1 me_rbp 100000 n_p=4 reps=3; python tools/prof_case.py C2 me_cirbp 20000 n_p=16 reps=2
python -c "import __graft_entry__ as g; g.smoke()"
