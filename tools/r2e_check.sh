set -u
OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity.py::test_c3_batch_vs_oracle > $OUT/r2e_pytest.log 2>&1
echo pytest=$?
tail -3 $OUT/r2e_pytest.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "c3_batch" > $OUT/r2e_pytest_c3.log 2>&1
echo pytest_c3=$?
tail -3 $OUT/r2e_pytest_c3.log
