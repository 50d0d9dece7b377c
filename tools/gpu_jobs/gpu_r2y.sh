timeout 900 python -m pytest tests/test_rk_banded.py -m gpu -x -q > gpurun_out/y_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/y_pytest.log
tail -n 25 gpurun_out/y_pytest.log
