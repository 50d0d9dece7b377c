python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/x_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_experiments.py -m gpu -x -q > gpurun_out/x_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/x_pytest.log
tail -n 25 gpurun_out/x_pytest.log
