python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/u_build.log 2>&1
timeout 900 python -m pytest tests/test_rk_banded.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/u_pytest.log
tail -n 30 gpurun_out/u_pytest.log
timeout 300 python tools/prof_step.py rk4 400 C1
