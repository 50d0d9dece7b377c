python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/w_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/w_pytest.log
tail -n 4 gpurun_out/w_pytest.log
timeout 300 python tools/prof_step.py strang 200 C0
timeout 300 python tools/prof_step.py if4 200 C0
timeout 300 python tools/rk_time.py
timeout 900 python tools/project_sharded.py 4 2>&1 | tail -2
