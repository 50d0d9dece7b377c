python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/t_build.log 2>&1
CGL_FULLRUN_LOG=gpurun_out/t_fullruns.jsonl timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/t_bench.log 2>&1; echo "rc=$?" >> gpurun_out/t_bench.log
tail -n 3 gpurun_out/t_pytest.log; cut -c1-300 gpurun_out/t_bench.log
