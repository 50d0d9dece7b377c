timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/d3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/d3_pytest.log
tail -n 4 gpurun_out/d3_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/d3_bench.log 2>&1; echo "rc=$?" >> gpurun_out/d3_bench.log
cut -c1-330 gpurun_out/d3_bench.log
