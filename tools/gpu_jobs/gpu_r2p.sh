python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/p_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/p_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p_pytest.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/p_probe.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/p_bench.log 2>&1; echo "rc=$?" >> gpurun_out/p_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/p_ref.log 2>&1; echo "rc=$?" >> gpurun_out/p_ref.log
tail -n 3 gpurun_out/p_pytest.log; head -14 gpurun_out/p_probe.log; cut -c1-600 gpurun_out/p_bench.log; cut -c1-600 gpurun_out/p_ref.log
