timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/p3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p3_pytest.log
tail -n 5 gpurun_out/p3_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/p3_bench.log 2>&1; cut -c1-260 gpurun_out/p3_bench.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/p3_probe.log 2>&1; grep -v "^{" gpurun_out/p3_probe.log
timeout 300 python tools/project_sharded_fourier.py 1 8 2>&1 | tail -3
