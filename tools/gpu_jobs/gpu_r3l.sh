timeout 1500 python -m pytest tests/test_fftpass.py tests/test_full_runs.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/l3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/l3_pytest.log
tail -n 15 gpurun_out/l3_pytest.log
timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "STR_" | grep -v "^{"
timeout 300 python tools/prof_step.py strang 100 C3
