nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/b_build.log 2>&1
timeout 900 python -m pytest tests/test_fftpass.py -x -q > gpurun_out/b_fft_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/b_fft_pytest.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/b_probe.log 2>&1; echo "rc=$?" >> gpurun_out/b_probe.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "C3 or fourier or Fourier or stepper" > gpurun_out/b_c3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/b_c3_pytest.log
timeout 600 python bench.py --steps 2 --warmup 2 --no-extras > gpurun_out/b_bench.log 2>&1; echo "rc=$?" >> gpurun_out/b_bench.log

tail -n 4 gpurun_out/b_fft_pytest.log gpurun_out/b_c3_pytest.log; cat gpurun_out/b_probe.log | head -20; cut -c1-400 gpurun_out/b_bench.log gpurun_out/b_bench_strang.log
CGL_FFT_NT=512 timeout 300 python tools/fft_probe.py 512 > gpurun_out/b_probe512.log 2>&1
head -14 gpurun_out/b_probe512.log
