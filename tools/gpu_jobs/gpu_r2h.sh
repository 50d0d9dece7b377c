python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/h_build.log 2>&1
timeout 900 python -m pytest tests/test_fftpass.py tests/test_gpu_parity.py -k "fft or C3 or Fourier or fourier" -x -q > gpurun_out/h_fft_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/h_fft_pytest.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/h_probe.log 2>&1; echo "rc=$?" >> gpurun_out/h_probe.log
timeout 600 python bench.py --steps 2 --warmup 2 --no-extras > gpurun_out/h_bench.log 2>&1; echo "rc=$?" >> gpurun_out/h_bench.log
timeout 600 python bench.py --steps 2 --warmup 2 --no-extras --scheme strang > gpurun_out/h_bench_strang.log 2>&1; echo "rc=$?" >> gpurun_out/h_bench_strang.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_pass_kernel -c 20 -o gpurun_out/h_fft_full python tools/fft_probe.py 512 --ncu > gpurun_out/h_ncu.log 2>&1
tail -n 3 gpurun_out/h_fft_pytest.log; head -14 gpurun_out/h_probe.log; cut -c1-300 gpurun_out/h_bench.log gpurun_out/h_bench_strang.log; tail -3 gpurun_out/h_ncu.log
