timeout 900 python -m pytest tests/test_fftpass.py tests/test_full_runs.py -m gpu -x -q > gpurun_out/o3_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/o3_pytest.log
tail -n 6 gpurun_out/o3_pytest.log
for v in 1 0 1 0; do echo "CGL_FFT_C32=$v"; CGL_FFT_C32=$v timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "STR_MID" | grep -v "^{"; done
timeout 300 python tools/prof_step.py strang 100 C3
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sharded_fourier or slab_sharded" 2>&1 | tail -2
