CGL_FFT_R32=2 timeout 900 python -m pytest tests/test_fftpass.py -m gpu -x -q > gpurun_out/z_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/z_pytest.log
tail -n 12 gpurun_out/z_pytest.log
for m in 0 1 2; do echo "CGL_FFT_R32=$m"; CGL_FFT_R32=$m timeout 300 python tools/fft_probe.py 512 > gpurun_out/z_probe$m.log 2>&1; grep -E "plain (fwd|inv) axis [01]|G axis" gpurun_out/z_probe$m.log | grep -v "^{"; done
timeout 600 python -m pytest tests/test_full_runs.py -m gpu -x -q -k "C3" > gpurun_out/z_full.log 2>&1; tail -n 5 gpurun_out/z_full.log
