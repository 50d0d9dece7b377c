for v in 1 0 1 0; do echo "CGL_FFT_R32A=$v"; CGL_FFT_R32A=$v timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "STR_A0F" | grep -v "^{"; done
timeout 900 python -m pytest tests/test_fftpass.py tests/test_full_runs.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/prof_step.py strang 100 C3
