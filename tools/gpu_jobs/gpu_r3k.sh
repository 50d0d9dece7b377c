for cp in 8 4 8 4; do echo "CP=$cp"; CGL_R32_CP=$cp timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "G axis" | grep -v "^{"; done
CGL_R32_CP=4 timeout 300 python -m pytest tests/test_fftpass.py -m gpu -x -q -k "fused_g" 2>&1 | tail -2
