for pf in 0 148 296 592 1184; do echo "PF=$pf"; CGL_FFT_R32_PF=$pf timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "G axis" | grep -v "^{"; done
