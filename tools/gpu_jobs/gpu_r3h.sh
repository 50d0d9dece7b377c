for nt in 0 1024; do echo "NT=$nt"; CGL_FFT_NT=$nt timeout 300 python tools/fft_probe.py 512 2>&1 | grep -E "plain (fwd|inv) axis [01]" | grep -v "^{"; done
