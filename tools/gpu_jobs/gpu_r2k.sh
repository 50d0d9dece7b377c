python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/k_build.log 2>&1
timeout 300 python tools/fft_probe.py 512 > gpurun_out/k_probe.log 2>&1
for v in gv1 gv2 sv1 sv2; do CGL_LIB_OVERRIDE=$PWD/tmp_ab/lib$v.so timeout 300 python tools/fft_probe.py 512 > gpurun_out/k_probe_$v.log 2>&1; done
head -14 gpurun_out/k_probe.log; grep -H "G axis\|STR_A0" gpurun_out/k_probe_*.log
