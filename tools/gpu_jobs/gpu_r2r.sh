python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/r_build.log 2>&1
timeout 600 python -m pytest tests/test_fftpass.py -m gpu -x -q -k "plane" > gpurun_out/r_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r_pytest.log
tail -n 5 gpurun_out/r_pytest.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/r_probe.log 2>&1; grep "PLANE" gpurun_out/r_probe.log
CGL_PLANE_NT=512 timeout 300 python tools/fft_probe.py 512 > gpurun_out/r_probe512.log 2>&1; grep "PLANE" gpurun_out/r_probe512.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft_plane -c 4 -o gpurun_out/r_plane_full python tools/fft_probe.py 512 --ncu > gpurun_out/r_ncu_full.log 2>&1
ncu -i gpurun_out/r_plane_full.ncu-rep --page raw --csv > gpurun_out/r_plane_raw.csv 2>/dev/null
ls -la gpurun_out/
