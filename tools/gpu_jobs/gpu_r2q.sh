python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/q_build.log 2>&1
timeout 600 python -m pytest tests/test_fftpass.py -m gpu -x -q -k "plane" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
tail -n 30 gpurun_out/q_pytest.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/q_probe.log 2>&1; grep -v "^{" gpurun_out/q_probe.log
CGL_PLANE_NT=512 timeout 300 python tools/fft_probe.py 512 > gpurun_out/q_probe512.log 2>&1; grep "PLANE" gpurun_out/q_probe512.log
CGL_PLANE_LAG=1 timeout 300 python tools/fft_probe.py 512 > gpurun_out/q_probe_lag1.log 2>&1; grep "PLANE" gpurun_out/q_probe_lag1.log
CGL_PLANE_LAG=4 timeout 300 python tools/fft_probe.py 512 > gpurun_out/q_probe_lag4.log 2>&1; grep "PLANE" gpurun_out/q_probe_lag4.log
timeout 300 python tools/prof_step.py if4 10 C3; timeout 300 python tools/prof_step.py strang 10 C3
