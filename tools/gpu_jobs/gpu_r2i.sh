python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/i_build.log 2>&1
CGL_FFT_NT=512 timeout 300 python tools/fft_probe.py 512 > gpurun_out/i_probe512.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launch_if4.csv python tools/prof_step.py if4 3 C3 > gpurun_out/i_ncu_if4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_launch_strang.csv python tools/prof_step.py strang 3 C3 > gpurun_out/i_ncu_strang.log 2>&1
python tools/summarize_launches.py gpurun_out/i_launch_if4.csv > gpurun_out/i_launch_if4.txt
python tools/summarize_launches.py gpurun_out/i_launch_strang.csv > gpurun_out/i_launch_strang.txt
head -14 gpurun_out/i_probe512.log; cat gpurun_out/i_launch_if4.txt gpurun_out/i_launch_strang.txt
