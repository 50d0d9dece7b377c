timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e3_launch_if4.csv python tools/prof_step.py if4 3 C3 > gpurun_out/e3_ncu_if4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e3_launch_strang.csv python tools/prof_step.py strang 3 C3 > gpurun_out/e3_ncu_strang.log 2>&1
python tools/summarize_launches.py gpurun_out/e3_launch_if4.csv > gpurun_out/e3_launch_if4.txt
python tools/summarize_launches.py gpurun_out/e3_launch_strang.csv > gpurun_out/e3_launch_strang.txt
cat gpurun_out/e3_launch_if4.txt gpurun_out/e3_launch_strang.txt
timeout 300 python tools/fft_probe.py 512 > gpurun_out/e3_probe.log 2>&1; grep -v "^{" gpurun_out/e3_probe.log
