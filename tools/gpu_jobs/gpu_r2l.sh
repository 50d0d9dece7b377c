python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/l_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/l_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/l_pytest.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/l_probe.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/l_bench.log 2>&1; echo "rc=$?" >> gpurun_out/l_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launch_if4.csv python tools/prof_step.py if4 3 C3 > gpurun_out/l_ncu_if4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_launch_strang.csv python tools/prof_step.py strang 3 C3 > gpurun_out/l_ncu_strang.log 2>&1
python tools/summarize_launches.py gpurun_out/l_launch_if4.csv > gpurun_out/l_launch_if4.txt
python tools/summarize_launches.py gpurun_out/l_launch_strang.csv > gpurun_out/l_launch_strang.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft_ -c 14 -o gpurun_out/l_fft_full python tools/fft_probe.py 512 --ncu > gpurun_out/l_ncu_full.log 2>&1
tail -n 3 gpurun_out/l_pytest.log; head -14 gpurun_out/l_probe.log; cut -c1-400 gpurun_out/l_bench.log; cat gpurun_out/l_launch_if4.txt gpurun_out/l_launch_strang.txt
