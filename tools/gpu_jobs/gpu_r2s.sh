python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/s_build.log 2>&1
timeout 900 python -m pytest tests/test_fftpass.py -m gpu -x -q > gpurun_out/s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s_pytest.log
tail -n 5 gpurun_out/s_pytest.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/s_probe.log 2>&1; grep -v "^{" gpurun_out/s_probe.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fft_pass_kernel|fft_strided" -c 14 -o gpurun_out/s_pass_full python tools/fft_probe.py 512 --ncu > gpurun_out/s_ncu_full.log 2>&1
ncu -i gpurun_out/s_pass_full.ncu-rep --page raw --csv > gpurun_out/s_pass_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/s_pass_raw.csv > gpurun_out/s_pass_stalls.txt
