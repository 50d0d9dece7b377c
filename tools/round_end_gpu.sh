# Round-end GPU pass on one B200 (what the numbers in DESIGN.md / profiles/ come from):
#   gpurun --timeout 3000 -- 'bash tools/round_end_gpu.sh'
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/end_build.log 2>&1
CGL_FULLRUN_LOG=gpurun_out/end_fullruns.jsonl timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/end_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/end_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/end_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/end_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/end_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/end_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/end_ref.log
timeout 300 python tools/fft_probe.py 512 > gpurun_out/end_probe.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/end_launch_if4.csv python tools/prof_step.py if4 3 C3 > gpurun_out/end_ncu_if4.log 2>&1
python tools/summarize_launches.py gpurun_out/end_launch_if4.csv > gpurun_out/end_launch_if4.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fft_" -c 16 -o gpurun_out/end_fft_full python tools/fft_probe.py 512 --ncu > gpurun_out/end_ncu_full.log 2>&1
ncu -i gpurun_out/end_fft_full.ncu-rep --page raw --csv > gpurun_out/end_fft_raw.csv 2>/dev/null
python tools/ncu_stalls.py gpurun_out/end_fft_raw.csv > gpurun_out/end_fft_stalls.txt
tail -n 3 gpurun_out/end_pytest.log gpurun_out/end_smoke.log; cut -c1-400 gpurun_out/end_bench.log gpurun_out/end_ref.log; cat gpurun_out/end_launch_if4.txt
