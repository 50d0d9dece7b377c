set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/g_pytest.log
timeout 600 python bench.py > gpurun_out/g_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/g_bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/g_ref.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/g_smoke.log 2>&1
bash tools/all_configs.sh > gpurun_out/g_configs.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/g_launches.csv python tools/prof_step.py if4 40 > gpurun_out/g_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ozgemm_persistent|rows_slice" --launch-skip 40 -c 8 -o gpurun_out/g_full python tools/prof_step.py if4 40 > gpurun_out/g_ncu2.log 2>&1
tail -n 3 gpurun_out/g_pytest.log gpurun_out/g_bench.log gpurun_out/g_ref.log gpurun_out/g_smoke.log
