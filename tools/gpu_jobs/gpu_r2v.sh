python -c "from paper_2403_02816_b200 import _build; _build.build()" > gpurun_out/v_build.log 2>&1
timeout 1200 python tools/project_sharded.py 1 2 4 8 > gpurun_out/v_project.log 2>&1; echo "rc=$?" >> gpurun_out/v_project.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/v_bench.log 2>&1; echo "rc=$?" >> gpurun_out/v_bench.log
tail -n 30 gpurun_out/v_project.log; cut -c1-700 gpurun_out/v_bench.log
